// Probe: throughput of TMA tensor loads of conv input tiles from an NCHW16c
// activation (tensor map dims [16c][W][H][img][Cb], SWIZZLE_64B), one CTA per
// SM, S boxes in flight per CTA. Compares the halo-mode box (whole padded rows,
// starting at w = -1: left/right columns out of bounds) with plain boxes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2002_02145_b200/csrc \
//        tools/probe_halo_tma.cu -o tools/probe_halo_tma
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100_ptx.cuh"
using namespace psconv;

constexpr int N = 256, Cb = 4, H = 56, W = 56;

__global__ void k_load(const __grid_constant__ CUtensorMap m, int loads, int stages, int w0, int bw, int bh,
                       int bn, uint32_t box_bytes, int stride_bytes, int nmax, long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar[16];  // <= 16 stages
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) ptx::mbar_init(&bar[s], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  ptx::prefetch_tmap(&m);
  long long t0 = clock64();
  uint32_t ph = 0;  // phase bits (a register, not a local array)
  for (int i = 0; i < loads; ++i) {
    const int s = i & (stages - 1);  // stages: a power of two
    if (i >= stages) {
      ptx::mbar_wait(&bar[s], (ph >> s) & 1u);
      ph ^= 1u << s;
    }
    // (bit ops only: runtime divisions here would cost more than the loads)
    const int cb = i & 3, hp = (i >> 2) & 7, n = ((i >> 5) + blockIdx.x) & (nmax - 1);
    ptx::mbar_expect_tx(&bar[s], box_bytes);
    ptx::tma_load_5d(sm + s * stride_bytes, &m, &bar[s], 0, w0, hp * bh - (w0 < 0 ? 1 : 0), n * bn, cb);
  }
  for (int i = loads; i < loads + stages; ++i) {
    const int s = i & (stages - 1);
    ptx::mbar_wait(&bar[s], (ph >> s) & 1u);
    ph ^= 1u << s;
  }
  long long t1 = clock64();
  if (blockIdx.x == 0) out[0] = t1 - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fnp);
  float* x;
  const size_t elems = size_t(N) * Cb * H * W * 16;
  cudaMalloc(&x, elems * 4);
  cudaMemset(x, 0, elems * 4);
  long long* out;
  cudaMalloc(&out, 16);
  cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Case {
    const char* name;
    int w0, bw, bh, bn;
  } cases[] = {
      {"halo 58x4 (w0=-1)", -1, 58, 4, 1},
      {"8x4x4", 0, 8, 4, 4},
      {"56x2", 0, 56, 2, 1},
  };
  for (int nmax : {64, 8}) {  // 8 images: the working set stays in L2
   for (int stages : {2, 4, 8})
    for (int grid : {1, 148})
      for (const Case& c : cases) {
        // [16c][W][H][img][Cb] over NCHW16c = [img][Cb][H][W][16]
        cuuint64_t dims[5] = {16, W, H, N, Cb};
        cuuint64_t strides[4] = {64, uint64_t(W) * 64, uint64_t(Cb) * H * W * 64, uint64_t(H) * W * 64};
        cuuint32_t box[5] = {16, cuuint32_t(c.bw), cuuint32_t(c.bh), cuuint32_t(c.bn), 1};
        cuuint32_t es[5] = {1, 1, 1, 1, 1};
        CUtensorMap m;
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, x, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
          printf("%s: encode failed %d\n", c.name, int(r));
          continue;
        }
        const uint32_t bytes = 64u * c.bw * c.bh * c.bn;
        const int stride = (bytes + 1023) / 1024 * 1024;
        const int loads = 64;
        for (int rep = 0; rep < 2; ++rep)
          k_load<<<grid, 32, 16 * 1024 + stages * stride>>>(m, loads, stages, c.w0, c.bw, c.bh, c.bn, bytes, stride,
                                                            nmax, out);
        long long h = 0;
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("stages %2d imgs %3d grid %3d %-20s: %5u B/box, %7.1f cycles/box, %.2f rows/cycle/SM  (%s)\n", stages, nmax, grid,
               c.name, bytes, double(h) / loads, (bytes / 64.0) / (double(h) / loads),
               cudaGetErrorString(cudaGetLastError()));
      }
  }
  return 0;
}
