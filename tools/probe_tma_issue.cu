// Probe: cost of issuing TMA tensor loads from one thread (B200, sm_100a).
// Measures cycles per UTMALDG issue and per completed load for a few box
// shapes, with the tensor map in kernel-parameter space (__grid_constant__)
// or in global memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2002_02145_b200/csrc \
//        tools/probe_tma_issue.cu -o tools/probe_tma_issue -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100_ptx.cuh"

using namespace psconv;

constexpr int kLoads = 32;

template <int RANK>
__device__ void issue(const CUtensorMap* m, void* dst, uint64_t* bar, int i) {
  if constexpr (RANK == 3) ptx::tma_load_3d(dst, m, bar, 0, (i & 7) * 64, i);
  else ptx::tma_load_5d(dst, m, bar, 0, (i & 3) * 8, (i & 7) * 4, 0, i & 15);
}

template <int RANK>
__global__ void probe(const __grid_constant__ CUtensorMap pm, const CUtensorMap* gm, int use_global,
                      uint32_t box_bytes, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const CUtensorMap* m = use_global ? gm : &pm;
    ptx::prefetch_tmap(m);
    // warm: one load
    ptx::mbar_expect_tx(&bar, box_bytes);
    issue<RANK>(m, smem, &bar, 0);
    ptx::mbar_wait(&bar, 0);
    uint32_t phase = 1;
    long long t0 = clock64();
    ptx::mbar_expect_tx(&bar, box_bytes * kLoads);
    for (int i = 0; i < kLoads; ++i) issue<RANK>(m, smem + (i & 1) * 32768, &bar, i);
    long long t1 = clock64();
    ptx::mbar_wait(&bar, phase);
    long long t2 = clock64();
    phase ^= 1;
    // dependent round trips: issue one, wait, repeat
    long long t3 = clock64();
    for (int i = 0; i < 8; ++i) {
      ptx::mbar_expect_tx(&bar, box_bytes);
      issue<RANK>(m, smem, &bar, i);
      ptx::mbar_wait(&bar, phase);
      phase ^= 1;
    }
    long long t4 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
      out[2] = (t4 - t3) / 8;
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fnp);
  float* buf;
  cudaMalloc(&buf, 64 << 20);
  cudaMemset(buf, 0, 64 << 20);
  long long* out;
  cudaMalloc(&out, 64);
  CUtensorMap* gm;
  cudaMalloc(&gm, sizeof(CUtensorMap));
  for (int grid : {1, 148}) {
    // 3D filter-like boxes {16, rows, 1}
    for (int rows : {8, 32, 64, 128}) {
      CUtensorMap m;
      cuuint64_t dims[3] = {16, 512, 4096};
      cuuint64_t str[2] = {64, 512 * 64};
      cuuint32_t box[3] = {16, cuuint32_t(rows), 1};
      cuuint32_t es[3] = {1, 1, 1};
      enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
      for (int g = 0; g < 2; ++g) {
        cudaFuncSetAttribute(probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        probe<3><<<grid, 32, 96 * 1024>>>(m, gm, g, rows * 64, out);
        long long h[3];
        cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
        printf("grid %3d 3D box 16x%-3d (%6d B) %s: issue %6.1f cyc/load, complete %7.1f cyc/load, round trip %6lld cyc\n",
               grid, rows, rows * 64, g ? "global" : "param ", double(h[0]) / kLoads, double(h[1]) / kLoads, h[2]);
      }
    }
    // 128-B rows (32 fp32, SWIZZLE_128B) and 16-B rows (4 fp32, no swizzle)
    for (int inner : {32, 4}) {
      for (int rows : {16, 32, 64}) {
        CUtensorMap m;
        cuuint64_t dims[3] = {cuuint64_t(inner), 512, 1024};
        cuuint64_t str[2] = {cuuint64_t(inner) * 4, 512ull * inner * 4};
        cuuint32_t box[3] = {cuuint32_t(inner), cuuint32_t(rows), 1};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         inner == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
          printf("encode failed %d\n", r);
          continue;
        }
        const int bytes = rows * inner * 4;
        probe<3><<<grid, 32, 96 * 1024>>>(m, gm, 0, bytes, out);
        long long h[3];
        cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
        printf("grid %3d 3D box %dx%-3d (%6d B): issue %6.1f cyc/load, complete %7.1f cyc/load, round trip %6lld cyc\n",
               grid, inner, rows, bytes, double(h[0]) / kLoads, double(h[1]) / kLoads, h[2]);
      }
    }
    // 5D activation-like boxes [16][Q][P][1][N]
    const int shapes[5][3] = {{8, 4, 4}, {8, 8, 2}, {8, 16, 1}, {2, 1, 64}, {16, 8, 1}};
    for (const auto& shp : shapes) {
      CUtensorMap m;
      cuuint64_t dims[5] = {16, 64, 64, 4, 128};
      cuuint64_t str[4] = {64, 64 * 64, 64 * 64 * 64, 4ull * 64 * 64 * 64};
      cuuint32_t box[5] = {16, cuuint32_t(shp[0]), cuuint32_t(shp[1]), 1, cuuint32_t(shp[2])};
      cuuint32_t es[5] = {1, 1, 1, 1, 1};
      CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, buf, dims, str, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", r);
        continue;
      }
      cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
      const int bytes = 64 * shp[0] * shp[1] * shp[2];
      for (int g = 0; g < 2; ++g) {
        cudaFuncSetAttribute(probe<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        probe<5><<<grid, 32, 96 * 1024>>>(m, gm, g, bytes, out);
        long long h[3];
        cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
        printf("grid %3d 5D box %dx%dx%d (%6d B) %s: issue %6.1f cyc/load, complete %7.1f cyc/load, round trip %6lld cyc\n",
               grid, shp[0], shp[1], shp[2], bytes, g ? "global" : "param ", double(h[0]) / kLoads,
               double(h[1]) / kLoads, h[2]);
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
