// Probe: how TMA lays out a box whose inner dimension (64 B = 16 fp32) is smaller than the
// swizzle span, for CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B / _128B / _64B: box {16, 2, 4, 2}
// over a [2 blocks][4 rows][16] view (value = element index), smem dumped with a sentinel
// past the box's dense size.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>
#include "../paper_2002_02145_b200/csrc/sm100_ptx.cuh"
using namespace psconv;

__global__ void k(const __grid_constant__ CUtensorMap m, float* out, int nfloats) {
  extern __shared__ __align__(1024) uint8_t raw[];
  float* sm = reinterpret_cast<float*>(raw);
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < nfloats; i += blockDim.x) sm[i] = -1.f;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  ptx::fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_expect_tx(&bar, 16 * 2 * 4 * 2 * 4);
    ptx::tma_load_4d(sm, &m, &bar, 0, 0, 0, 0);
  }
  ptx::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < nfloats; i += blockDim.x) out[i] = sm[i];
}

__global__ void k2(const __grid_constant__ CUtensorMap m, float* out, int nfloats) {
  extern __shared__ __align__(1024) uint8_t raw[];
  float* sm = reinterpret_cast<float*>(raw);
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < nfloats; i += blockDim.x) sm[i] = -1.f;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  ptx::fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_expect_tx(&bar, 2 * 16 * 4 * 2 * 4);
    ptx::tma_load_4d(sm, &m, &bar, 0, 0, 0, 0);        // block 0
    ptx::tma_load_4d(sm + 16, &m, &bar, 0, 1, 0, 0);   // block 1 at +64 B
  }
  ptx::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < nfloats; i += blockDim.x) out[i] = sm[i];
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  // global: [row 4][block 2][16] is NOT the order we want; use [block 2][row 8][16] and view dims
  // {16 c, 2 block (stride 8*64), 4 row (stride 64), 2 group (stride 4*64)}
  std::vector<float> h(2 * 8 * 16);
  for (size_t i = 0; i < h.size(); ++i) h[i] = float(i);
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  const int nf = 1024;
  cudaMalloc(&o, nf * 4);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = (Enc)fp;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  const char* names[] = {"128B_ATOM_32B", "128B", "64B"};
  CUtensorMapSwizzle sw[] = {CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_SWIZZLE_64B};
  for (int t = 0; t < 3; ++t) {
    CUtensorMap m;
    const cuuint64_t dims[4] = {16, 2, 4, 2};
    const cuuint64_t strides[3] = {8 * 64, 64, 4 * 64};
    const cuuint32_t box[4] = {16, 2, 4, 2};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     sw[t], CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("== %s encode=%d\n", names[t], (int)r);
    if (r) continue;
    cudaMemset(o, 0, nf * 4);
    k<<<1, 128, 8192>>>(m, o, nf);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> got(nf);
    cudaMemcpy(got.data(), o, nf * 4, cudaMemcpyDeviceToHost);
    printf("err=%s\n", cudaGetErrorString(e));
    // print per 128-B row: the source index of each 16-B chunk's first element
    for (int row = 0; row < 24; ++row) {
      printf("row %2d:", row);
      for (int c = 0; c < 8; ++c) printf(" %5.0f", got[row * 32 + c * 4]);
      printf("\n");
    }
  }
  {
    CUtensorMap m;
    const cuuint64_t dims[4] = {16, 2, 4, 2};
    const cuuint64_t strides[3] = {8 * 64, 64, 4 * 64};
    const cuuint32_t box[4] = {16, 1, 4, 2};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("== two boxes, +64 B: encode=%d\n", (int)r);
    cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
    cudaMemset(o, 0, nf * 4);
    k2<<<1, 128, 8192>>>(m, o, nf);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> got(nf);
    cudaMemcpy(got.data(), o, nf * 4, cudaMemcpyDeviceToHost);
    printf("err=%s\n", cudaGetErrorString(e));
    for (int row = 0; row < 12; ++row) {
      printf("row %2d:", row);
      for (int c = 0; c < 8; ++c) printf(" %5.0f", got[row * 32 + c * 4]);
      printf("\n");
    }
  }
  return 0;
}
