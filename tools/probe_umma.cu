// Probe: one tcgen05.mma kind::tf32 (M=128, N=16, K=8 x2) from manually filled
// SWIZZLE_64B smem, and the same tiles loaded with TMA. Prints max error.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../paper_2002_02145_b200/csrc/sm100_ptx.cuh"
using namespace psconv;

__device__ uint32_t swz(uint32_t off) { return off ^ (((off >> 7) & 3) << 4); }

template <int N>
__global__ void k_probe(const float* A, const float* B, float* D, int mode, uint32_t idesc_override,
                        float* smem_dump, const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sa = sm;             // 128 x 64 B = 8 KB
  uint8_t* sb = sm + 8192;      // 16 x (N*4) bytes, atoms of 16 n at 1024 B
  uint64_t* bar = (uint64_t*)(sm + 8192 + 16 * 1024);
  uint32_t* slot = (uint32_t*)(bar + 4);
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar[0], 1); ptx::mbar_init(&bar[1], 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(slot, 32);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  uint32_t tmem = *slot;
  if (mode == 0) {
    for (int i = threadIdx.x; i < 128 * 16; i += blockDim.x) {
      int m = i / 16, k = i % 16;
      *(float*)(sa + swz(m * 64 + k * 4)) = A[i];
    }
    for (int i = threadIdx.x; i < 16 * N; i += blockDim.x) {
      int k = i / N, n = i % N;
      int atom = n / 16, nn = n % 16;
      *(float*)(sb + atom * 1024 + swz(k * 64 + nn * 4)) = B[i];
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
  } else {
    if (threadIdx.x == 0) {
      ptx::mbar_expect_tx(&bar[0], 8192 + 16 * N * 4);
      ptx::tma_load_4d(sa, &ta, &bar[0], 0, 0, 0, 0);
      ptx::tma_load_4d(sb, &tb, &bar[0], 0, 0, 0, 0);
    }
    ptx::mbar_wait(&bar[0], 0);
  }
  if (threadIdx.x < 128) {
    // dump raw smem A (first 8 KB) for inspection
    for (int i = threadIdx.x; i < 2048; i += 128) smem_dump[i] = ((float*)sa)[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::tc_fence_after();
    uint32_t idesc = idesc_override ? idesc_override : ptx::idesc_tf32_m128<N>();
    uint32_t a = ptx::smem_u32(sa), b = ptx::smem_u32(sb);
    for (int h = 0; h < 2; ++h) {
      uint64_t da = ptx::smem_desc_sw64(a + h * 32, 16, 512);
      uint64_t db = ptx::smem_desc_sw64(b + h * 512, 1024, 512);
      ptx::mma_tf32(tmem, da, db, idesc, h);
    }
    ptx::mma_commit(&bar[1]);
  }
  __syncwarp();
  ptx::mbar_wait(&bar[1], 0);
  ptx::tc_fence_after();
  if (warp < 4) {
    uint32_t v[16];
    ptx::tmem_ld16(tmem + ((warp * 32) << 16), v);
    ptx::tmem_wait_ld();
    int m = warp * 32 + lane;
    for (int j = 0; j < 16; ++j) D[m * N + j] = __uint_as_float(v[j]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 32); }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int N = 16;
  float hA[128 * 16], hB[16 * N], hD[128 * N], ref[128 * N], dump[2048];
  for (int i = 0; i < 128 * 16; ++i) hA[i] = (float)((i * 37) % 17 - 8) / 8.0f;
  for (int i = 0; i < 16 * N; ++i) hB[i] = (float)((i * 11) % 13 - 6) / 4.0f;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) { double s = 0; for (int k = 0; k < 16; ++k) s += hA[m * 16 + k] * hB[k * N + n]; ref[m * N + n] = s; }
  float *A, *B, *D, *dd;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD); cudaMalloc(&dd, sizeof dump);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  void* fnp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeTiledFn enc = (EncodeTiledFn)fnp;
  CUtensorMap ta, tb;
  { cuuint64_t dims[4] = {16, 128, 1, 1}; cuuint64_t st[3] = {64, 8192, 8192}; cuuint32_t box[4] = {16, 128, 1, 1}; cuuint32_t es[4] = {1,1,1,1};
    printf("encA %d\n", enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, A, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)); }
  { cuuint64_t dims[4] = {16, 16, 1, 1}; cuuint64_t st[3] = {64, 1024, 1024}; cuuint32_t box[4] = {16, 16, 1, 1}; cuuint32_t es[4] = {1,1,1,1};
    printf("encB %d\n", enc(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, B, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)); }
  cudaFuncSetAttribute(k_probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  uint32_t overrides[] = {0u, 0u};
  for (int mode = 0; mode < 2; ++mode) {
    for (uint32_t ov : {0u, (ptx::idesc_tf32_m128<N>() & ~(0x1Fu << 24)) | ((128u >> 4) << 23)}) {
      cudaMemset(D, 0, sizeof hD);
      k_probe<N><<<1, 128, 64 * 1024>>>(A, B, D, mode, ov, dd, ta, tb);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
      cudaMemcpy(dump, dd, sizeof dump, cudaMemcpyDeviceToHost);
      double mx = 0, mref = 0; int nz = 0;
      for (int i = 0; i < 128 * N; ++i) { mx = fmax(mx, fabs(hD[i] - ref[i])); mref = fmax(mref, fabs(ref[i])); nz += hD[i] != 0; }
      printf("mode=%d idesc=%08x err=%s maxerr=%g maxref=%g nonzero=%d D[0..3]=%g %g %g %g ref=%g %g %g %g smemA[0..3]=%g %g %g %g\n", mode,
             ov ? ov : ptx::idesc_tf32_m128<N>(), cudaGetErrorString(e), mx, mref, nz, hD[0], hD[1], hD[2], hD[3], ref[0], ref[1], ref[2], ref[3], dump[0], dump[1], dump[2], dump[3]);
      if (e != cudaSuccess) return 1;
    }
  }
  (void)overrides;
  return 0;
}
