// Probe: can a tcgen05.mma kind::tf32 K-major SWIZZLE_64B A operand start at an
// arbitrary 64-B row of a swizzled tile (row shift s), and what must the
// descriptor's matrix-base-offset field (bits 49-51) hold?  This decides whether
// a 3x3 stride-1 convolution can load the input halo once and address the nine
// (kj, ki) shifted operands in place.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2002_02145_b200/csrc \
//        tools/probe_shift.cu -o tools/probe_shift
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>

#include "sm100_ptx.cuh"
using namespace psconv;

constexpr int kRows = 256, N = 16;

__device__ uint32_t swz(uint32_t off) { return off ^ (((off >> 7) & 3) << 4); }

__global__ void k_shift(const float* A, const float* B, float* D, int shift, int base_mode) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sa = sm;                  // kRows x 64 B
  uint8_t* sb = sm + kRows * 64;     // 16 x 64 B (K-major B: n rows of 16 k)
  uint64_t* bar = (uint64_t*)(sb + 1024);
  uint32_t* slot = (uint32_t*)(bar + 2);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(slot, 32);
  for (int i = threadIdx.x; i < kRows * 16; i += blockDim.x) {
    const int m = i / 16, k = i % 16;
    *(float*)(sa + swz(m * 64 + k * 4)) = A[i];
  }
  for (int i = threadIdx.x; i < N * 16; i += blockDim.x) {
    const int n = i / 16, k = i % 16;  // B stored K-major: row n holds k = 0..15
    *(float*)(sb + swz(n * 64 + k * 4)) = B[k * N + n];
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = ptx::idesc_tf32_m128<N>();
    const uint32_t a = ptx::smem_u32(sa) + shift * 64, b = ptx::smem_u32(sb);
    for (int h = 0; h < 2; ++h) {
      uint64_t da = ptx::smem_desc_sw64(a + h * 32, 16, 512);
      uint64_t bo = 0;
      if (base_mode == 1) bo = ((a + h * 32) >> 7) & 7;   // (addr >> 7) & 7
      if (base_mode == 2) bo = ((a + h * 32) >> 6) & 7;   // 64-B row phase
      if (base_mode == 3) bo = ((a + h * 32) >> 7) & 3;
      da |= bo << 49;
      const uint64_t db = ptx::smem_desc_sw64(b + h * 32, 16, 512);
      ptx::mma_tf32(tmem, da, db, idesc, h);
    }
    ptx::mma_commit(&bar[0]);
  }
  __syncwarp();
  ptx::mbar_wait(&bar[0], 0);
  ptx::tc_fence_after();
  if (warp < 4) {
    uint32_t v[16];
    ptx::tmem_ld16(tmem + ((warp * 32) << 16), v);
    ptx::tmem_wait_ld();
    const int m = warp * 32 + lane;
    for (int j = 0; j < 16; ++j) D[m * N + j] = __uint_as_float(v[j]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 32);
  }
}

int main() {
  static float hA[kRows * 16], hB[16 * N], hD[128 * N];
  for (int i = 0; i < kRows * 16; ++i) hA[i] = (float)((i * 37) % 17 - 8) / 8.0f + (float)(i / 16) / 64.0f;
  for (int i = 0; i < 16 * N; ++i) hB[i] = (float)((i * 11) % 13 - 6) / 4.0f;
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA);
  cudaMalloc(&B, sizeof hB);
  cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_shift, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int base_mode = 0; base_mode < 4; ++base_mode) {
    for (int shift : {0, 1, 2, 3, 4, 5, 7, 8, 9, 58, 61}) {
      cudaMemset(D, 0, sizeof hD);
      k_shift<<<1, 128, 64 * 1024>>>(A, B, D, shift, base_mode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
      // reference with tf32-truncated operands is within ~1e-3 of fp32; use a loose check
      double mx = 0;
      int bad_rows = 0;
      for (int m = 0; m < 128; ++m) {
        double row_err = 0;
        for (int n = 0; n < N; ++n) {
          double s = 0;
          for (int k = 0; k < 16; ++k) s += (double)hA[(m + shift) * 16 + k] * hB[k * N + n];
          row_err = fmax(row_err, fabs(s - hD[m * N + n]));
        }
        mx = fmax(mx, row_err);
        bad_rows += row_err > 0.05;
      }
      printf("base_mode %d shift %2d: max err %.4g, bad rows %d\n", base_mode, shift, mx, bad_rows);
    }
  }
  return 0;
}
