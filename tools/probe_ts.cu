// Probe: tcgen05.mma kind::tf32 with the A operand in tensor memory (written by
// tcgen05.st, lane = row, 16 fp32 columns = K) and B K-major SWIZZLE_64B in
// shared memory; also times back-to-back TS MMAs (N = 64 / 128).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2002_02145_b200/csrc \
//        tools/probe_ts.cu -o tools/probe_ts
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>

#include "sm100_ptx.cuh"
using namespace psconv;

__device__ uint32_t swz(uint32_t off) { return off ^ (((off >> 7) & 3) << 4); }

template <int N>
__global__ void k_ts(const float* A, const float* B, float* D, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sb = sm;  // N rows x 64 B (K-major B)
  __shared__ uint64_t bar[2];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::mbar_init(&bar[1], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(&slot, 512);
  for (int i = threadIdx.x; i < N * 16; i += blockDim.x) {
    const int n = i / 16, k = i % 16;
    *(float*)(sb + swz(n * 64 + k * 4)) = B[k * N + n];
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t a_col = 256;  // A at columns 256..271
  {
    const int m = warp * 32 + lane;
    uint32_t v[16];
    for (int k = 0; k < 16; ++k) v[k] = __float_as_uint(A[m * 16 + k]);
    ptx::tmem_st16(tmem + ((warp * 32) << 16) + a_col, v);
    ptx::tmem_wait_st();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = ptx::idesc_tf32_m128<N>();
    const uint32_t b = ptx::smem_u32(sb);
    for (int h = 0; h < 2; ++h)
      ptx::mma_tf32_ts(tmem, tmem + a_col + 8 * h, ptx::smem_desc_sw64(b + h * 32, 16, 512), idesc, h);
    ptx::mma_commit(&bar[0]);
    ptx::mbar_wait(&bar[0], 0);
    // rate: 256 TS MMAs into columns 0..N-1
    long long t0 = clock64();
    for (int i = 0; i < 256; ++i)
      ptx::mma_tf32_ts(tmem + 128, tmem + a_col + 8 * (i & 1), ptx::smem_desc_sw64(b + (i & 1) * 32, 16, 512),
                       idesc, 1u);
    ptx::mma_commit(&bar[1]);
    ptx::mbar_wait(&bar[1], 0);
    cyc[0] = clock64() - t0;
  }
  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  {
    uint32_t v[16];
    for (int j = 0; j < N / 16; ++j) {
      ptx::tmem_ld16(tmem + ((warp * 32) << 16) + j * 16, v);
      ptx::tmem_wait_ld();
      const int m = warp * 32 + lane;
      for (int c = 0; c < 16; ++c) D[m * N + j * 16 + c] = __uint_as_float(v[c]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// two k-steps from two TMEM slots (cols 192 / 224) into one accumulator
__global__ void k_ts2(const float* A, const float* B, float* D) {
  constexpr int N = 64;
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(&slot, 512);
  for (int t = 0; t < 2; ++t)
    for (int i = threadIdx.x; i < N * 16; i += blockDim.x) {
      const int n = i / 16, k = i % 16;
      *(float*)(sm + t * 4096 + swz(n * 64 + k * 4)) = B[t * 16 * N + k * N + n];
    }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  for (int t = 0; t < 2; ++t) {
    const int m = warp * 32 + lane;
    uint32_t v[16];
    for (int k = 0; k < 16; ++k) v[k] = __float_as_uint(A[t * 128 * 16 + m * 16 + k]);
    ptx::tmem_st16(tmem + ((warp * 32) << 16) + 192 + 32 * t, v);
  }
  ptx::tmem_wait_st();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = ptx::idesc_tf32_m128<N>();
    for (int t = 0; t < 2; ++t)
      for (int h = 0; h < 2; ++h)
        ptx::mma_tf32_ts(tmem, tmem + 192 + 32 * t + 8 * h,
                         ptx::smem_desc_sw64(ptx::smem_u32(sm + t * 4096) + h * 32, 16, 512), idesc, t | h);
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
  }
  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  for (int j = 0; j < N / 16; ++j) {
    uint32_t v[16];
    ptx::tmem_ld16(tmem + ((warp * 32) << 16) + j * 16, v);
    ptx::tmem_wait_ld();
    const int m = warp * 32 + lane;
    for (int c = 0; c < 16; ++c) D[m * N + j * 16 + c] = __uint_as_float(v[c]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

void run2() {
  constexpr int N = 64;
  static float hA[2 * 128 * 16], hB[2 * 16 * N], hD[128 * N];
  for (int i = 0; i < 2 * 128 * 16; ++i) hA[i] = (float)((i * 37) % 17 - 8) / 8.0f;
  for (int i = 0; i < 2 * 16 * N; ++i) hB[i] = (float)((i * 11) % 13 - 6) / 4.0f;
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_ts2, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k_ts2<<<1, 128, 64 * 1024>>>(A, B, D);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int t = 0; t < 2; ++t)
        for (int k = 0; k < 16; ++k) s += (double)hA[t * 2048 + m * 16 + k] * hB[t * 16 * N + k * N + n];
      mx = fmax(mx, fabs(s - hD[m * N + n]));
    }
  printf("two k-steps from TMEM slots 192/224: %s max err %.3g\n", cudaGetErrorString(e), mx);
}

template <int N>
void run() {
  static float hA[128 * 16], hB[16 * N], hD[128 * N];
  // full-mantissa A: tells whether the TS path truncates to tf32 like the SS path
  for (int i = 0; i < 128 * 16; ++i) hA[i] = (float)((i * 37) % 17 - 8) / 8.0f + 1.2345678e-3f * (float)((i * 13) % 7);
  for (int i = 0; i < 16 * N; ++i) hB[i] = (float)((i * 11) % 13 - 6) / 4.0f;
  float *A, *B, *D;
  long long* cyc;
  cudaMalloc(&A, sizeof hA);
  cudaMalloc(&B, sizeof hB);
  cudaMalloc(&D, sizeof hD);
  cudaMalloc(&cyc, 8);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_ts<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k_ts<N><<<1, 128, 64 * 1024>>>(A, B, D, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double mx = 0, mt = 0, mr = 0;
  auto trunc_tf32 = [](float x) { unsigned u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; };
  auto round_tf32 = [](float x) { unsigned u; memcpy(&u, &x, 4); u += 0x1000u; u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; };
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0, st = 0, sr = 0;
      for (int k = 0; k < 16; ++k) {
        s += (double)hA[m * 16 + k] * hB[k * N + n];
        st += (double)trunc_tf32(hA[m * 16 + k]) * hB[k * N + n];
        sr += (double)round_tf32(hA[m * 16 + k]) * hB[k * N + n];
      }
      mx = fmax(mx, fabs(s - hD[m * N + n]));
      mt = fmax(mt, fabs(st - hD[m * N + n]));
      mr = fmax(mr, fabs(sr - hD[m * N + n]));
    }
  printf("N=%d TS mma: %s max err vs fp32 %.3g, vs trunc-tf32 %.3g, vs round-tf32 %.3g, %.1f cyc/mma\n", N,
         cudaGetErrorString(e), mx, mt, mr, c / 256.0);
}

int main() {
  run2();
  run<64>();
  run<128>();
  return 0;
}
