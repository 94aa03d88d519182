// Probe: tcgen05.mma kind::tf32 rate for the CTA pair (cta_group::2, M = 256) vs a single
// CTA (M = 128), N = 64 / 128 / 256, A from shared memory (SS) or tensor memory (TS).
// Cycles per MMA on the leader; per-SM work of one pair MMA = one single-CTA MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2002_02145_b200/csrc \
//        tools/probe_mma_pair.cu -o tools/probe_mma_pair
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100_ptx.cuh"
using namespace psconv;

__device__ __forceinline__ void mma_tf32_pair_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                                 uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

template <int N, bool PAIR, bool TS>
__global__ void __cluster_dims__(2, 1, 1) k_rate(int n_mma, long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  const unsigned rank = blockIdx.x & 1;
  for (int i = threadIdx.x; i < (64 * 1024) / 4; i += blockDim.x) ((float*)sm)[i] = 0.f;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) {
    if (PAIR) ptx::tmem_alloc_pair(&slot, 512);
    else ptx::tmem_alloc(&slot, 512);
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync_all();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0 && (!PAIR || rank == 0)) {
    const uint32_t idesc = ptx::idesc_tf32_m128<N, PAIR ? 256 : 128>();
    const uint64_t da = ptx::smem_desc_sw64(ptx::smem_u32(sm), 16, 512);
    const uint64_t db = ptx::smem_desc_sw64(ptx::smem_u32(sm + 16384), 16, 512);
    const uint32_t ta = tmem + 256;  // A columns after the N <= 256 accumulator
    long long t0 = clock64();
    for (int it = 0; it < n_mma; it += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (PAIR) {
          if (TS) mma_tf32_pair_ts(tmem, ta + 8 * (u & 1), db + 2 * (u & 1), idesc, 1u);
          else ptx::mma_tf32_pair(tmem, da + 2 * (u & 1), db + 2 * (u & 1), idesc, 1u);
        } else {
          if (TS) ptx::mma_tf32_ts(tmem, ta + 8 * (u & 1), db + 2 * (u & 1), idesc, 1u);
          else ptx::mma_tf32(tmem, da + 2 * (u & 1), db + 2 * (u & 1), idesc, 1u);
        }
      }
    }
    if (PAIR) ptx::mma_commit_pair(&bar);
    else ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0) out[0] = t2 - t0;
  }
  if (PAIR && rank == 1 && threadIdx.x == 0) ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync_all();
  if (warp == 0) {
    ptx::tc_fence_after();
    if (PAIR) ptx::tmem_dealloc_pair(tmem, 512);
    else ptx::tmem_dealloc(tmem, 512);
  }
}

template <int N, bool PAIR, bool TS>
void run(int grid) {
  long long* out;
  cudaMalloc(&out, 16);
  cudaFuncSetAttribute(k_rate<N, PAIR, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  const int n = 1024;
  k_rate<N, PAIR, TS><<<grid, 128, 80 * 1024>>>(n, out);
  k_rate<N, PAIR, TS><<<grid, 128, 80 * 1024>>>(n, out);
  long long h;
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("grid %3d %s %s N=%3d: %6.1f cyc per MMA (%s rows), ideal per SM %d\n", grid, PAIR ? "pair  " : "single",
         TS ? "TS" : "SS", N, double(h) / n, PAIR ? "256" : "128", 128 * N * 8 * 2 / 4096);
  cudaFree(out);
}

int main() {
  for (int grid : {2, 148}) {
    run<64, false, false>(grid);
    run<64, true, false>(grid);
    run<64, false, true>(grid);
    run<64, true, true>(grid);
    run<128, false, false>(grid);
    run<128, true, false>(grid);
    run<128, true, true>(grid);
    run<256, false, false>(grid);
    run<256, true, false>(grid);
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
