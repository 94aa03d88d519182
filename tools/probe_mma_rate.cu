// Probe: tcgen05.mma kind::tf32 issue / execution rate from one thread
// (M=128, K=8, N = 64 / 128 / 256), operands in SWIZZLE_64B shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2002_02145_b200/csrc \
//        tools/probe_mma_rate.cu -o tools/probe_mma_rate
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100_ptx.cuh"
using namespace psconv;

template <int N, int UNROLL, int NACC = 1, int M = 128>
__global__ void k_rate(int iters, long long* out, int shift, int boff) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (64 * 1024) / 4; i += blockDim.x) ((float*)sm)[i] = 0.f;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(&slot, 256);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = ptx::idesc_tf32_m128<N, M>();
    // A may start `shift` 64-B rows into the swizzled tile (halo-mode operands)
    // shift < 0: walk the nine 3x3 halo taps (row offsets kj*58 + ki) two MMAs per tap
    // (compile-time offsets); boff: B tile offset in smem
    const uint64_t da0 = ptx::smem_desc_sw64(ptx::smem_u32(sm), 16, 512);
    const uint64_t da = da0 + ((max(shift, 0) * 64) >> 4);
    const uint64_t db = ptx::smem_desc_sw64(ptx::smem_u32(sm + boff), 16, 512);
    long long t0 = clock64();
    if (shift < 0) {
      for (int it = 0; it < 14; ++it) {  // 252 MMAs (~256)
#pragma unroll
        for (int tap = 0; tap < 9; ++tap)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            ptx::mma_tf32(tmem, da0 + ((((tap / 3) * 58 + tap % 3) * 64) >> 4) + 2 * h, db + 2 * h, idesc, 1u);
      }
    } else {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
          ptx::mma_tf32(tmem + (u % NACC) * N, da + 2 * (u & 1), db + 2 * (u & 1), idesc, 1u);
      }
    }
    long long t1 = clock64();
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 256);
  }
}

template <int N, int U, int NACC = 1, int M = 128>
void run(int grid, int shift = 0, int boff = 8192) {
  long long* out;
  cudaMalloc(&out, 16);
  cudaFuncSetAttribute(k_rate<N, U, NACC, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  const int iters = 256 / U;
  k_rate<N, U, NACC, M><<<grid, 128, 80 * 1024>>>(iters, out, shift, boff);
  k_rate<N, U, NACC, M><<<grid, 128, 80 * 1024>>>(iters, out, shift, boff);
  long long h[2];
  cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("acc %d shift %d boff %d ", NACC, shift, boff);
  printf("M=%d ", M);
  printf("grid %3d N=%3d unroll %d: issue %6.1f cyc/mma, complete %6.1f cyc/mma (ideal %d at 4096 flop/cyc)\n",
         grid, N, U, double(h[0]) / 256, double(h[1]) / 256, 128 * N * 8 * 2 / 4096);
  cudaFree(out);
}

int main() {
  for (int grid : {1, 148}) {  // M = 64 (output channels on M, pixels on N): rate per SM
    run<64, 8, 1, 64>(grid);
    run<128, 8, 1, 64>(grid);
    run<256, 8, 1, 64>(grid);
  }
  for (int bo : {8192, 16384, 24576, 32768, 40960}) {
    run<64, 8>(1, 0, bo);
    run<64, 8>(1, 1, bo);
    run<64, 8>(1, -1, bo);
  }
  for (int sh : {0, 1, 2, 58, 59}) run<256, 8>(1, sh);
  for (int grid : {1, 148}) {
    run<64, 1>(grid);
    run<64, 8>(grid);
    run<128, 8>(grid);
    run<256, 8>(grid);
    run<64, 8, 2>(grid);
    run<64, 8, 4>(grid);
    run<32, 8, 1>(grid);
    run<32, 8, 4>(grid);
    run<128, 8, 2>(grid);
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
