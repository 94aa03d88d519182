// Probe: the 3xTF32 k-step MMA pattern of conv_fwd_sm100 at BN = 64 (N-concat), one CTA
// per SM, issue from one thread, 144 k-steps:
//   ts   : A_hi / A_lo from TMEM slots: per K-half A_hi x [B_hi;B_lo] (N = 128) + A_lo x B_hi
//          (N = 64), a commit per k-step (the kernel's TMEM-A path)
//   ts+st: the same with 4 splitter warps writing the next slots with tcgen05.st meanwhile
//   ss   : A_hi / A_lo from shared memory (SW64), same MMAs
//   ss3  : three separate N = 64 MMAs per K-half (no N-concat), A from smem
// Reports cycles per k-step (ideal at 2048 tf32 FMA/cycle/SM: 2 x (64 + 32) = 192).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2002_02145_b200/csrc \
//        tools/probe_kstep.cu -o tools/probe_kstep
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100_ptx.cuh"
using namespace psconv;

constexpr int KSTEPS = 144;
constexpr int SLOTS = 6, SLOT_COL = 320;

template <int MODE>  // 0 ts, 1 ts+st, 2 ss, 3 ss3, 4 mixed+st (A_hi smem, A_lo TMEM, 16 cols written),
                     // 5 ts+st with two splitter groups on alternate k-steps, 6 ts+st batched (2 k-steps per wait)
__global__ void k_step(long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t slot_free[SLOTS], slot_full[SLOTS], done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (48 * 1024) / 4; i += blockDim.x) ((float*)sm)[i] = 1e-3f * (i & 7);
  if (threadIdx.x == 0) {
    for (int s = 0; s < SLOTS; ++s) {
      ptx::mbar_init(&slot_free[s], 1);
      ptx::mbar_init(&slot_full[s], 128);
    }
    ptx::mbar_init(&done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(&tslot, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  // smem: A (8 KB) | A_lo (8 KB) | B [B_hi;B_lo] 128 rows (8 KB) at 16 KB
  const uint64_t da = ptx::smem_desc_sw64(ptx::smem_u32(sm), 16, 512);
  const uint64_t dalo = ptx::smem_desc_sw64(ptx::smem_u32(sm + 8192), 16, 512);
  const uint64_t db = ptx::smem_desc_sw64(ptx::smem_u32(sm + 16384), 16, 512);
  const uint64_t dblo = ptx::smem_desc_sw64(ptx::smem_u32(sm + 16384 + 4096), 16, 512);
  constexpr uint32_t i64 = ptx::idesc_tf32_m128<64>(), i128 = ptx::idesc_tf32_m128<128>();
  if (warp == 0) {
    long long t0 = clock64();
    for (int k = 0; k < KSTEPS; ++k) {
      const int s = k % SLOTS;
      if (MODE == 1 || MODE >= 4) {
        ptx::mbar_wait(&slot_full[s], (k / SLOTS) & 1);
        ptx::tc_fence_after();
      }
      if (ptx::elect_one()) {
        const uint32_t ah = tmem + SLOT_COL + s * 32;
        for (int h = 0; h < 2; ++h) {
          if (MODE <= 1 || MODE >= 5) {
            ptx::mma_tf32_ts(tmem, ah + h * 8, db + h * 2, i128, k | h);
            ptx::mma_tf32_ts(tmem, ah + 16 + h * 8, db + h * 2, i64, 1u);
          } else if (MODE == 4) {
            ptx::mma_tf32(tmem, da + h * 2, db + h * 2, i128, k | h);
            ptx::mma_tf32_ts(tmem, ah + h * 8, db + h * 2, i64, 1u);
          } else if (MODE == 2) {
            ptx::mma_tf32(tmem, da + h * 2, db + h * 2, i128, k | h);
            ptx::mma_tf32(tmem, dalo + h * 2, db + h * 2, i64, 1u);
          } else {
            ptx::mma_tf32(tmem, dalo + h * 2, db + h * 2, i64, k | h);
            ptx::mma_tf32(tmem, da + h * 2, dblo + h * 2, i64, 1u);
            ptx::mma_tf32(tmem, da + h * 2, db + h * 2, i64, 1u);
          }
        }
        ptx::mma_commit(&slot_free[s]);  // per k-step (the kernel frees the TMEM A slot)
      }
      __syncwarp();
    }
    long long t1 = clock64();
    if (ptx::elect_one()) ptx::mma_commit(&done);
    __syncwarp();
    ptx::mbar_wait(&done, 0);
    long long t2 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  } else if ((MODE == 1 || MODE == 4 || MODE == 6) && warp >= 4 && warp < 8) {
    const int quad = warp & 3, lane = threadIdx.x & 31;
    const uint32_t lb = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(1e-3f * (lane + i));
    const int batch = MODE == 6 ? 2 : 1;
    for (int k0 = 0; k0 < KSTEPS; k0 += batch) {
      for (int k = k0; k < k0 + batch; ++k) {
        const int s = k % SLOTS;
        if (k >= SLOTS) ptx::mbar_wait(&slot_free[s], ((k / SLOTS) - 1) & 1);
        ptx::tc_fence_after();
        ptx::tmem_st16(lb + SLOT_COL + s * 32, v);
        if (MODE != 4) ptx::tmem_st16(lb + SLOT_COL + s * 32 + 16, v);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      for (int k = k0; k < k0 + batch; ++k) ptx::mbar_arrive(&slot_full[k % SLOTS]);
    }
  } else if (MODE == 5 && warp >= 4 && warp < 12) {
    const int quad = warp & 3, lane = threadIdx.x & 31, grp = (warp - 4) / 4;
    const uint32_t lb = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(1e-3f * (lane + i));
    for (int k = grp; k < KSTEPS; k += 2) {
      const int s = k % SLOTS;
      if (k >= SLOTS) ptx::mbar_wait(&slot_free[s], ((k / SLOTS) - 1) & 1);
      ptx::tc_fence_after();
      ptx::tmem_st16(lb + SLOT_COL + s * 32, v);
      ptx::tmem_st16(lb + SLOT_COL + s * 32 + 16, v);
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&slot_full[s]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

template <int MODE>
void run(const char* name, int grid) {
  long long* out;
  cudaMalloc(&out, 16);
  cudaFuncSetAttribute(k_step<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int r = 0; r < 2; ++r) k_step<MODE><<<grid, 384, 64 * 1024>>>(out);
  long long h[2];
  cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("%-6s grid %3d: issue %7.1f cyc/k-step, complete %7.1f cyc/k-step (ideal 192)\n", name, grid,
         double(h[0]) / KSTEPS, double(h[1]) / KSTEPS);
  cudaFree(out);
}

int main() {
  for (int g : {1, 148}) {
    run<0>("ts", g);
    run<1>("ts+st", g);
    run<2>("ss", g);
    run<3>("ss3", g);
    run<4>("mix+st", g);
    run<5>("ts+st2g", g);
    run<6>("ts+stb2", g);
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
