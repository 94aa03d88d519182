// Probe: tcgen05.mma kind::tf32 with MN-major operands in the SWIZZLE_128B_BASE32B layout
// (descriptor layout type 1; CUTLASS sm100_common.inl: "for mn-major tf32 operands, SW128_32B
// is the only available smem layout"). An MN-major tf32 operand is rows of 32 MN elements
// (128 B) per reduction index, 4 rows per swizzle atom (bytes [5,7) ^= bytes [7,9)), reduction
// groups of 4 rows at SBO, 32-element MN groups at LBO.
//
// Host builds an smem image + descriptors; the kernel copies it to smem, issues the MMAs, and
// reads D (128 x N). Checks against a double reference; then times R back-to-back MMAs.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>
#include "../paper_2002_02145_b200/csrc/sm100_ptx.cuh"
using namespace psconv;

constexpr int kImg = 96 * 1024;

__global__ void k_mma(const uint4* img, int img_words, uint64_t da, uint64_t db, int nk, uint32_t astep,
                      uint32_t bstep, uint32_t idesc, int N, float* D, int reps, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(sm + kImg);
  uint32_t* slot = (uint32_t*)(bar + 2);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < img_words; i += blockDim.x) ((uint4*)sm)[i] = img[i];
  if (threadIdx.x == 0) { ptx::mbar_init(&bar[0], 1); ptx::mbar_init(&bar[1], 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(slot, 256);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t base = ptx::smem_u32(sm) >> 4;
  if (threadIdx.x == 0) {
    ptx::tc_fence_after();
    for (int k = 0; k < nk; ++k)
      ptx::mma_tf32(tmem, da + base + k * astep, db + base + k * bstep, idesc, k > 0);
    ptx::mma_commit(&bar[0]);
  }
  ptx::mbar_wait(&bar[0], 0);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp < 4) {
    uint32_t v[16];
    for (int c = 0; c < N; c += 16) {
      ptx::tmem_ld16(tmem + ((warp * 32) << 16) + c, v);
      ptx::tmem_wait_ld();
      for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * 256 + c + j] = __uint_as_float(v[j]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (reps > 0 && threadIdx.x == 0) {  // rate: reps x nk MMAs into the same accumulator
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int k = 0; k < nk; ++k) ptx::mma_tf32(tmem, da + base + k * astep, db + base + k * bstep, idesc, 1);
    ptx::mma_commit(&bar[1]);
    ptx::mbar_wait(&bar[1], 0);
    *cyc = clock64() - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 256); }
}

static uint64_t desc(uint32_t off, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)(off >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46) |
         ((uint64_t)layout << 61);
}
static uint32_t swz64(uint32_t off) { return off ^ (((off >> 7) & 3) << 4); }
static uint32_t swz128_32(uint32_t off) { return off ^ (((off >> 7) & 3) << 5); }

struct Exp {
  const char* name;
  std::vector<uint8_t> img;
  uint64_t da, db;
  int nk;
  uint32_t astep, bstep, idesc;
  int N;
};

int main() {
  const int M = 128, K = 16;
  static float A[128][16], B[16][256];
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < K; ++k) A[m][k] = (float)(((m * 7 + k * 3) % 11) - 5) / 4.0f;
  for (int k = 0; k < K; ++k)
    for (int n = 0; n < 256; ++n) B[k][n] = (float)(((k * 5 + n * 3) % 9) - 4) / 2.0f;
  auto idesc = [](int N, int amaj, int bmaj) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) |
           ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  };
  // A K-major SW64 at offset 0 (8 KB): row m = 64 B of k
  auto put_a_k = [&](Exp& e) {
    for (int m = 0; m < M; ++m)
      for (int k = 0; k < K; ++k) memcpy(&e.img[swz64(m * 64 + k * 4)], &A[m][k], 4);
    e.da = desc(0, 16, 512, 4);
    e.astep = 2;  // +32 B per K=8
  };
  // A MN-major SW128_32B at offset 0: 4 MN groups (32 m) of K rows (128 B) at LBO = K*128
  auto put_a_mn = [&](Exp& e) {
    for (int m = 0; m < M; ++m)
      for (int k = 0; k < K; ++k) {
        const uint32_t off = (m / 32) * (K * 128) + k * 128 + (m % 32) * 4;
        memcpy(&e.img[swz128_32(off)], &A[m][k], 4);
      }
    e.da = desc(0, K * 128, 512, 1);
    e.astep = 1024 / 16;  // +8 rows per K=8
  };
  // B MN-major SW128_32B at offset 16 KB: N/32 groups of K rows at LBO = lbo
  auto put_b_mn = [&](Exp& e, int N, uint32_t lbo) {
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) {
        const uint32_t off = (n / 32) * lbo + k * 128 + (n % 32) * 4;
        memcpy(&e.img[16384 + swz128_32(off)], &B[k][n], 4);
      }
    e.db = desc(16384, lbo, 512, 1);
    e.bstep = 1024 / 16;
  };
  // B K-major SW64 at offset 16 KB (rate baseline): row n = 64 B of k
  auto put_b_k = [&](Exp& e, int N) {
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) memcpy(&e.img[16384 + swz64(n * 64 + k * 4)], &B[k][n], 4);
    e.db = desc(16384, 16, 512, 4);
    e.bstep = 2;
  };
  std::vector<Exp> exps;
  for (int N : {32, 64, 128, 256}) {
    Exp e{};
    e.img.assign(kImg, 0);
    e.name = "A:K-SW64  B:MN-SW128_32B";
    e.N = N;
    e.nk = 2;
    put_a_k(e);
    put_b_mn(e, N, K * 128);
    e.idesc = idesc(N, 0, 1);
    exps.push_back(e);
  }
  for (int N : {64, 256}) {
    Exp e{};
    e.img.assign(kImg, 0);
    e.name = "A:MN-SW128_32B B:MN-SW128_32B";
    e.N = N;
    e.nk = 2;
    put_a_mn(e);
    put_b_mn(e, N, K * 128);
    e.idesc = idesc(N, 1, 1);
    exps.push_back(e);
  }
  for (int N : {64, 256}) {
    Exp e{};
    e.img.assign(kImg, 0);
    e.name = "A:K-SW64  B:K-SW64 (baseline)";
    e.N = N;
    e.nk = 2;
    put_a_k(e);
    put_b_k(e, N);
    e.idesc = idesc(N, 0, 0);
    exps.push_back(e);
  }
  {  // B MN-major with non-contiguous MN groups (LBO = 4 KB): the wgrad tap/tile pitch case
    Exp e{};
    e.img.assign(kImg, 0);
    e.name = "A:MN B:MN LBO=4096";
    e.N = 128;
    e.nk = 2;
    put_a_mn(e);
    put_b_mn(e, 128, 4096);
    e.idesc = idesc(128, 1, 1);
    exps.push_back(e);
  }
  uint4* dimg;
  float* dD;
  long long* dc;
  cudaMalloc(&dimg, kImg);
  cudaMalloc(&dD, 128 * 256 * 4);
  cudaMalloc(&dc, 8);
  cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, kImg + 2048);
  static float hD[128 * 256];
  for (auto& e : exps) {
    cudaMemcpy(dimg, e.img.data(), kImg, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, sizeof hD);
    const int reps = 64;
    k_mma<<<1, 128, kImg + 2048>>>(dimg, kImg / 16, e.da, e.db, e.nk, e.astep, e.bstep, e.idesc, e.N, dD, reps, dc);
    cudaError_t err = cudaDeviceSynchronize();
    long long cyc = 0;
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    double mx = 0, mr = 0;
    int nz = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < e.N; ++n) {
        double r = 0;
        for (int k = 0; k < K; ++k) r += (double)A[m][k] * B[k][n];
        mx = fmax(mx, fabs(hD[m * 256 + n] - r));
        mr = fmax(mr, fabs(r));
        nz += hD[m * 256 + n] != 0;
      }
    printf("%-34s N=%3d err=%s maxerr=%.4g maxref=%.4g nonzero=%d/%d  %.1f cyc per K=8 MMA\n", e.name, e.N,
           cudaGetErrorString(err), mx, mr, nz, M * e.N, double(cyc) / (reps * e.nk));
    if (err != cudaSuccess) return 1;
  }
  return 0;
}
