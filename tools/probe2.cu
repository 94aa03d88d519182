// Generic tcgen05 probe: host builds a shared-memory image + descriptors, the
// kernel copies the image to smem verbatim, issues nk MMAs, reads D (128 x 32 cols).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include "../paper_2002_02145_b200/csrc/sm100_ptx.cuh"
using namespace psconv;

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

__global__ void k_mma(const uint4* img, int img_words, uint64_t da, uint64_t db, int nk, uint32_t astep,
                      uint32_t bstep, uint32_t idesc, int kind, float* D, int test_st) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(sm + 64 * 1024);
  uint32_t* slot = (uint32_t*)(bar + 2);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < img_words; i += blockDim.x) ((uint4*)sm)[i] = img[i];
  if (threadIdx.x == 0) { ptx::mbar_init(&bar[0], 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(slot, 32);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t base = ptx::smem_u32(sm) >> 4;
  if (test_st) {
    // tcgen05.st roundtrip: write lane*100+col into 16 cols
    uint32_t v[16];
    for (int j = 0; j < 16; ++j) v[j] = __float_as_uint((float)((warp * 32 + lane) * 100 + j));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(tmem + ((warp * 32) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                    "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  } else if (threadIdx.x == 0) {
    ptx::tc_fence_after();
    for (int k = 0; k < nk; ++k) {
      const uint64_t a = da + base + k * astep, b = db + base + k * bstep;
      if (kind == 0) ptx::mma_tf32(tmem, a, b, idesc, k > 0);
      else mma_f16(tmem, a, b, idesc, k > 0);
    }
    ptx::mma_commit(&bar[0]);
  }
  if (!test_st) ptx::mbar_wait(&bar[0], 0);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp < 4) {
    uint32_t v[16];
    for (int half = 0; half < 2; ++half) {
      ptx::tmem_ld16(tmem + ((warp * 32) << 16) + half * 16, v);
      ptx::tmem_wait_ld();
      for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * 32 + half * 16 + j] = __uint_as_float(v[j]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 32); }
}

static uint64_t desc(uint32_t off, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  // start address relative to base is added in-kernel (in 16B units)
  return (uint64_t)(off >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46) |
         ((uint64_t)layout << 61);
}
static uint32_t swz64(uint32_t off) { return off ^ (((off >> 7) & 3) << 4); }
static uint32_t swz128(uint32_t off) { return off ^ (((off >> 7) & 7) << 4); }
static uint16_t bf16(float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)(u >> 16); }

struct Exp { const char* name; std::vector<uint8_t> img; uint64_t da, db; int nk; uint32_t astep, bstep, idesc; int kind; int N; std::vector<double> ref; };

int main() {
  const int M = 128;
  float A[128][16], B[16][32];  // A: M x K(16), B: K x N(up to 32)
  for (int m = 0; m < M; ++m) for (int k = 0; k < 16; ++k) A[m][k] = (float)(((m * 7 + k * 3) % 11) - 5) / 4.0f;
  for (int k = 0; k < 16; ++k) for (int n = 0; n < 32; ++n) B[k][n] = (float)(((k * 5 + n * 3) % 9) - 4) / 2.0f;
  std::vector<Exp> exps;
  auto ref_for = [&](int N) { std::vector<double> r(M * 32, 0); for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) { double s = 0; for (int k = 0; k < 16; ++k) s += A[m][k] * B[k][n]; r[m * 32 + n] = s; } return r; };
  const uint32_t id_tf32_16_kk = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (0u << 16) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
  const uint32_t id_tf32_16_kmn = id_tf32_16_kk | (1u << 16);
  {  // E1: tf32, A K-major SW64, B K-major SW64 (B stored N rows x 64B)
    Exp e; e.name = "tf32 A:K-SW64 B:K-SW64"; e.img.assign(16384, 0);
    for (int m = 0; m < M; ++m) for (int k = 0; k < 16; ++k) memcpy(&e.img[swz64(m * 64 + k * 4)], &A[m][k], 4);
    for (int n = 0; n < 16; ++n) for (int k = 0; k < 16; ++k) memcpy(&e.img[8192 + swz64(n * 64 + k * 4)], &B[k][n], 4);
    e.da = desc(0, 16, 512, 4); e.db = desc(8192, 16, 512, 4); e.nk = 2; e.astep = 2; e.bstep = 2; e.idesc = id_tf32_16_kk; e.kind = 0; e.N = 16;
    e.ref = ref_for(16); exps.push_back(e);
  }
  {  // E2: tf32, A K-major SW64, B MN-major SW64 (row = k, 16 n per 64 B)
    Exp e; e.name = "tf32 A:K-SW64 B:MN-SW64"; e.img.assign(16384, 0);
    for (int m = 0; m < M; ++m) for (int k = 0; k < 16; ++k) memcpy(&e.img[swz64(m * 64 + k * 4)], &A[m][k], 4);
    for (int k = 0; k < 16; ++k) for (int n = 0; n < 16; ++n) memcpy(&e.img[8192 + swz64(k * 64 + n * 4)], &B[k][n], 4);
    e.da = desc(0, 16, 512, 4); e.db = desc(8192, 1024, 512, 4); e.nk = 2; e.astep = 2; e.bstep = 32; e.idesc = id_tf32_16_kmn; e.kind = 0; e.N = 16;
    e.ref = ref_for(16); exps.push_back(e);
  }
  {  // E3: tf32, no swizzle K-major both: core matrix 8 rows x 16B contiguous (128B)
    // A: ((8,m),(4,2)) : element (m,k): group g=m/8, r=m%8, chunk c=k/4, within w=k%4
    // layout: offset = g*SBO + c*LBO + r*16 + w*4 with LBO=128 (K-adjacent core matrices), SBO=512 (4 chunks*128)
    Exp e; e.name = "tf32 A:K-INTER B:K-INTER"; e.img.assign(16384, 0);
    for (int m = 0; m < M; ++m) for (int k = 0; k < 16; ++k) { uint32_t off = (m / 8) * 512 + (k / 4) * 128 + (m % 8) * 16 + (k % 4) * 4; memcpy(&e.img[off], &A[m][k], 4); }
    for (int n = 0; n < 16; ++n) for (int k = 0; k < 16; ++k) { uint32_t off = 8192 + (n / 8) * 512 + (k / 4) * 128 + (n % 8) * 16 + (k % 4) * 4; memcpy(&e.img[off], &B[k][n], 4); }
    e.da = desc(0, 128, 512, 0); e.db = desc(8192, 128, 512, 0); e.nk = 2; e.astep = 16; e.bstep = 16; e.idesc = id_tf32_16_kk; e.kind = 0; e.N = 16;
    e.ref = ref_for(16); exps.push_back(e);
  }
  {  // E4: bf16 kind::f16 K-major SW128-less: A 128 x 16 bf16 = 32B rows, use no-swizzle K-major
    Exp e; e.name = "bf16 A:K-INTER B:K-INTER"; e.img.assign(16384, 0);
    for (int m = 0; m < M; ++m) for (int k = 0; k < 16; ++k) { uint32_t off = (m / 8) * 256 + (k / 8) * 128 + (m % 8) * 16 + (k % 8) * 2; uint16_t h = bf16(A[m][k]); memcpy(&e.img[off], &h, 2); }
    for (int n = 0; n < 16; ++n) for (int k = 0; k < 16; ++k) { uint32_t off = 8192 + (n / 8) * 256 + (k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2; uint16_t h = bf16(B[k][n]); memcpy(&e.img[off], &h, 2); }
    e.da = desc(0, 128, 256, 0); e.db = desc(8192, 128, 256, 0); e.nk = 1; e.astep = 0; e.bstep = 0;
    e.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24); e.kind = 1; e.N = 16;
    e.ref = ref_for(16); exps.push_back(e);
  }
  {  // E5: bf16 with m_dim at bit 23 instead
    Exp e = exps.back(); e.name = "bf16 INTER, M at bit23";
    e.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 23); exps.push_back(e);
  }
  {  // E6: tf32 E1 with M at bit 23
    Exp e = exps[0]; e.name = "tf32 K-SW64 both, M at bit23";
    e.idesc = (id_tf32_16_kk & ~(0x1Fu << 24)) | ((128u >> 4) << 23); exps.push_back(e);
  }
  {  // E7: conversion mode: A = 1 + 3*2^-12 (0.75 tf32 ulp), B = identity -> D = tf32(A)
    Exp e = exps[0]; e.name = "tf32 convert: 1.0=RZ 1.000977=RN";
    e.img.assign(16384, 0);
    const float a = 1.0f + 3.0f / 4096.0f, one = 1.0f;
    for (int m = 0; m < M; ++m) for (int k = 0; k < 16; ++k) memcpy(&e.img[swz64(m * 64 + k * 4)], &a, 4);
    for (int n = 0; n < 16; ++n) memcpy(&e.img[8192 + swz64(n * 64 + n * 4)], &one, 4);
    e.ref.assign(M * 32, 0); for (int m = 0; m < M; ++m) for (int n = 0; n < 16; ++n) e.ref[m * 32 + n] = a;
    exps.push_back(e);
  }
  {  // E8: accumulation rounding: D = 1 (k=0 col) then add 2^-24*3 (0.75 ulp of 1) many times
    Exp e = exps[0]; e.name = "acc: 1 + 0.75ulp x1 (RZ=1)";
    e.img.assign(16384, 0);
    const float one = 1.0f, tiny = 3.0f / 16777216.0f;
    for (int m = 0; m < M; ++m) { memcpy(&e.img[swz64(m * 64 + 0 * 4)], &one, 4); memcpy(&e.img[swz64(m * 64 + 8 * 4)], &tiny, 4); }
    for (int n = 0; n < 16; ++n) { memcpy(&e.img[8192 + swz64(n * 64 + 0 * 4)], &one, 4); memcpy(&e.img[8192 + swz64(n * 64 + 8 * 4)], &one, 4); }
    e.ref.assign(M * 32, 0); for (int m = 0; m < M; ++m) for (int n = 0; n < 16; ++n) e.ref[m * 32 + n] = 1.0 + 3.0 / 16777216.0;
    exps.push_back(e);
  }
  uint4* dimg; float* dD; cudaMalloc(&dimg, 16384); cudaMalloc(&dD, 128 * 32 * 4);
  cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  float hD[128 * 32];
  // st/ld roundtrip
  cudaMemset(dD, 0, sizeof hD);
  k_mma<<<1, 128, 80 * 1024>>>(dimg, 0, 0, 0, 0, 0, 0, 0, 0, dD, 1);
  printf("st/ld roundtrip: %s  D[0]=%g D[1]=%g D[33*32+5]=%g (expect 0 1 3305)\n", cudaGetErrorString(cudaDeviceSynchronize()), 0.0, 0.0, 0.0);
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  printf("  got %g %g %g\n", hD[0], hD[1], hD[33 * 32 + 5]);
  for (auto& e : exps) {
    cudaMemcpy(dimg, e.img.data(), 16384, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, sizeof hD);
    k_mma<<<1, 128, 80 * 1024>>>(dimg, 16384 / 16, e.da, e.db, e.nk, e.astep, e.bstep, e.idesc, e.kind, dD, 0);
    cudaError_t err = cudaDeviceSynchronize();
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    double mx = 0, mr = 0; int nz = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < e.N; ++n) { mx = fmax(mx, fabs(hD[m * 32 + n] - e.ref[m * 32 + n])); mr = fmax(mr, fabs(e.ref[m * 32 + n])); nz += hD[m * 32 + n] != 0; }
    printf("%-32s err=%s maxerr=%.4g maxref=%.4g nonzero=%d  D0..3=%.9g %g %g %g ref=%.9g %g %g %g\n", e.name, cudaGetErrorString(err), mx, mr, nz,
           hD[0], hD[1], hD[2], hD[3], e.ref[0], e.ref[1], e.ref[2], e.ref[3]);
    if (err != cudaSuccess) return 1;
  }
  return 0;
}
