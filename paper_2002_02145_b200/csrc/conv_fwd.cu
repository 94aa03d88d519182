// GPU layer entry: plans, tensor maps, launches, and the device-side helpers
// (seeded generator, layout packing, 3xTF32 weight split).
//
// Replaces the reference's driver loop nest (emit_source, include/nestrank/
// emit.hpp:60-134) + the external LIBXSMM microkernel with
// one persistent sm_100a kernel per conv_fwd call.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "conv_kernel.cuh"
#include "conv_pp.cuh"
#include "internal.hpp"
#include "seeded.hpp"
#include "wgrad_kernel.cuh"

static_assert(psconv::kSmemStageBudget == psconv::kStageBudget, "stage budget");
static_assert(psconv::kSmemMaxStages == psconv::kMaxStages, "max stages");

struct conv_plan {
  conv_desc d;
  int mode;
  int device;
  int num_sms;
  psconv::Schedule sched;
  float* flt_pack = nullptr;   // prepacked K-major filter: hi (| lo for 3xTF32), see prepack
  bool b128 = false;           // filter rows of 32 channels (128 B, SWIZZLE_128B) vs 16 (64 B)
  bool ncat = false;           // 3xTF32 N-concat: prepacked rows [B_hi;B_lo] per N tile (ConvParams::ncat)
  unsigned* absmax = nullptr;  // f16x2: |max| bits of [0] the filter, [1] the call's input range
  // (c,s)-folded input (recipe fold:C, SURVEY §8d stem note): the layer has C <= 8
  // real input channels in one 16-channel block; G = 16 / C consecutive kw taps
  // are packed into one block, so the kernel runs the descriptor kd (kw' =
  // ceil(kw / G), no w padding, tap dilation G) over the folded copy xfold.
  int fold = 0, fold_g = 1, fold_phases = 1;
  // few-channel kernel (recipe pp:C, conv_pp.cuh): C <= 4 real channels, tap
  // pairs over input parity planes; the filter is packed per tap-pair MMA
  int pp = 0;
  psconv::PpGeom ppg{};
  conv_desc kd{};                 // kernel descriptor (== d unless folded)
  float* xfold = nullptr;         // [nImg][phases][H][Wq][16]
  float* wfold = nullptr;         // folded filter, KCRS16c16k of kd
  // backward-data plan (conv_plan_create_bwd_data): d is the TRANSPOSED stride-1
  // convolution dX = conv(dY, W^T flipped); the forward filter is transformed
  // into wtrans before the repack
  bool bwd_data = false;
  conv_desc fwd{};                // the forward layer's descriptor
  float* wtrans = nullptr;
  // strided backward data (stride s > 1): dX splits into sh x sw output phases (a, b) =
  // (h mod sh, w mod sw). Phase (a, b) is a stride-1 transposed conv over dY whose taps are
  // the forward taps r = sh*u + rho_h, s = sw*v + rho_w (flipped), with asymmetric implied
  // padding; a child plan runs it and stores through a strided view of dX (out_sh/out_sw
  // over the parent extent out_H x out_W). Phases without taps are zero-filled.
  std::vector<conv_plan*> phase_plans;  // parent: one child per phase with taps
  std::vector<std::pair<int, int>> zero_phases;
  int ph_a = 0, ph_b = 0, ph_rho_h = 0, ph_rho_w = 0;  // child: its phase and first taps
  int out_sh = 1, out_sw = 1;
  int64_t out_H = 0, out_W = 0;
  // backward-weight plan (conv_plan_create_bwd_weight): d is the forward layer; the
  // pixel-major wgrad kernel's geometry and its split partial workspace (wgrad_kernel.cuh)
  bool bwd_weight = false;
  psconv::WgradParams wg{};
  float* wg_ws = nullptr;
  float* wg_x32 = nullptr;  // TMA path: X / dY relaid into 32-channel blocks (+ 3xTF32 lo halves)
  float* wg_y32 = nullptr;
  mutable bool prepacked = false;  // flt_pack holds the filter given to conv_plan_prepack
  int64_t flt_elems = 0;
  // conv_fwd_host staging (lazily created): double-buffered device chunks,
  // copy-in / copy-out streams and their events
  struct HostPipe {
    int64_t chunk = 0;                 // images per chunk
    static constexpr int kSlots = 3;   // device chunk buffers in flight
    float* din[kSlots] = {};
    float* dout[kSlots] = {};
    float* dflt = nullptr;
    cudaStream_t sin = nullptr, sout = nullptr;
    cudaEvent_t start = nullptr, flt = nullptr, end = nullptr;
    cudaEvent_t h2d[kSlots] = {}, conv[kSlots] = {}, d2h[kSlots] = {};
  };
  mutable HostPipe* pipe = nullptr;
  // split-K scratch (ConvParams::split_ctr / split_ws), sized at plan creation for the
  // largest launch of the plan (img_count = nImg): ticket/done counters per split tile
  // slot (zero between launches) and one 128 x bn partial per (slot, split)
  int* split_ctr = nullptr;
  float* split_ws = nullptr;
  int64_t split_slots = 0;  // split tiles x CTAs per cluster the scratch holds
  int split_k = 1;          // units per split tile the scratch holds
  int64_t user_flt_elems = 0;  // the caller's filter (KCRS16c16k of d): nOfm*nIfm*kh*kw
};

namespace psconv {
namespace {

#define CUDA_OK(expr)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      throw RuntimeError(std::string(#expr) + ": " + cudaGetErrorString(_e));           \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) throw RuntimeError("cuTensorMapEncodeTiled unavailable (driver too old?)");
  return fn;
}

// promo: L2 sector promotion of the TMA's fills. 256 B (default) suits dense boxes; boxes
// that skip 64-B pixels (element strides > 1, the stride-2 layers' A) use 64 B so the skipped
// pixels are not fetched from DRAM with the used ones.
void encode(CUtensorMap* m, const float* base, int rank, const cuuint64_t* dims,
            const cuuint64_t* strides_bytes, const cuuint32_t* box, const cuuint32_t* estr,
            CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_64B,
            CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
  static const int promo_env = [] {  // A/B switch (profiling): 0 none, 64, 128, 256
    const char* e = std::getenv("PSCONV_A_PROMO");
    return e ? std::atoi(e) : -1;
  }();
  if (promo != CU_TENSOR_MAP_L2_PROMOTION_L2_256B && promo_env >= 0)
    promo = promo_env == 0     ? CU_TENSOR_MAP_L2_PROMOTION_NONE
            : promo_env == 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
            : promo_env == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                               : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float*>(base),
                                 dims, strides_bytes, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 swz, promo,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw RuntimeError("cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

// ---------------------------------------------------------------- helpers
// Filter prepack: KCRS16c16k [Kb][C*R*S/16 blocks][16c][16k] -> K-major rows
// (one row of input channels per output channel), the B-operand layout
// tcgen05 kind::tf32 accepts (K-major; MN-major reads as zeros, probe2.cu):
//   b128 = 0: [Cb][R*S][K][16c]      64-B rows, SWIZZLE_64B
//   b128 = 1: [Cb/2][R*S][K][32c]   128-B rows holding channel blocks 2i, 2i+1
//             (SWIZZLE_128B): half the TMA row requests per k-step, which is
//             what bounds operand delivery (tools/probe_tma_issue.cu).
// 3xTF32: also split x -> hi = x with the 13 low mantissa bits cleared
// (exactly representable in tf32) and lo = x - hi (exact in fp32).
// One 256-thread block per 16x16 [c][k] block, transposed through smem.
// ncat_bn > 0 (3xTF32 N-concat): hi and lo rows interleaved per N tile of ncat_bn
// output channels in one [.. ][2K][..] layout: rows tile*2bn + k%bn (hi), + bn (lo).
__global__ void prepack_filter_kernel(const float* __restrict__ flt, float* __restrict__ hi,
                                      float* __restrict__ lo, int K, int CRS, int RS, int split,
                                      int b128, int ncat_bn) {
  __shared__ float tile[16][17];
  ptx::griddep_launch_dependents();  // the conv kernel may start its prologue now
  const int blk = blockIdx.x;  // = kb * CRS + crs, crs = cb * RS + rs
  const int kb = blk / CRS, crs = blk % CRS;
  const int t = threadIdx.x;
  tile[t >> 4][t & 15] = flt[static_cast<int64_t>(blk) * 256 + t];  // [c][k]
  __syncthreads();
  const int k16 = t >> 4, c16 = t & 15;
  const float x = tile[c16][k16];
  const int cb = crs / RS, rs = crs % RS;
  const int64_t k = kb * 16 + k16;
  if (ncat_bn > 0) {
    const int64_t K2 = 2 * static_cast<int64_t>(K);
    const int64_t kh = (k / ncat_bn) * 2 * ncat_bn + k % ncat_bn;
    const int64_t row0 = b128 ? (static_cast<int64_t>(cb >> 1) * RS + rs) * K2 : (static_cast<int64_t>(cb) * RS + rs) * K2;
    const int64_t w = b128 ? 32 : 16, c = b128 ? (cb & 1) * 16 + c16 : c16;
    const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    hi[(row0 + kh) * w + c] = h;
    hi[(row0 + kh + ncat_bn) * w + c] = x - h;
    return;
  }
  const int64_t o = b128 ? ((static_cast<int64_t>(cb >> 1) * RS + rs) * K + k) * 32 + (cb & 1) * 16 + c16
                         : ((static_cast<int64_t>(cb) * RS + rs) * K + k) * 16 + c16;
  if (split) {
    const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    hi[o] = h;
    lo[o] = x - h;
  } else {
    hi[o] = x;
  }
}

// |max| over n floats (n % 4 == 0) into *out (as ordered uint bits; *out zeroed first)
__global__ void absmax_kernel(const float* __restrict__ x, int64_t n, unsigned* out) {
  ptx::griddep_wait();  // PDL launch: the input may come from the preceding kernel
  ptx::griddep_launch_dependents();
  unsigned m = 0;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n / 4; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 v = x4[i];
    m = max(m, max(max(__float_as_uint(fabsf(v.x)), __float_as_uint(fabsf(v.y))),
                   max(__float_as_uint(fabsf(v.z)), __float_as_uint(fabsf(v.w)))));
  }
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// f16x2 filter prepack: the fp32 prepack's rows, each 16-channel group holding
// fp16 hi (32 B) then lo (32 B) of x * sB, sB = pow2_scale(|max|)
__global__ void prepack_filter_f16_kernel(const float* __restrict__ flt, uint16_t* __restrict__ out, int K,
                                          int CRS, int RS, int b128, const unsigned* __restrict__ absmax) {
  __shared__ float tile[16][17];
  const int blk = blockIdx.x;
  const int t = threadIdx.x;
  tile[t >> 4][t & 15] = flt[static_cast<int64_t>(blk) * 256 + t];
  __syncthreads();
  const int k16 = t >> 4, c16 = t & 15;
  const float x = tile[c16][k16] * pow2_scale(*absmax);
  const int kb = blk / CRS, crs = blk % CRS;
  const int cb = crs / RS, rs = crs % RS;
  const int64_t k = kb * 16 + k16;
  const int64_t o = b128 ? ((static_cast<int64_t>(cb >> 1) * RS + rs) * K + k) * 32 + (cb & 1) * 16 + c16
                         : ((static_cast<int64_t>(cb) * RS + rs) * K + k) * 16 + c16;
  const int64_t g = (o - c16) * 2;  // the 16-channel group in halves (64 B = 32 halves)
  const __half h = __float2half_rn(x);
  const __half l = __float2half_rn(x - __half2float(h));
  out[g + c16] = *reinterpret_cast<const uint16_t*>(&h);
  out[g + 16 + c16] = *reinterpret_cast<const uint16_t*>(&l);
}

// NCHW16c element e (relative to image img_begin) <- value(seed, logical NCHW index)
__global__ void fill_input_kernel(float* __restrict__ out, uint64_t seed, int64_t n_elems,
                                  int64_t img_begin, int Cb, int H, int W, int c_logical) {
  const uint64_t key = seeded::mix(seed);
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n_elems;
       e += int64_t(gridDim.x) * blockDim.x) {
    int64_t t = e;
    const int c16 = int(t & 15);
    t >>= 4;
    const int w = int(t % W);
    t /= W;
    const int h = int(t % H);
    t /= H;
    const int cb = int(t % Cb);
    const int64_t n = t / Cb + img_begin;
    const int c = cb * 16 + c16;
    float v = 0.f;
    if (c < c_logical) v = seeded::value(key, ((n * c_logical + c) * H + h) * W + w);
    out[e] = v;
  }
}

// KCRS16c16k element e <- value(seed, logical KCRS index)
__global__ void fill_filter_kernel(float* __restrict__ out, uint64_t seed, int64_t n_elems,
                                   int Cb, int R, int S, int c_logical) {
  const uint64_t key = seeded::mix(seed);
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n_elems;
       e += int64_t(gridDim.x) * blockDim.x) {
    int64_t t = e;
    const int k16 = int(t & 15);
    t >>= 4;
    const int c16 = int(t & 15);
    t >>= 4;
    const int s = int(t % S);
    t /= S;
    const int r = int(t % R);
    t /= R;
    const int cb = int(t % Cb);
    const int64_t kb = t / Cb;
    const int c = cb * 16 + c16;
    const int64_t k = kb * 16 + k16;
    float v = 0.f;
    if (c < c_logical) v = seeded::value(key, ((k * c_logical + c) * R + r) * S + s);
    out[e] = v;
  }
}

__global__ void pack_input_kernel(const float* __restrict__ nchw, float* __restrict__ out,
                                  int64_t n_elems, int Cb, int H, int W, int c_logical) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n_elems;
       e += int64_t(gridDim.x) * blockDim.x) {
    int64_t t = e;
    const int c16 = int(t & 15);
    t >>= 4;
    const int w = int(t % W);
    t /= W;
    const int h = int(t % H);
    t /= H;
    const int cb = int(t % Cb);
    const int64_t n = t / Cb;
    const int c = cb * 16 + c16;
    out[e] = c < c_logical ? nchw[((n * c_logical + c) * H + h) * W + w] : 0.f;
  }
}

__global__ void pack_filter_kernel(const float* __restrict__ kcrs, float* __restrict__ out,
                                   int64_t n_elems, int Cb, int R, int S, int c_logical) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n_elems;
       e += int64_t(gridDim.x) * blockDim.x) {
    int64_t t = e;
    const int k16 = int(t & 15);
    t >>= 4;
    const int c16 = int(t & 15);
    t >>= 4;
    const int s = int(t % S);
    t /= S;
    const int r = int(t % R);
    t /= R;
    const int cb = int(t % Cb);
    const int64_t kb = t / Cb;
    const int c = cb * 16 + c16;
    const int64_t k = kb * 16 + k16;
    out[e] = c < c_logical ? kcrs[((k * c_logical + c) * R + r) * S + s] : 0.f;
  }
}

// row-major B[K][N] -> KCRS16c16k [N/16][K/16][1][1][16c][16k] (the GEMM's 1x1 filter)
__global__ void gemm_pack_b_kernel(const float* __restrict__ b, float* __restrict__ out, int64_t K,
                                   int64_t N) {
  const int64_t n_elems = K * N;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n_elems;
       e += int64_t(gridDim.x) * blockDim.x) {
    int64_t t = e;
    const int k16 = int(t & 15);
    t >>= 4;
    const int c16 = int(t & 15);
    t >>= 4;
    const int64_t cb = t % (K / 16);
    const int64_t kb = t / (K / 16);
    out[e] = b[(cb * 16 + c16) * N + kb * 16 + k16];
  }
}

__global__ void unpack_output_kernel(const float* __restrict__ in16, float* __restrict__ nkpq,
                                     int64_t n_elems, int Kb, int PQ) {
  // element e of NKPQ: ((n*K + k)*PQ + pq)
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n_elems;
       e += int64_t(gridDim.x) * blockDim.x) {
    int64_t t = e;
    const int pq = int(t % PQ);
    t /= PQ;
    const int k = int(t % (Kb * 16));
    const int64_t n = t / (Kb * 16);
    nkpq[e] = in16[((n * Kb + k / 16) * PQ + pq) * 16 + (k & 15)];
  }
}

void launch_fold_filter(const conv_plan* P, const float* flt, cudaStream_t st);
int grid_for(int64_t n);

void launch_bwd_filter(const conv_plan* P, const float* flt, cudaStream_t st);

// Filter pack of the few-channel kernel (conv_pp.cuh): per tap-pair MMA i and
// N tile, a [kh][bn/8][8 rows][4 channels] block (SWIZZLE_NONE K-major core
// matrices): kh 0 = tap_a's channels 0..3, kh 1 = tap_b's (zero for the
// partner of an odd tap, and for channels >= C).
struct PpTaps {
  int tap_a[psconv::kPpMaxMma], tap_b[psconv::kPpMaxMma];
};
// (split: 3xTF32 N-concat blocks of 2 bn rows, [kh][2 bn / 8 groups][8][4]: groups < bn/8
// hold hi = trunc_tf32(x), the rest lo = x - hi; n_elems counts both halves)
__global__ void pp_pack_filter_kernel(const float* __restrict__ flt, float* __restrict__ out,
                                      int split, int64_t n_elems, int bn, int nmma, int RS,
                                      int C, const __grid_constant__ PpTaps taps) {
  ptx::griddep_launch_dependents();
  const int rows = split ? 2 * bn : bn;  // B rows per MMA block
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n_elems;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int c4 = int(e & 3), nr = int((e >> 2) & 7);
    const int64_t rest = e >> 5;
    const int g = int(rest % (rows / 8)), kh = int((rest / (rows / 8)) & 1);
    const int64_t blk = rest / (rows / 4);  // tk * nmma + i
    const int i = int(blk % nmma), tk = int(blk / nmma);
    const int tap = kh == 0 ? taps.tap_a[i] : taps.tap_b[i];
    const bool is_lo = split && g >= bn / 8;
    const int ng = is_lo ? g - bn / 8 : g;
    const int64_t n = int64_t(tk) * bn + ng * 8 + nr;
    float x = 0.f;
    if (tap >= 0 && c4 < C) x = flt[((n / 16) * RS + tap) * 256 + c4 * 16 + (n & 15)];
    if (split) {
      const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
      out[e] = is_lo ? x - h : h;
    } else {
      out[e] = x;
    }
  }
}

void launch_prepack(const conv_plan* P, const float* flt, cudaStream_t st) {
  if (P->pp) {
    const psconv::PpGeom& g = P->ppg;
    PpTaps t{};
    for (int i = 0; i < g.nmma; ++i) {
      t.tap_a[i] = g.tap_a[i];
      t.tap_b[i] = g.tap_b[i];
    }
    const bool split3 = P->mode != PSCONV_MODE_TF32;  // (f16x2 plans: the pp kernel's 3xTF32 arithmetic)
    const int64_t n = int64_t(g.b_bytes) / 4 * (split3 ? 2 : 1);
    pp_pack_filter_kernel<<<int((n + 255) / 256), 256, 0, st>>>(
        flt, P->flt_pack, split3 ? 1 : 0, n, g.bn, g.nmma, int(P->d.kh * P->d.kw), P->pp, t);
    CUDA_OK(cudaGetLastError());
    return;
  }
  if (P->bwd_data) {
    launch_bwd_filter(P, flt, st);
    flt = P->wtrans;
  }
  if (P->fold) {
    launch_fold_filter(P, flt, st);
    flt = P->wfold;
  }
  if (P->mode == PSCONV_MODE_F16X2) {
    // |max| of the filter -> B scale, then rows of fp16 hi|lo (same row layout as the
    // fp32 prepack: 64-B rows, or 128-B rows pairing channel blocks)
    const conv_desc& kd = P->kd;
    const int Kb = int(kd.nOfm / 16), CRS = int(kd.nIfm / 16 * kd.kh * kd.kw);
    const int64_t n = int64_t(kd.nOfm) * kd.nIfm * kd.kh * kd.kw;
    CUDA_OK(cudaMemsetAsync(P->absmax, 0, sizeof(unsigned), st));
    absmax_kernel<<<grid_for(n / 4), 256, 0, st>>>(flt, n, P->absmax);
    prepack_filter_f16_kernel<<<Kb * CRS, 256, 0, st>>>(flt, reinterpret_cast<uint16_t*>(P->flt_pack), int(kd.nOfm),
                                                        CRS, int(kd.kh * kd.kw), P->b128 ? 1 : 0, P->absmax);
    CUDA_OK(cudaGetLastError());
    return;
  }
  const conv_desc& kd = P->kd;
  const int Kb = int(kd.nOfm / 16), CRS = int(kd.nIfm / 16 * kd.kh * kd.kw);
  const bool split3 = P->mode == PSCONV_MODE_3XTF32;
  prepack_filter_kernel<<<Kb * CRS, 256, 0, st>>>(flt, P->flt_pack,
                                                  split3 ? P->flt_pack + P->flt_elems : nullptr,
                                                  int(kd.nOfm), CRS, int(kd.kh * kd.kw),
                                                  split3 ? 1 : 0, P->b128 ? 1 : 0,
                                                  P->ncat ? P->sched.bn : 0);
  CUDA_OK(cudaGetLastError());
}

// (c,s) fold of the input into `phases` column-phase planes:
//   out[n][ph][h][wq][s'*C + c] = in[n][0][h][wq*phases + ph - pw + s'][c]
// for s' < G, c < C (zero outside the row and in the 16 - G*C spare channels).
// With phases = stride_w the strided conv reads each plane at unit stride (no
// half-used rows). One thread writes one folded pixel (4 x 16-B stores) from
// one 16-B load per tap (C <= 4) or two (C <= 8).
__global__ void fold_input_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t n_px,
                                  int H, int W, int Wq, int phases, int pw, int C, int G) {
  ptx::griddep_launch_dependents();
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n_px;
       e += int64_t(gridDim.x) * blockDim.x) {
    int64_t t = e;
    const int wq = int(t % Wq);
    t /= Wq;
    const int h = int(t % H);
    t /= H;
    const int ph = int(t % phases);
    const int64_t n = t / phases;
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = 0.f;
    const int w0 = wq * phases + ph - pw;
    const float* row = in + (n * H + h) * int64_t(W) * 16;
    // all taps' loads issued together (G <= 8)
    float4 x[8], y[8];
#pragma unroll
    for (int sp = 0; sp < 8; ++sp) {
      const int col = w0 + sp;
      const bool ok = sp < G && col >= 0 && col < W;
      x[sp] = ok ? __ldg(reinterpret_cast<const float4*>(row + col * 16)) : make_float4(0.f, 0.f, 0.f, 0.f);
      y[sp] = (ok && C > 4) ? __ldg(reinterpret_cast<const float4*>(row + col * 16) + 1)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int sp = 0; sp < 8; ++sp) {
      const float c8[8] = {x[sp].x, x[sp].y, x[sp].z, x[sp].w, y[sp].x, y[sp].y, y[sp].z, y[sp].w};
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < C && sp < G && sp * C + c < 16) v[(sp * C + c) & 15] = c8[c];
    }
    float4* dst = reinterpret_cast<float4*>(out + e * 16);
#pragma unroll
    for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
}

// the matching filter fold: KCRS16c16k [Kb][1][R][S][16c][16k] -> [Kb][1][R][S'][16c][16k]
__global__ void fold_filter_kernel(const float* __restrict__ flt, float* __restrict__ out, int64_t n_elems,
                                   int R, int S, int Sf, int C, int G) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n_elems;
       e += int64_t(gridDim.x) * blockDim.x) {
    int64_t t = e;
    const int k16 = int(t & 15);
    t >>= 4;
    const int c16 = int(t & 15);
    t >>= 4;
    const int sg = int(t % Sf);
    t /= Sf;
    const int r = int(t % R);
    const int64_t kb = t / R;
    const int sp = c16 / C, c = c16 % C;
    const int sx = sg * G + sp;
    float v = 0.f;
    if (sp < G && sx < S) v = flt[((kb * R + r) * S + sx) * 256 + c * 16 + k16];
    out[e] = v;
  }
}

// Backward data: the forward filter KCRS16c16k [Kb][Cb][R][S][16c][16k] becomes the
// filter of the transposed conv, [Cb][Kb][U][V][16k][16c] with the taps flipped:
// W'[c][k][u][v] = W[k][c][sh*(U-1-u) + rho_h][sw*(V-1-v) + rho_w] -- for stride 1
// (U, V = R, S, rho = 0) W[k][c][R-1-u][S-1-v]; for a phase of a strided layer the
// forward taps of that phase (r = rho_h mod sh, s = rho_w mod sw).
__global__ void bwd_filter_kernel(const float* __restrict__ w, float* __restrict__ out, int64_t n_elems,
                                  int Kb, int Cb, int R, int S, int U, int V, int sh, int sw, int rho_h,
                                  int rho_w) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n_elems;
       e += int64_t(gridDim.x) * blockDim.x) {
    int64_t t = e;
    const int c16 = int(t & 15);  // output channel of the transposed conv (forward input c)
    t >>= 4;
    const int k16 = int(t & 15);  // its input channel (forward output k)
    t >>= 4;
    const int v = int(t % V);
    t /= V;
    const int u = int(t % U);
    t /= U;
    const int kb = int(t % Kb);
    const int cb = int(t / Kb);
    const int r = sh * (U - 1 - u) + rho_h, s = sw * (V - 1 - v) + rho_w;
    out[e] = w[((((int64_t(kb) * Cb + cb) * R + r) * S + s) * 16 + c16) * 16 + k16];
  }
}

void launch_bwd_filter(const conv_plan* P, const float* flt, cudaStream_t st) {
  const conv_desc& f = P->fwd;
  const int U = int(P->d.kh), V = int(P->d.kw);
  const int64_t n = f.nOfm * f.nIfm * U * V;
  bwd_filter_kernel<<<grid_for(n), 256, 0, st>>>(flt, P->wtrans, n, int(f.nOfm / 16), int(f.nIfm / 16),
                                                 int(f.kh), int(f.kw), U, V, int(f.stride_h),
                                                 int(f.stride_w), P->ph_rho_h, P->ph_rho_w);
  CUDA_OK(cudaGetLastError());
}

// dX positions of a phase without filter taps (h = a mod sh, w = b mod sw): zero
__global__ void zero_phase_kernel(float* __restrict__ out, int64_t n_px, int H, int W, int Ha, int Wb,
                                  int sh, int sw, int a, int b) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n_px * 4;
       e += int64_t(gridDim.x) * blockDim.x) {
    int64_t t = e >> 2;  // (img, cb, i, j) of the phase; 4 float4 per 16-channel pixel
    const int j = int(t % Wb);
    t /= Wb;
    const int i = int(t % Ha);
    t /= Ha;  // img * Cb + cb
    const int64_t px = (t * H + int64_t(sh) * i + a) * W + int64_t(sw) * j + b;
    reinterpret_cast<float4*>(out + px * 16)[e & 3] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

void launch_fold_filter(const conv_plan* P, const float* flt, cudaStream_t st) {
  const int64_t n = P->kd.nOfm * 16 * P->kd.kh * P->kd.kw;
  fold_filter_kernel<<<grid_for(n), 256, 0, st>>>(flt, P->wfold, n, int(P->d.kh), int(P->d.kw),
                                                  int(P->kd.kw), P->fold, P->fold_g);
  CUDA_OK(cudaGetLastError());
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return int(g);
}

// ---------------------------------------------------------------- launch geometry
// Switches to the plan's device for the duration of an entry point (every C-ABI call that
// launches or allocates), restoring the caller's current device on exit.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int device) {
    int cur = 0;
    CUDA_OK(cudaGetDevice(&cur));
    if (cur != device) {
      CUDA_OK(cudaSetDevice(device));
      prev = cur;
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// cudaFuncAttributeMaxDynamicSharedMemorySize is per device context: set once per
// (kernel instantiation, device) -- the caller's current device is the plan's (DeviceGuard).
struct SmemAttr {
  std::mutex mu;
  uint64_t done = 0;  // bit d: set on device d
  template <typename K>
  cudaError_t ensure(K kernel, int bytes, int device) {
    std::lock_guard<std::mutex> g(mu);
    if (device < 64 && ((done >> device) & 1u)) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess && device < 64) done |= uint64_t(1) << device;
    return e;
  }
};

// Output-tile groups of a launch over img_count images (conv_fwd_sm100's persistent
// schedule: M tiles of the pixel box, CS of them per cluster, times the N tiles).
int64_t launch_groups(const conv_plan* P, int64_t img_count) {
  const conv_desc& d = P->kd;
  const Schedule& s = P->sched;
  const int64_t mt = ((d.ofw + s.qb - 1) / s.qb) * ((d.ofh + s.pb - 1) / s.pb) * ((img_count + s.nb - 1) / s.nb);
  return (mt + s.cs - 1) / s.cs * (d.nOfm / s.bn);
}

// Pipeline stages per whole tile (halo mode: one B stage per (channel group, tap)).
int launch_nst(const conv_plan* P) {
  const conv_desc& d = P->kd;
  const Schedule& s = P->sched;
  const int Cb = int(d.nIfm / 16);
  if (s.halo) return (Cb % s.kps == 0 ? Cb / s.kps : Cb) * int(s.tc ? d.kh : d.kh * d.kw);
  return (Cb * int(d.kh * d.kw) + s.kps - 1) / s.kps;
}

// Split-K work units (recipe ks:S): the tail split cuts only the tiles of the last, partial
// wave into ksplit stage ranges; kt:1 (split_all) cuts every tile. Fused epilogues (ReLU
// needs the whole sum) and halo mode never split.
struct SplitGeom {
  int ksplit, split_stages, split_from, units;
};
SplitGeom split_geom(const conv_plan* P, int groups, int nst, bool fused) {
  const Schedule& s = P->sched;
  SplitGeom g{};
  g.ksplit = (fused || s.halo) ? 1 : std::max(1, s.ksplit);
  g.split_stages = (nst + g.ksplit - 1) / g.ksplit;
  g.ksplit = (nst + g.split_stages - 1) / g.split_stages;  // no empty units
  const int clusters = P->num_sms / s.cs;
  g.split_from = g.ksplit > 1 ? (s.split_all ? 0 : groups / clusters * clusters) : groups;
  if (g.split_from == groups) g.ksplit = 1;  // no partial wave: nothing to split
  g.units = g.split_from + (groups - g.split_from) * g.ksplit;
  return g;
}

// ---------------------------------------------------------------- launch
template <int BN, bool SPLIT3, int CS, int EPI, int EG, bool F16>
void launch_conv(const conv_plan* P, const ConvParams& prm, const CUtensorMap& a,
                 const CUtensorMap& b, const CUtensorMap& blo, const CUtensorMap& o, cudaStream_t st) {
  if constexpr (BN / CS < 8 || (SPLIT3 && CS == 2) || (EG == 2 && BN < 64) || (F16 && (!SPLIT3 || CS == 2))) {
    throw RuntimeError("unsupported (bn, cluster, mode, epilogue groups) combination");
  } else {
    constexpr bool PAIR = CS == 2;
    using Cfg = KernelCfg<BN, SPLIT3, PAIR, EG>;
    static SmemAttr attr_once;  // per instantiation, per device
    CUDA_OK(attr_once.ensure(conv_fwd_sm100<BN, SPLIT3, PAIR, EPI, EG, F16>, Cfg::kSmemBytes, P->device));
    const int max_clusters = P->num_sms / CS;
    const int clusters = prm.groups < max_clusters ? prm.groups : max_clusters;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(clusters * CS);
    cfg.blockDim = dim3(Cfg::kThreads);
    cfg.dynamicSmemBytes = Cfg::smem_bytes(prm.ring_bytes, prm.ostages);
    cfg.stream = st;
    // programmatic stream serialization (PDL): the prologue overlaps the
    // preceding kernel; the producer's griddepcontrol.wait orders the operands
    cudaLaunchAttribute attr[2];
    int na = 0;
    static const bool no_pdl = std::getenv("PSCONV_NO_PDL") != nullptr;
    if (!no_pdl) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    if (CS > 1) {  // plain launch for single-CTA clusters
      attr[na].id = cudaLaunchAttributeClusterDimension;
      attr[na].val.clusterDim.x = CS;
      attr[na].val.clusterDim.y = 1;
      attr[na].val.clusterDim.z = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    CUDA_OK(cudaLaunchKernelEx(&cfg, conv_fwd_sm100<BN, SPLIT3, PAIR, EPI, EG, F16>, prm, a, b, blo, o));
  }
}

template <bool SPLIT3, int CS, int EPI, int EG, bool F16>
void dispatch_bn_eg(int bn, const conv_plan* P, const ConvParams& prm, const CUtensorMap& a,
                    const CUtensorMap& b, const CUtensorMap& blo, const CUtensorMap& o, cudaStream_t st) {
  switch (bn) {
    case 16: return launch_conv<16, SPLIT3, CS, EPI, EG, F16>(P, prm, a, b, blo, o, st);
    case 32: return launch_conv<32, SPLIT3, CS, EPI, EG, F16>(P, prm, a, b, blo, o, st);
    case 64: return launch_conv<64, SPLIT3, CS, EPI, EG, F16>(P, prm, a, b, blo, o, st);
    case 128: return launch_conv<128, SPLIT3, CS, EPI, EG, F16>(P, prm, a, b, blo, o, st);
    case 256: return launch_conv<256, SPLIT3, CS, EPI, EG, F16>(P, prm, a, b, blo, o, st);
    default: throw RuntimeError("unsupported bn");
  }
}

// two epilogue groups (recipe eg:2) for bn >= 64; the fused (bias/ReLU)
// epilogue always runs one group (fewer instantiations)
template <bool SPLIT3, int CS, int EPI, bool F16>
void dispatch_bn(int bn, const conv_plan* P, const ConvParams& prm, const CUtensorMap& a,
                 const CUtensorMap& b, const CUtensorMap& blo, const CUtensorMap& o, cudaStream_t st) {
  if constexpr (EPI != kEpiFused) {
    if (prm.egroups == 2 && bn >= 64) return dispatch_bn_eg<SPLIT3, CS, EPI, 2, F16>(bn, P, prm, a, b, blo, o, st);
  }
  return dispatch_bn_eg<SPLIT3, CS, EPI, 1, F16>(bn, P, prm, a, b, blo, o, st);
}

template <bool SPLIT3, bool F16 = false>
void dispatch_cs(int cs, int bn, const conv_plan* P, const ConvParams& prm, const CUtensorMap& a,
                 const CUtensorMap& b, const CUtensorMap& blo, const CUtensorMap& o, cudaStream_t st) {
  switch (cs) {
    case 1:
      if (prm.ksplit > 1) return dispatch_bn<SPLIT3, 1, kEpiSplit, F16>(bn, P, prm, a, b, blo, o, st);
      return prm.bias || prm.relu ? dispatch_bn<SPLIT3, 1, kEpiFused, F16>(bn, P, prm, a, b, blo, o, st)
                                  : dispatch_bn<SPLIT3, 1, kEpiStore, F16>(bn, P, prm, a, b, blo, o, st);
    case 2:
      if constexpr (!F16) {
        if (prm.ksplit > 1) return dispatch_bn<SPLIT3, 2, kEpiSplit, false>(bn, P, prm, a, b, blo, o, st);
        return prm.bias || prm.relu ? dispatch_bn<SPLIT3, 2, kEpiFused, false>(bn, P, prm, a, b, blo, o, st)
                                    : dispatch_bn<SPLIT3, 2, kEpiStore, false>(bn, P, prm, a, b, blo, o, st);
      }
      [[fallthrough]];
    default: throw RuntimeError("unsupported cluster size");
  }
}

// Launches the plan on images [0, img_count) of `in` / `out` (already offset to
// the first image). Validation is the caller's (conv_fwd / conv_fwd_host).
template <int BN, bool SPLIT3>
void launch_pp_kernel(const conv_plan* P, const PpParams& prm, const CUtensorMap& ta, const CUtensorMap& tout,
                      int smem, cudaStream_t st) {
  static SmemAttr attr_once;  // per instantiation, per device
  CUDA_OK(attr_once.ensure(conv_pp_sm100<BN, SPLIT3>, 227 * 1024, P->device));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min(prm.groups, P->num_sms));
  cfg.blockDim = dim3(PpCfg<BN, SPLIT3>::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = std::getenv("PSCONV_NO_PDL") ? 0 : 1;
  CUDA_OK(cudaLaunchKernelEx(&cfg, conv_pp_sm100<BN, SPLIT3>, prm, ta, tout));
}

// few-channel kernel (recipe pp:C): input parity planes read at 16 B per pixel
void launch_pp(const conv_plan* P, const float* in, const float* flt, float* out, int64_t img_count,
               cudaStream_t st, unsigned flags) {
  const conv_desc& d = P->d;
  const PpGeom& g = P->ppg;
  if (!(flags & PSCONV_FLAG_PREPACKED)) {
    launch_prepack(P, flt, st);
    P->prepacked = false;
  }
  const int Kb = int(d.nOfm / 16), H = int(d.ifh), W = int(d.ifw), Pp = int(d.ofh), Q = int(d.ofw);
  CUtensorMap ta, tout;
  {
    const cuuint64_t dims[5] = {16, cuuint64_t(Q), cuuint64_t(Pp), cuuint64_t(Kb), cuuint64_t(img_count)};
    const cuuint64_t strides[4] = {64, cuuint64_t(Q) * 64, cuuint64_t(Pp) * Q * 64, cuuint64_t(Kb) * Pp * Q * 64};
    const cuuint32_t box[5] = {16, 8, 16, 1, 1};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    encode(&tout, out, 5, dims, strides, box, estr);
  }
  {
    // channels 0..3 of each pixel (16 B), parity planes via element strides
    const cuuint64_t dims[5] = {16, cuuint64_t(W), cuuint64_t(H), cuuint64_t(img_count), 1};
    const cuuint64_t strides[4] = {64, cuuint64_t(W) * 64, cuuint64_t(H) * W * 64, cuuint64_t(H) * W * 64};
    const cuuint32_t box[5] = {4, cuuint32_t(g.PC * g.s), cuuint32_t(g.PR * g.s), 1, 1};
    const cuuint32_t estr[5] = {1, cuuint32_t(g.s), cuuint32_t(g.s), 1, 1};
    encode(&ta, in, 5, dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_NONE);
  }
  PpParams prm{};
  prm.img_count = int(img_count);
  prm.P = Pp;
  prm.Q = Q;
  prm.s = g.s;
  prm.ph = int(d.pad_h);
  prm.pw = int(d.pad_w);
  prm.tiles_q = (Q + 7) / 8;
  prm.tiles_p = (Pp + 15) / 16;
  prm.tiles_k = g.tiles_k;
  const int64_t groups = int64_t(prm.tiles_q) * prm.tiles_p * img_count * g.tiles_k;
  if (groups >= (int64_t(1) << 31)) throw ConfigError("too many tiles");
  prm.groups = int(groups);
  prm.nmma = g.nmma;
  prm.planes = g.planes;
  prm.plane_bytes = g.plane_bytes;
  prm.pitch = g.pitch;
  prm.box_bytes = g.box_bytes;
  prm.stage_bytes = g.stage_bytes;
  prm.lo_off = g.lo_off;
  prm.stages = g.stages;
  prm.b_bytes = g.b_bytes;
  for (int i = 0; i < g.nmma; ++i) {
    prm.a_off[i] = g.a_off[i];
    prm.a_lbo[i] = g.a_lbo[i];
  }
  prm.bpack = P->flt_pack;
  prm.accumulate = (flags & PSCONV_FLAG_ACCUMULATE) ? 1 : 0;
  const bool split3 = P->mode != PSCONV_MODE_TF32;  // (f16x2 plans: the pp kernel's 3xTF32 arithmetic)
  if (g.bn == 64)
    split3 ? launch_pp_kernel<64, true>(P, prm, ta, tout, g.smem_bytes, st)
           : launch_pp_kernel<64, false>(P, prm, ta, tout, g.smem_bytes, st);
  else
    split3 ? launch_pp_kernel<128, true>(P, prm, ta, tout, g.smem_bytes, st)
           : launch_pp_kernel<128, false>(P, prm, ta, tout, g.smem_bytes, st);
}

void launch_range(const conv_plan* P, const float* in, const float* flt, float* out, int64_t img_count,
                  cudaStream_t st, unsigned flags, const float* bias = nullptr) {
  const bool prepacked = (flags & PSCONV_FLAG_PREPACKED) != 0;
  if (!P->phase_plans.empty() || !P->zero_phases.empty()) {
    // strided backward data: one stride-1 transposed conv per output phase, each storing
    // through its strided view of dX (out + the phase's first pixel); tap-less phases zeroed
    const conv_desc& f = P->fwd;
    const int H = int(f.ifh), W = int(f.ifw), sh = int(f.stride_h), sw = int(f.stride_w);
    for (const conv_plan* c : P->phase_plans)
      launch_range(c, in, flt, out + (int64_t(c->ph_a) * W + c->ph_b) * 16, img_count, st, flags, bias);
    if (!(flags & PSCONV_FLAG_ACCUMULATE))
      for (const auto& ab : P->zero_phases) {
        const int Ha = (H - ab.first + sh - 1) / sh, Wb = (W - ab.second + sw - 1) / sw;
        const int64_t n_px = img_count * (f.nIfm / 16) * Ha * Wb;
        zero_phase_kernel<<<grid_for(n_px * 4), 256, 0, st>>>(out, n_px, H, W, Ha, Wb, sh, sw, ab.first,
                                                              ab.second);
        CUDA_OK(cudaGetLastError());
      }
    if (!prepacked) P->prepacked = false;
    return;
  }
  if (P->pp) {
    if (bias || (flags & PSCONV_FLAG_RELU)) throw ConfigError("gpu pp kernel: no fused bias/ReLU epilogue");
    return launch_pp(P, in, flt, out, img_count, st, flags);
  }
  const conv_desc& d = P->kd;  // the kernel's descriptor (folded for fold:C plans)
  if (P->fold) {  // planes [img][phase][H][Wq][16], Wq = kd.ifw
    const int64_t n_px = img_count * P->fold_phases * d.ifh * d.ifw;
    fold_input_kernel<<<grid_for(n_px), 256, 0, st>>>(in, P->xfold, n_px, int(P->d.ifh), int(P->d.ifw),
                                                      int(d.ifw), P->fold_phases, int(P->d.pad_w), P->fold,
                                                      P->fold_g);
    CUDA_OK(cudaGetLastError());
    in = P->xfold;
  }
  const Schedule& s = P->sched;
  const int Cb = int(d.nIfm / 16), Kb = int(d.nOfm / 16);
  const int H = int(d.ifh), W = int(d.ifw), R = int(d.kh), S = int(d.kw);
  const int Pp = int(d.ofh), Q = int(d.ofw);
  const bool split3 = split_mode(P->mode);  // 3xTF32 / f16x2: split-stage geometry
  const bool f16 = P->mode == PSCONV_MODE_F16X2;
  unsigned* amax_a = nullptr;
  if (f16) {
    // |max| of the input range -> the A scale (read by the kernel after griddepcontrol.wait),
    // in the plan's input slot, cleared first by every call (eager or captured alike: a
    // replayed graph and a later eager call never see each other's value)
    const int64_t n = img_count * Cb * H * W * 16;
    amax_a = P->absmax + 1;
    CUDA_OK(cudaMemsetAsync(amax_a, 0, sizeof(unsigned), st));
    absmax_kernel<<<grid_for(n / 4), 256, 0, st>>>(in, n, amax_a);
    CUDA_OK(cudaGetLastError());
  }

  // A: input viewed as [img_count][Cb][H][W][16] from the range's first image
  CUtensorMap ta, tb, tblo, tout;
  // output viewed as [img_count][Kb][P][Q][16] from the first image; the box is
  // the pixel tile (no stride factor); stores outside the layer are clipped
  {
    // (a phase of a strided backward-data plan stores every out_sw-th pixel of every
    // out_sh-th row of the parent's out_H x out_W output)
    const float* base = out;
    const cuuint64_t oH = P->out_H ? cuuint64_t(P->out_H) : cuuint64_t(Pp);
    const cuuint64_t oW = P->out_W ? cuuint64_t(P->out_W) : cuuint64_t(Q);
    const cuuint64_t dims[5] = {16, cuuint64_t(Q), cuuint64_t(Pp), cuuint64_t(Kb),
                                cuuint64_t(img_count)};
    const cuuint64_t strides[4] = {64 * cuuint64_t(P->out_sw), oW * 64 * P->out_sh, oH * oW * 64,
                                   cuuint64_t(Kb) * oH * oW * 64};
    const cuuint32_t box[5] = {16, cuuint32_t(s.qb), cuuint32_t(s.pb), 1, cuuint32_t(s.nb)};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    encode(&tout, base, 5, dims, strides, box, estr);
  }
  const int rows = s.qb * s.pb * s.nb;
  const bool a_packed = rows % 8 == 0;
  const bool a_group = Cb % s.kps == 0 && a_packed;  // one A box spans the stage's blocks
  // A: input NCHW16c [img_count][Cb][H][W][16] viewed with its dims ordered
  // [16c][W][H][img][Cb] (TMA dims need not follow memory order): the box
  // [16][Qb*sw][Pb*sh][Nb][kps] lands as kps contiguous 128-row tiles, one per
  // input-channel block of the stage.
  {
    const float* base = in;
    const int a_cb = P->fold ? P->fold_phases : Cb;  // folded input: column-phase planes
    const cuuint64_t dims[5] = {16, cuuint64_t(W), cuuint64_t(H), cuuint64_t(img_count),
                                cuuint64_t(a_cb)};
    const cuuint64_t strides[4] = {64, cuuint64_t(W) * 64, cuuint64_t(a_cb) * H * W * 64,
                                   cuuint64_t(H) * W * 64};
    if (s.halo) {  // halo box: hr padded rows of hw pixels, kps blocks
      const HaloGeom h = halo_geom(d, s, P->mode);
      const cuuint32_t box[5] = {16, cuuint32_t(h.hw), cuuint32_t(h.hr), 1, cuuint32_t(s.kps)};
      const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
      encode(&ta, base, 5, dims, strides, box, estr);
    } else {
      const cuuint32_t box[5] = {16, cuuint32_t(s.qb * d.stride_w), cuuint32_t(s.pb * d.stride_h),
                                 cuuint32_t(s.nb), cuuint32_t(a_group ? s.kps : 1)};
      const cuuint32_t estr[5] = {1, cuuint32_t(d.stride_w), cuuint32_t(d.stride_h), 1, 1};
      encode(&ta, base, 5, dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_64B,
             d.stride_w > 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    }
  }
  // B: filter prepacked K-major [CRS][K][16c] (hi, and lo for 3xTF32)
  const int K = Kb * 16;
  const float* b_hi = P->flt_pack;
  const float* b_lo = P->mode == PSCONV_MODE_3XTF32 ? P->flt_pack + P->flt_elems : P->flt_pack;
  if (!prepacked) {
    launch_prepack(P, flt, st);
    P->prepacked = false;  // buffer now holds this call's filter
  }
  // B viewed as [16c][K][R*S][Cb] (b128: [32c][K][R*S][Cb/2]); box {c, rows, 1, blocks}
  // (ncat: [B_hi;B_lo] rows per N tile -> 2K rows, boxes of 2 bn rows)
  const int kr = P->ncat ? 2 : 1;
  // tap concat (recipe tc:1): the prepacked [..][R*S][K][..] rows are [..][R][S*K][..] -- a
  // filter row's S taps are one slice of S*K rows (bn == K), loaded as one B box
  const int tcs = s.tc ? S : 1;
  if (P->b128) {
    const cuuint64_t dims[4] = {32, cuuint64_t(K) * kr * tcs, cuuint64_t(R) * S / tcs, cuuint64_t(Cb / 2)};
    const cuuint64_t strides[3] = {128, cuuint64_t(K) * kr * tcs * 128, cuuint64_t(K) * kr * 128 * R * S};
    const cuuint32_t box[4] = {32, cuuint32_t(s.bn / s.cs) * kr * tcs, 1, cuuint32_t(s.kps / 2)};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    encode(&tb, b_hi, 4, dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_128B);
    encode(&tblo, b_lo, 4, dims, strides, box, estr, CU_TENSOR_MAP_SWIZZLE_128B);
  } else {
    const cuuint64_t dims[4] = {16, cuuint64_t(K) * kr * tcs, cuuint64_t(R) * S / tcs, cuuint64_t(Cb)};
    const cuuint64_t strides[3] = {64, cuuint64_t(K) * kr * tcs * 64, cuuint64_t(K) * kr * 64 * R * S};
    const cuuint32_t box[4] = {16, cuuint32_t(s.bn / s.cs) * kr * tcs, 1,
                               cuuint32_t(Cb % s.kps == 0 ? s.kps : 1)};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    encode(&tb, b_hi, 4, dims, strides, box, estr);
    encode(&tblo, b_lo, 4, dims, strides, box, estr);
  }
  ConvParams prm{};
  prm.img_count = int(img_count);
  prm.Cb = Cb;
  prm.H = H;
  prm.W = W;
  prm.Kb = Kb;
  prm.P = Pp;
  prm.Q = Q;
  prm.R = R;
  prm.S = S;
  prm.sh = int(d.stride_h);
  prm.sw = int(d.stride_w);
  prm.ph = int(d.pad_h);
  prm.pw = int(d.pad_w);
  prm.Qb = s.qb;
  prm.Pb = s.pb;
  prm.Nb = s.nb;
  prm.tiles_q = (Q + s.qb - 1) / s.qb;
  prm.tiles_p = (Pp + s.pb - 1) / s.pb;
  prm.tiles_n = int((img_count + s.nb - 1) / s.nb);
  prm.tiles_k = int(d.nOfm / s.bn);
  const int64_t mt = int64_t(prm.tiles_q) * prm.tiles_p * prm.tiles_n;
  const int64_t mg = (mt + s.cs - 1) / s.cs;
  if (mg * prm.tiles_k >= (int64_t(1) << 31)) throw ConfigError("too many tiles");
  prm.mtiles = int(mt);
  prm.mgroups = int(mg);
  prm.groups = int(mg * prm.tiles_k);
  // recipe loop order -> rasterisation: pixel-loop order and ofm_tile position
  int pos[3];
  for (int i = 0; i < 3; ++i) pos[s.raster[i]] = i;
  prm.m_order = pos[0] < pos[2] ? 0 : 1;
  prm.k_outer = pos[1] == 0 ? 1 : 0;
  prm.m_block = s.m_block;
  prm.tap_dw = P->fold ? P->fold_g : 1;
  prm.ksteps = Cb * R * S;
  prm.kps = s.kps;
  prm.cb_group = Cb % s.kps == 0 ? 1 : 0;
  prm.b128 = P->b128 ? 1 : 0;
  prm.cbg = prm.cb_group ? Cb / s.kps : Cb;
  prm.nst = (prm.ksteps + s.kps - 1) / s.kps;
  prm.stages = s.stages;
  {
    const int mult = split3 ? 2 : 1;
    const int brows = s.bn / s.cs;
    prm.stage_bytes = stage_bytes(s, P->mode);
    // one A box for the stage's channel blocks when its rows are whole 8-row
    // swizzle atoms; else one box per block at 8 KB pitch
    prm.a_boxes = (prm.cb_group && a_packed) ? 1 : (prm.cb_group ? s.kps : 1);
    prm.a_pitch = (prm.cb_group && a_packed) ? rows * 64 : 8192;
    prm.a_lo_off = s.kps * 8192;
    prm.b_off = s.kps * 8192 * (s.tmem_a ? 1 : mult);
    prm.b_lo_off = prm.b_off + s.kps * brows * 64;
    prm.tmem_a = s.tmem_a;
    prm.egroups = s.egroups;
    prm.ostages = s.ostages;
    prm.absmax_a = amax_a;
    prm.absmax_b = P->absmax;
    prm.ncat = P->ncat ? 1 : 0;
    if (s.tmem_a) {  // TMEM A ring after the accumulators (2 x bn) and the running sum (bn)
      // accumulators (2 buffers; [D1|D2] of 2 bn columns at bn <= 64) + the running sum,
      // which exists only when a tile's reduction is split into accumulation chunks: with
      // one chunk per tile the ring gets those columns too (bn 64: 8 slots instead of 6,
      // two whole stages of kps = 4, so the splitter fills stage s+1 while the MMAs read
      // stage s -- with 6 slots the two serialised, measured by the CTA-0 clock trace)
      const int chunk_st = ((s.chunk > 0 ? s.chunk : prm.ksteps) + s.kps - 1) / s.kps;
      const bool sum = chunk_st < prm.nst;
      prm.a_slot_col = (((s.bn <= 64 ? 4 : 2) + (sum ? 1 : 0)) * s.bn + 31) / 32 * 32;
      prm.a_slots = std::min(kMaxStages, (512 - prm.a_slot_col) / 32);
      if (prm.a_slots < s.kps) throw RuntimeError("internal: TMEM A ring smaller than a stage");
    }
    prm.ring_bytes = (prm.stages * prm.stage_bytes + 1023) / 1024 * 1024;
    if (s.halo) {
      const HaloGeom h = halo_geom(d, s, P->mode);
      prm.halo = 1;
      prm.hw = h.hw;
      prm.hr = h.hr;
      prm.a_tile = h.a_tile;
      prm.stage_bytes = h.a_stage;
      prm.a_lo_off = h.a_lo_off;
      prm.hb_stages = s.hb_stages;
      prm.hb_stage_bytes = h.b_stage;
      prm.b_res = s.b_res;
      prm.b_lo_off = h.b_lo_off;
      prm.hb_ring_off = prm.stages * h.a_stage;
      prm.ring_bytes = prm.hb_ring_off + (s.b_res ? int(R * S / tcs) * prm.cbg : prm.hb_stages) * h.b_stage;
      prm.nst = prm.cbg * R * S / tcs;  // taps (tap concat: filter rows) per tile = B stages
      prm.tc = s.tc;
      if (prm.stages > kHaloB || prm.hb_stages < (s.b_res ? 1 : 2) || prm.hb_stages > kMaxStages - kHaloB)
        throw RuntimeError("internal: bad halo stage plan");
    }
    if (prm.stages < 2 || prm.stages > kMaxStages || prm.ring_bytes > kStageBudget - (prm.ostages - kOutStages) * kOutStageBytes)
      throw RuntimeError("internal: bad pipeline stage plan");
  }
  const int chunk = s.chunk > 0 ? s.chunk : prm.ksteps;
  prm.chunk_stages = (chunk + s.kps - 1) / s.kps;
  prm.tile_chunks = (prm.nst + prm.chunk_stages - 1) / prm.chunk_stages;
  {
    // split-K units (not with a fused epilogue, whose ReLU needs the whole sum; not halo)
    const SplitGeom sg = split_geom(P, prm.groups, prm.nst, bias != nullptr || (flags & PSCONV_FLAG_RELU));
    prm.ksplit = sg.ksplit;
    prm.split_stages = sg.split_stages;
    prm.split_from = sg.split_from;
    prm.units = sg.units;
    prm.split_ctr = nullptr;
    prm.split_ws = nullptr;
    if (prm.ksplit > 1) {  // scratch sized by conv_plan_create for img_count = nImg
      if (int64_t(prm.groups - prm.split_from) * s.cs > P->split_slots || prm.ksplit > P->split_k)
        throw RuntimeError("internal: split-K scratch smaller than the launch");
      prm.split_ctr = P->split_ctr;
      prm.split_ws = P->split_ws;
    }
  }
  for (int i = 0; i < 3; ++i) prm.kord[i] = s.kord[i];
  prm.accumulate = (flags & PSCONV_FLAG_ACCUMULATE) ? 1 : 0;
  prm.bias = bias;
  prm.relu = (flags & PSCONV_FLAG_RELU) ? 1 : 0;
  // profiling switch (never set in production; results are wrong when non-zero)
  static const int debug_env = [] {
    const char* e = std::getenv("PSCONV_DEBUG");
    return e ? std::atoi(e) : 0;
  }();
  prm.debug = debug_env;
  static unsigned long long* trace_buf = nullptr;
  if ((debug_env & 8) && !trace_buf) CUDA_OK(cudaMalloc(&trace_buf, kTraceWords * 8));
  if (debug_env & 8) CUDA_OK(cudaMemsetAsync(trace_buf, 0, kTraceWords * 8, st));
  prm.debug = debug_env & ~8;  // 1 2 4: skip loads / MMAs / stores; 16: generic halo issuer
  prm.trace = (debug_env & 8) ? trace_buf : nullptr;
  prm.out = out;
  prm.out_img_stride = int64_t(Kb) * Pp * Q * 16;
  if (P->mode == PSCONV_MODE_F16X2)
    dispatch_cs<true, true>(s.cs, s.bn, P, prm, ta, tb, tblo, tout, st);
  else if (split3)
    dispatch_cs<true>(s.cs, s.bn, P, prm, ta, tb, tblo, tout, st);
  else
    dispatch_cs<false>(s.cs, s.bn, P, prm, ta, tb, tblo, tout, st);
  if (prm.trace) {  // profiling: dump CTA 0's clocks (producer | MMA issuer | splitter | epilogue)
    std::vector<unsigned long long> h(kTraceWords);
    CUDA_OK(cudaStreamSynchronize(st));
    CUDA_OK(cudaMemcpy(h.data(), prm.trace, kTraceWords * 8, cudaMemcpyDeviceToHost));
    const long long t0 = static_cast<long long>(h[8 * kTraceStages]);
    auto rel = [&](int i) { return h[i] ? static_cast<long long>(h[i]) - t0 : -1LL; };
    std::fprintf(stderr, "events: setup %lld first-acc %lld last-store %lld stores-done %lld exit %lld\n",
                 rel(8 * kTraceStages + 1), rel(8 * kTraceStages + 4), rel(8 * kTraceStages + 5),
                 rel(8 * kTraceStages + 6), rel(8 * kTraceStages + 7));
    for (int i = 0; i < kTraceStages; ++i) {
      if (!h[i * 4] && !h[4 * kTraceStages + i * 4] && !h[kTraceSplit + 2 * i]) continue;
      std::fprintf(stderr, "trace %3d prod %8lld %8lld %8lld  mma %8lld %8lld %8lld %8lld  split %8lld %8lld\n", i,
                   rel(i * 4), rel(i * 4 + 1), rel(i * 4 + 2), rel(4 * kTraceStages + i * 4),
                   rel(4 * kTraceStages + i * 4 + 3), rel(4 * kTraceStages + i * 4 + 1),
                   rel(4 * kTraceStages + i * 4 + 2), rel(kTraceSplit + 2 * i), rel(kTraceSplit + 2 * i + 1));
    }
    for (int r = 0; r < 16; ++r)
      if (h[kTraceEpiR + 5 * r])
        std::fprintf(stderr, "round %2d start %8lld loaded %8lld bar1 %8lld staged %8lld issued %8lld\n", r,
                     rel(kTraceEpiR + 5 * r), rel(kTraceEpiR + 5 * r + 1), rel(kTraceEpiR + 5 * r + 2),
                     rel(kTraceEpiR + 5 * r + 3), rel(kTraceEpiR + 5 * r + 4));
    for (int c = 0; c < 32; ++c)
      if (h[kTraceEpi + 2 * c])
        std::fprintf(stderr, "epi %2d acc_full %8lld released %8lld\n", c, rel(kTraceEpi + 2 * c),
                     rel(kTraceEpi + 2 * c + 1));
  }
}

}  // namespace
}  // namespace psconv

namespace psconv {
namespace {
// Plan construction for a validated descriptor (conv_plan_create) or for an internal
// phase conv of a strided backward-data plan, whose implied bottom padding is asymmetric
// (the TMA zero-fills the rows past dY; conv_plan_create_bwd_data).
conv_plan* create_plan(const conv_desc& d, int mode, int device, const char* recipe) {
    if (mode != PSCONV_MODE_3XTF32 && mode != PSCONV_MODE_TF32 && mode != PSCONV_MODE_F16X2)
      throw ConfigError("unknown mode " + std::to_string(mode));
    Recipe r;
    Schedule s;
    conv_desc kd = d;
    int fold = 0, fold_g = 1, fold_phases = 1;
    if (recipe && *recipe) {
      r = Recipe::parse(recipe);
      if (r.fold && !r.pp) {
        // (c,s) fold: one 16-channel block holding C real channels, G taps per block
        fold = r.fold;
        fold_g = 16 / fold;
        if (d.nIfm != 16 || d.gemm_block != 16 || fold_g < 2 || d.kw < 2)
          throw ConfigError("fold:C needs nIfm = gemm_block = 16, C <= 8 and kw > 1");
        kd.kw = (d.kw + fold_g - 1) / fold_g;
        // the folded copy carries the left padding. (Splitting it into stride_w
        // column-phase planes read at unit stride measured slower on the stem --
        // 848 vs 639 us for the conv: TMA element strides fetch only the used
        // 64-B rows, so there is no waste to remove; fold_phases stays 1.)
        fold_phases = 1;
        kd.ifw = d.ifw + d.pad_w;
        kd.pad_w = 0;
      }
      s = resolve_schedule(kd, r, mode);
    } else {
      const auto cands = candidate_schedules(d, mode);
      if (cands.empty()) throw ConfigError("no GPU schedule for this descriptor");
      double best = 1e300;
      for (const auto& c : cands) {
        const double us = model_schedule(d, c, mode).us_total;
        if (us < best) {
          best = us;
          s = c;
        }
      }
    }
    int ndev = 0;
    CUDA_OK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw ConfigError("invalid device " + std::to_string(device));
    cudaDeviceProp prop;
    CUDA_OK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
      throw RuntimeError("psconv kernels are built for sm_100a; device is sm_" +
                         std::to_string(prop.major) + std::to_string(prop.minor));
    auto* P = new conv_plan();
    P->d = d;
    P->mode = mode;
    P->device = device;
    P->num_sms = prop.multiProcessorCount;
    P->sched = s;
    P->kd = kd;
    P->fold = fold;
    P->fold_g = fold_g;
    P->fold_phases = fold_phases;
    if (s.pp) {
      P->pp = s.pp;
      P->ppg = pp_geom(d, s.bn, mode);
    }
    // 128-B filter rows pair channel blocks inside a stage: needs even kps dividing Cb
    P->b128 = s.kps % 2 == 0 && (d.nIfm / 16) % s.kps == 0 && std::getenv("PSCONV_NO_B128") == nullptr;
    P->ncat = mode == PSCONV_MODE_3XTF32 && s.bn <= 64 && !s.pp && s.cs == 1 &&
              std::getenv("PSCONV_NO_NCAT") == nullptr;
    P->flt_elems = kd.nOfm * kd.nIfm * kd.kh * kd.kw;
    P->user_flt_elems = d.nOfm * d.nIfm * d.kh * d.kw;
    if (!s.pp) {
      // split-K scratch for the largest launch (all nImg images): the tail split cuts at
      // most one partial wave (< clusters tiles), kt:1 every tile
      const int64_t groups = launch_groups(P, d.nImg);
      if (groups >= (int64_t(1) << 31)) {
        delete P;
        throw ConfigError("too many tiles");
      }
      const SplitGeom sg = split_geom(P, int(groups), launch_nst(P), false);
      if (sg.ksplit > 1) {
        const int64_t clusters = P->num_sms / s.cs;
        const int64_t tiles = s.split_all ? groups : std::min<int64_t>(groups, clusters);
        P->split_slots = tiles * s.cs;
        P->split_k = sg.ksplit;
      }
    }
    {
      DeviceGuard guard(device);
      const int copies = mode == PSCONV_MODE_3XTF32 ? 2 : 1;
      cudaError_t e = cudaMalloc(&P->flt_pack, copies * P->flt_elems * sizeof(float));
      if (e == cudaSuccess) e = cudaMalloc(&P->absmax, 2 * sizeof(unsigned));
      if (e == cudaSuccess) e = cudaMemset(P->absmax, 0, 2 * sizeof(unsigned));
      if (e == cudaSuccess && fold) e = cudaMalloc(&P->wfold, P->flt_elems * sizeof(float));
      if (e == cudaSuccess && fold)
        e = cudaMalloc(&P->xfold, size_t(kd.nImg) * fold_phases * kd.ifh * kd.ifw * 16 * sizeof(float));
      if (e == cudaSuccess && P->split_slots > 0) {
        e = cudaMalloc(&P->split_ctr, size_t(P->split_slots) * 2 * sizeof(int));
        if (e == cudaSuccess) e = cudaMemset(P->split_ctr, 0, size_t(P->split_slots) * 2 * sizeof(int));
        if (e == cudaSuccess)
          e = cudaMalloc(&P->split_ws, size_t(P->split_slots) * P->split_k * 128 * s.bn * sizeof(float));
      }
      if (e != cudaSuccess) {
        cudaFree(P->flt_pack);
        cudaFree(P->absmax);
        cudaFree(P->wfold);
        cudaFree(P->xfold);
        cudaFree(P->split_ctr);
        cudaFree(P->split_ws);
        delete P;
        throw RuntimeError(std::string("cudaMalloc: ") + cudaGetErrorString(e));
      }
    }
    return P;
}
}  // namespace
}  // namespace psconv

namespace psconv {
namespace {
// ---------------------------------------------------------------- backward weight
// Geometry of the pixel-major wgrad kernel (wgrad_kernel.cuh) for the forward layer f:
// tile roles / sizes by a small cost model (MMA cycles at the measured N floor, operand
// bytes per K=8 step at ~64 B/cycle/SM of L2->SMEM delivery, pixel-box and tap waste), the
// pixel box per stage (rows multiple of 8, >= 3-4 ring slots), and the split of the pixel
// range so that the units fill the SMs once. A recipe "gpu=sw:S,kn:K,cn:C,nt:T,box:QxP,
// sp:SPLITS,st:STAGES,ch:K8" overrides any of the choices.
struct WgPick {
  int swap = -1, kn = 0, cn = 0, ntap = 0, qb = 0, pb = 0, splits = 0, stages = 0, chunk = -1, tma = -1;
  int pp = 0;  // tap fold for few-channel layers: the real channel count
  int cl = 0;  // 1: single CTAs, 2: CTA pairs (default: pairs where eligible)
};
WgPick parse_wgrad_recipe(const char* recipe) {
  WgPick w;
  if (!recipe || !*recipe) return w;
  std::string r(recipe);
  const auto pos = r.find("gpu=");
  if (pos == std::string::npos) throw ConfigError("backward-weight recipe: expected 'gpu=key:value,...'");
  std::string body = r.substr(pos + 4);
  size_t i = 0;
  while (i < body.size()) {
    size_t j = body.find(',', i);
    if (j == std::string::npos) j = body.size();
    const std::string kv = body.substr(i, j - i);
    const auto c = kv.find(':');
    if (c == std::string::npos) throw ConfigError("backward-weight recipe: bad item '" + kv + "'");
    const std::string k = kv.substr(0, c), v = kv.substr(c + 1);
    auto num = [&](const std::string& t) {
      char* e = nullptr;
      const long x = std::strtol(t.c_str(), &e, 10);
      if (t.empty() || *e || x < 0) throw ConfigError("backward-weight recipe: bad value '" + kv + "'");
      return int(x);
    };
    if (k == "sw") w.swap = num(v);
    else if (k == "kn") w.kn = num(v);
    else if (k == "cn") w.cn = num(v);
    else if (k == "nt") w.ntap = num(v);
    else if (k == "sp") w.splits = num(v);
    else if (k == "st") w.stages = num(v);
    else if (k == "ch") w.chunk = num(v);
    else if (k == "pp") w.pp = num(v);
    else if (k == "cl") {
      w.cl = num(v);
      if (w.cl < 1 || w.cl > 2) throw ConfigError("backward-weight recipe: cl:1|2");
    }
    else if (k == "tma") {
      w.tma = num(v);
      if (w.tma > 1) throw ConfigError("backward-weight recipe: tma:0|1");
    } else if (k == "box") {
      const auto x = v.find('x');
      if (x == std::string::npos) throw ConfigError("backward-weight recipe: box:QxP");
      w.qb = num(v.substr(0, x));
      w.pb = num(v.substr(x + 1));
    } else {
      throw ConfigError("backward-weight recipe: unknown key '" + k + "'");
    }
    i = j + 1;
  }
  return w;
}

std::string wgrad_recipe(const WgradParams& g) {
  return "gpu=sw:" + std::to_string(g.swap) + ",kn:" + std::to_string(g.kn) + ",cn:" + std::to_string(g.cn) +
         ",nt:" + std::to_string(g.ntap) + ",box:" + std::to_string(g.Qb) + "x" + std::to_string(g.Pb) +
         ",sp:" + std::to_string(g.splits) + ",st:" + std::to_string(g.stages) + ",ch:" + std::to_string(g.chunk_k8) +
         ",tma:" + std::to_string(g.tma) + (g.fc ? ",pp:" + std::to_string(g.fc) : std::string()) +
         (g.pair ? ",cl:2" : "");
}

constexpr int kWgSmemBudget = 227 * 1024 - 6144;  // ring; the rest: alignment, barriers, row/tap tables

WgradParams wgrad_geom_core(const conv_desc& f, int mode, int num_sms, const WgPick& want) {
  const bool split3 = mode == PSCONV_MODE_3XTF32;
  const int C = int(f.nIfm), K = int(f.nOfm), RS = int(f.kh * f.kw);
  const int Cb = C / 16, Kb = K / 16;
  const int P = int(f.ofh), Q = int(f.ofw);
  const int mult = split3 ? 2 : 1;
  auto cdiv = [](int64_t a, int64_t b) { return (a + b - 1) / b; };
  // pixel box for a per-row stage footprint: least waste, then most rows
  auto pick_box = [&](int row_bytes, int min_stages, int& qb, int& pb) {
    const int rows_max = std::max(8, (kWgSmemBudget / min_stages / row_bytes) / 8 * 8);
    double best = 1e30;
    qb = pb = 0;
    for (int q = 1; q <= Q + 7; ++q) {
      if (q > Q && q != (Q + 7) / 8 * 8) continue;
      for (int pp = 1; pp <= P; ++pp) {
        const int rows = q * pp;
        if (rows % 8 || rows > rows_max || rows > 256) continue;
        const double waste = double(cdiv(Q, q) * q * cdiv(P, pp) * pp) / (double(P) * Q);
        // per-stage fixed cost (barrier round trip, box issue) ~ 24 rows of N = 256 MMA time:
        // l3 3x3 TF32 dW 165 -> 142 us going from 32- to 56-row stages, 16-row stages 263 us
        const double score = waste * (1.0 + 24.0 / rows);
        if (score < best - 1e-12) {
          best = score;
          qb = q;
          pb = pp;
        }
      }
    }
    if (!qb) throw ConfigError("backward weight: no pixel box fits");
  };
  struct Cand {
    int swap, kn, cn, ntap, bn;
    double cost;
  };
  std::vector<Cand> cands;
  const int mma_mult = split3 ? 3 : 1;
  auto consider = [&](int swap, int kn, int cn, int ntap) {
    const int bn = swap ? kn : ntap * cn;
    const int m = swap ? ntap * cn : kn;
    if (m != 128 || bn < 32 || bn > 256 || bn % 32) return;
    if (bn != 32 && bn != 64 && bn != 128 && bn != 192 && bn != 256) return;
    if (split3 && bn > 128) return;
    if (cn > std::max(32, (C + 31) / 32 * 32) || kn > std::max(32, (K + 31) / 32 * 32)) return;
    if (want.swap >= 0 && want.swap != swap) return;
    if (want.kn && want.kn != kn) return;
    if (want.cn && want.cn != cn) return;
    if (want.ntap && want.ntap != ntap) return;
    const int64_t tiles = cdiv(K, kn) * cdiv(C, cn) * cdiv(RS, ntap);
    const double mma = std::max(bn / 2.0, bn <= 64 ? 45.0 : 0.0) * mma_mult;
    const double deliver = (128.0 + bn) * 8 * 4 / 64.0;
    const double smem = split3 ? (128.0 + bn) * 8 * 4 * 6 / 128.0 : 0.0;  // TMA + split r/w + 3 MMA reads
    const double k8 = std::max(mma, std::max(deliver, smem));
    cands.push_back({swap, kn, cn, ntap, bn, double(tiles) * k8});
  };
  for (int kn : {32, 64, 128, 256})
    for (int cn : {32, 64, 128, 256})
      for (int nt : {1, 2, 3, 4, 7, 8, 9}) {
        consider(0, kn, cn, nt);
        consider(1, kn, cn, nt);
      }
  if (cands.empty()) throw ConfigError("backward weight: no tile geometry for this layer / recipe");
  const Cand* best = &cands[0];
  for (const Cand& c : cands)
    if (c.cost < best->cost * (1 - 1e-9) || (c.cost <= best->cost * (1 + 1e-9) && c.bn > best->bn)) best = &c;
  WgradParams g{};
  g.N = int(f.nImg);
  g.Cb = Cb;
  g.Kb = Kb;
  g.H = int(f.ifh);
  g.W = int(f.ifw);
  g.P = P;
  g.Q = Q;
  g.R = int(f.kh);
  g.S = int(f.kw);
  g.sh = int(f.stride_h);
  g.sw = int(f.stride_w);
  g.ph = int(f.pad_h);
  g.pw = int(f.pad_w);
  g.swap = best->swap;
  g.kn = best->kn;
  g.cn = best->cn;
  g.ntap = best->ntap;
  g.bn = best->bn;
  g.tiles_k = int(cdiv(K, g.kn));
  g.tiles_c = int(cdiv(C, g.cn));
  g.tiles_t = int(cdiv(RS, g.ntap));
  g.tiles = g.tiles_k * g.tiles_c * g.tiles_t;
  // CTA pairs (cta_group::2, M = 256): two 128-channel output tiles share the pixel range and
  // each CTA stages half of the input channels -- per SM 8 KB of operands per K=8 step instead
  // of 12 at bn = 256. TMA path only; chosen unless the recipe says cl:1 or tma:0.
  // A refinement of the TMA path, decided after it (below); the box is picked for the
  // single-CTA stage and the pair then gets a deeper ring.
  const bool pair_cand = g.swap == 0 && g.ntap == 1 && g.kn == 128 && K % 256 == 0 && g.cn >= 64 && !want.pp;
  if (want.cl == 2 && (!pair_cand || want.tma == 0))
    throw ConfigError("backward-weight recipe: cl:2 needs tma:1, sw:0, nt:1, kn:128, K % 256 == 0, cn >= 64");
  // The pixel box / ring are sized for the CTA's staging footprint: a pair candidate is sized
  // for the pair (half the input channels per CTA: deeper stages, fewer barrier round trips --
  // l4 3x3 TF32 dW 177 -> 130 us at 56 instead of 32 rows); if the gather wins instead, the box
  // is re-picked for the single-CTA footprint.
  const bool pair_try = pair_cand && want.tma != 0 && want.cl != 1;
  auto layout = [&](int xch) {
    const int row_bytes = (xch + g.kn) * 4 * mult;
    if (want.qb) {
      g.Qb = want.qb;
      g.Pb = want.pb;
      if ((g.Qb * g.Pb) % 8 || g.Qb * g.Pb > 256 || g.Qb < 1 || g.Pb < 1)
        throw ConfigError("backward-weight recipe: box rows (QxP) must be a multiple of 8, at most 256");
    } else {
      pick_box(row_bytes, 3, g.Qb, g.Pb);
    }
    g.rows = g.Qb * g.Pb;
    g.tiles_q = int(cdiv(Q, g.Qb));
    g.tiles_p = int(cdiv(P, g.Pb));
    const int64_t nstage = int64_t(g.N) * g.tiles_p * g.tiles_q;
    if (nstage >= (int64_t(1) << 31)) throw ConfigError("backward weight: too many pixel stages");
    g.nstage = int(nstage);
    g.x_bytes = xch * g.rows * 4;
    g.y_bytes = g.kn * g.rows * 4;
    g.stage_bytes = (g.x_bytes + g.y_bytes) * mult;
    g.stages = want.stages ? want.stages : std::min(kWgMaxStages, kWgSmemBudget / g.stage_bytes);
    // one unit per SM: split the pixel stages so that splits x tiles ~ the SM count (at least
    // 2 stages per unit); more units than SMs only when the tiles alone exceed them
    int splits = want.splits;
    if (!splits) splits = int(std::max<int64_t>(1, std::min<int64_t>(num_sms / g.tiles, nstage / 2)));
    splits = int(std::min<int64_t>(splits, nstage));
    g.stage_per_split = int(cdiv(nstage, splits));
    g.splits = int(cdiv(nstage, g.stage_per_split));
    g.units = g.splits * g.tiles;
  };
  layout(pair_try ? g.cn / 2 : g.ntap * g.cn);
  // 3xTF32 accumulation chunks (~32 K=8 steps: error ~6e-8 per step)
  g.chunk_k8 = split3 ? (want.chunk >= 0 ? want.chunk : 32) : 0;
  if (split3 && g.chunk_k8 > 0 && g.chunk_k8 < g.rows / 8) g.chunk_k8 = g.rows / 8;
  g.Cb2 = (Cb + 1) / 2;
  g.Kb2 = (Kb + 1) / 2;
  // TMA path: one relayout pass over X and dY buys dense TMA boxes (about twice the cp.async
  // gather's L2->SM rate). Pick by modelled time: L2->SM bytes at the measured rates (TMA
  // ~10.4 TB/s, gather ~4.5 TB/s: l3 3x3 TF32, tools/_wgt.py), the MMA time at the N floor, the
  // compulsory HBM bytes, plus the relayout pass (read X + dY, write them once per copy) for TMA.
  // HBM-heavy 1x1 layers keep the gather (l1 1x1 64->256 TF32: 272 vs 510 us).
  const bool fits = g.Qb * g.sw <= 256 && g.Pb * g.sh <= 256;
  if (want.tma >= 0) {
    g.tma = want.tma;
  } else if (want.cl == 2) {
    g.tma = 1;
  } else {
    const double xb = 4.0 * f.nImg * Cb * 16 * f.ifh * f.ifw, yb = 4.0 * f.nImg * Kb * 16 * P * Q;
    const double l2 = double(g.units) * g.stage_per_split * (g.ntap * g.cn + g.kn) * g.rows * 4.0;  // hi bytes
    const double k8 = double(g.units) * g.stage_per_split * (g.rows / 8);
    const double mma_cyc = std::max(g.bn / 2.0, g.bn <= 64 ? 45.0 : 0.0) * (split3 ? 3 : 1);
    const double t_mma = k8 * mma_cyc / num_sms / 1.8e9;
    const double hbm = (xb + yb) / 6.0e12;
    // (3xTF32 gather: the producers also split every piece, ~2.2x slower per byte, measured)
    const double t_cp = std::max({t_mma, l2 / (split3 ? 2.0e12 : 4.5e12), hbm});
    const double t_tma = (xb + yb) * (split3 ? 3 : 2) / 6.0e12 + std::max({t_mma, l2 * mult / 10.4e12, hbm});
    g.tma = (fits && t_tma < t_cp) ? 1 : 0;
  }
  if (want.pp) g.tma = 1;  // the tap fold's relayout is the TMA input
  g.pair = (pair_try && g.tma) ? 1 : 0;
  if (pair_try && !g.pair) layout(g.ntap * g.cn);  // the gather won: single-CTA footprint
  if (g.stages < 2 || g.stages > kWgMaxStages || g.stages * g.stage_bytes > kWgSmemBudget)
    throw ConfigError("backward weight: the stage ring does not fit shared memory");
  if (g.tma && (g.Qb * g.sw > 256 || g.Pb * g.sh > 256))
    throw ConfigError("backward weight: tma:1 needs Qb*stride_w and Pb*stride_h <= 256");
  return g;
}

// Few-channel layers (recipe pp:C, C real channels in the first 16-channel block, e.g. the
// ResNet stem's 3): the wgrad of the 1x1 conv over the folded input X' (per output pixel the
// R*S*C window values, padded to a multiple of 32) -- R*S*C / 32 channel groups instead of R*S
// taps x 32 channels of which C are real (the stem: 5 groups for 49 taps of 3 channels).
WgradParams wgrad_geom(const conv_desc& f, int mode, int num_sms, const char* recipe) {
  WgPick want = parse_wgrad_recipe(recipe);
  if (!want.pp) return wgrad_geom_core(f, mode, num_sms, want);
  const int fc = want.pp;
  if (fc > 16 || f.nIfm != 16) throw ConfigError("backward-weight recipe: pp:C needs nIfm = 16 and C <= 16");
  if (want.tma == 0) throw ConfigError("backward-weight recipe: pp:C runs on the TMA path");
  if (want.ntap > 1) throw ConfigError("backward-weight recipe: pp:C folds the taps (no nt:)");
  const int64_t T = f.kh * f.kw * fc;
  conv_desc fd = f;
  fd.nIfm = (T + 31) / 32 * 32;
  fd.kh = fd.kw = 1;
  fd.stride_h = fd.stride_w = 1;
  fd.pad_h = fd.pad_w = 0;
  fd.ifh = f.ofh;
  fd.ifw = f.ofw;
  WgradParams g = wgrad_geom_core(fd, mode, num_sms, want);
  g.fc = fc;
  g.oCb = int(f.nIfm / 16);
  g.oR = int(f.kh);
  g.oS = int(f.kw);
  g.oH = int(f.ifh);
  g.oW = int(f.ifw);
  g.osh = int(f.stride_h);
  g.osw = int(f.stride_w);
  g.oph = int(f.pad_h);
  g.opw = int(f.pad_w);
  return g;
}

template <int BN, bool SPLIT3, bool TMA, bool PAIR = false>
void launch_wgrad_kernel(const conv_plan* P, const WgradParams& g, const CUtensorMap* tm, cudaStream_t st) {
  using Cfg = WgCfg<BN, SPLIT3, TMA, PAIR>;
  const int smem = g.stages * g.stage_bytes + 6144;
  static SmemAttr attr_once;  // the largest ring any plan may use (set once per device)
  CUDA_OK(attr_once.ensure(wgrad_sm100<BN, SPLIT3, TMA, PAIR>, kWgSmemBudget + 6144, P->device));
  cudaLaunchConfig_t cfg{};
  int grid = std::min(g.units, P->num_sms);
  if (PAIR) grid &= ~1;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (!std::getenv("PSCONV_NO_PDL")) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (PAIR) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  CUDA_OK(cudaLaunchKernelEx(&cfg, wgrad_sm100<BN, SPLIT3, TMA, PAIR>, g, tm[0], tm[1], tm[2], tm[3]));
}

template <int BN, bool SPLIT3>
void launch_wgrad_bn(const conv_plan* P, const WgradParams& g, const CUtensorMap* tm, cudaStream_t st) {
  if (g.pair) {
    if constexpr (BN >= 64) return launch_wgrad_kernel<BN, SPLIT3, true, true>(P, g, tm, st);
    throw RuntimeError("internal: wgrad pair bn");
  }
  if (g.tma)
    launch_wgrad_kernel<BN, SPLIT3, true>(P, g, tm, st);
  else
    launch_wgrad_kernel<BN, SPLIT3, false>(P, g, tm, st);
}

void launch_relayout(const float* in, float* out, bool lo, int Cb, int Cb2, int64_t N, int64_t HW, cudaStream_t st) {
  const int64_t pieces = N * Cb2 * HW * 8;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid_for(pieces));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_OK(cudaLaunchKernelEx(&cfg, wgrad_relayout_kernel, in, out, lo ? out + pieces * 4 : nullptr, Cb, Cb2, HW,
                             pieces));
}

void launch_wgrad(const conv_plan* P, const float* x, const float* dy, float* dw, cudaStream_t st) {
  WgradParams g = P->wg;
  g.x = x;
  g.dy = dy;
  static const int debug_env = [] {  // profiling switch, results wrong when set
    const char* e = std::getenv("PSCONV_DEBUG");
    return e ? std::atoi(e) : 0;
  }();
  g.debug = debug_env & 3;
  const bool split3 = P->mode == PSCONV_MODE_3XTF32;
  CUtensorMap tm[4];
  std::memset(tm, 0, sizeof tm);
  if (g.tma) {
    const int64_t HW = int64_t(g.H) * g.W, PQ = int64_t(g.P) * g.Q;
    if (g.fc) {
      const int64_t pieces = int64_t(g.N) * g.Cb2 * HW * 8, n_rows = int64_t(g.N) * g.P;
      const int win = (kFoldQ - 1) * g.osw + g.oS;
      const int fold_smem = g.oR * win * ((g.fc + 3) / 4) * 16 + g.Cb2 * 32 * 4 + kFoldQ * 36 * 4;
      static SmemAttr fold_attr;
      CUDA_OK(fold_attr.ensure(wgrad_fold_kernel, 160 * 1024, P->device));
      if (fold_smem > 160 * 1024) throw RuntimeError("backward weight: tap-fold window larger than shared memory");
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(int(std::min<int64_t>(n_rows * ((g.Q + kFoldQ - 1) / kFoldQ), 148 * 16)));
      cfg.blockDim = dim3(kFoldQ);
      cfg.dynamicSmemBytes = fold_smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      CUDA_OK(cudaLaunchKernelEx(&cfg, wgrad_fold_kernel, g, x, P->wg_x32, split3 ? P->wg_x32 + pieces * 4 : nullptr,
                                 n_rows));
    } else {
      launch_relayout(x, P->wg_x32, split3, g.Cb, g.Cb2, g.N, HW, st);
    }
    launch_relayout(dy, P->wg_y32, split3, g.Kb, g.Kb2, g.N, PQ, st);
    const cuuint32_t ex[5] = {1, cuuint32_t(g.sw), cuuint32_t(g.sh), 1, 1};
    const cuuint32_t e1[5] = {1, 1, 1, 1, 1};
    {  // X32 [N][Cb2][H][W][32]: box {32, Qb*sw, Pb*sh, cn/32, 1}
      const cuuint64_t dims[5] = {32, cuuint64_t(g.W), cuuint64_t(g.H), cuuint64_t(g.Cb2), cuuint64_t(g.N)};
      const cuuint64_t strides[4] = {128, cuuint64_t(g.W) * 128, cuuint64_t(HW) * 128, cuuint64_t(g.Cb2) * HW * 128};
      const cuuint32_t box[5] = {32, cuuint32_t(g.Qb * g.sw), cuuint32_t(g.Pb * g.sh),
                                 cuuint32_t(g.cn / (g.pair ? 64 : 32)), 1};  // (pair: this CTA's half)
      encode(&tm[0], P->wg_x32, 5, dims, strides, box, ex, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
             g.sw > 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
      tm[1] = tm[0];
      if (split3)
        encode(&tm[1], P->wg_x32 + int64_t(g.N) * g.Cb2 * HW * 32, 5, dims, strides, box, ex,
               CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
               g.sw > 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    }
    {  // dY32 [N][Kb2][P][Q][32]: box {32, Qb, Pb, kn/32, 1}
      const cuuint64_t dims[5] = {32, cuuint64_t(g.Q), cuuint64_t(g.P), cuuint64_t(g.Kb2), cuuint64_t(g.N)};
      const cuuint64_t strides[4] = {128, cuuint64_t(g.Q) * 128, cuuint64_t(PQ) * 128, cuuint64_t(g.Kb2) * PQ * 128};
      const cuuint32_t box[5] = {32, cuuint32_t(g.Qb), cuuint32_t(g.Pb), cuuint32_t(g.kn / 32), 1};
      encode(&tm[2], P->wg_y32, 5, dims, strides, box, e1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
      tm[3] = tm[2];
      if (split3)
        encode(&tm[3], P->wg_y32 + int64_t(g.N) * g.Kb2 * PQ * 32, 5, dims, strides, box, e1,
               CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    }
  }
#define PSCONV_WG(B) (split3 ? launch_wgrad_bn<B, true>(P, g, tm, st) : launch_wgrad_bn<B, false>(P, g, tm, st))
  switch (g.bn) {
    case 32: PSCONV_WG(32); break;
    case 64: PSCONV_WG(64); break;
    case 128: PSCONV_WG(128); break;
    case 192: launch_wgrad_bn<192, false>(P, g, tm, st); break;
    case 256: launch_wgrad_bn<256, false>(P, g, tm, st); break;
    default: throw RuntimeError("internal: wgrad bn");
  }
#undef PSCONV_WG
  const int64_t nblk = g.fc ? int64_t(g.Kb) * g.oCb * g.oR * g.oS : int64_t(g.Kb) * g.Cb * g.R * g.S;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(int(std::min<int64_t>(nblk, 148 * 16)));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_OK(cudaLaunchKernelEx(&cfg, wgrad_reduce_kernel, g, dw));
}
}  // namespace
}  // namespace psconv

using namespace psconv;

extern "C" {

int psconv_device_sm_count(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return n;
}


int conv_plan_create(const conv_desc* d_in, int mode, int device, const char* recipe,
                     conv_plan** out) {
  return guarded([&] {
    if (!d_in || !out) throw ConfigError("null argument");
    *out = nullptr;
    conv_desc d = *d_in;
    validate_desc(d);
    *out = create_plan(d, mode, device, recipe);
  });
}

int conv_plan_create_bwd_data(const conv_desc* d_in, int mode, int device, const char* recipe,
                              conv_plan** out) {
  return guarded([&] {
    if (!d_in || !out) throw ConfigError("null argument");
    *out = nullptr;
    conv_desc f = *d_in;
    validate_desc(f);
    const int64_t sh = f.stride_h, sw = f.stride_w;
    // Output phase (a, b) of dX: h = sh*i + a reads dY rows p = i + c_a - u through the
    // forward taps r = sh*u + rho_a, rho_a = (a + pad_h) mod sh, u < U_a = ceil((kh - rho_a)
    // / sh), c_a = (a + pad_h - rho_a) / sh -- i.e. the stride-1 conv of dY with the taps
    // flipped (u' = U_a - 1 - u) and top padding U_a - 1 - c_a (the bottom padding is
    // whatever the phase needs: rows past dY are TMA zero fill). Stride 1: one phase,
    // padding kh - 1 - pad_h (the plain transposed conv).
    std::vector<conv_plan*> kids;
    std::vector<std::pair<int, int>> zeros;
    auto cleanup = [&] {
      for (conv_plan* c : kids) conv_plan_destroy(c);
    };
    try {
      for (int64_t a = 0; a < sh; ++a)
        for (int64_t b = 0; b < sw; ++b) {
          const int64_t Ha = (f.ifh - a + sh - 1) / sh, Wb = (f.ifw - b + sw - 1) / sw;
          if (Ha <= 0 || Wb <= 0) continue;
          const int64_t rh = (a + f.pad_h) % sh, rw = (b + f.pad_w) % sw;
          const int64_t U = f.kh > rh ? (f.kh - rh + sh - 1) / sh : 0;
          const int64_t V = f.kw > rw ? (f.kw - rw + sw - 1) / sw : 0;
          if (U == 0 || V == 0) {
            zeros.emplace_back(int(a), int(b));
            continue;
          }
          const int64_t ch = (a + f.pad_h - rh) / sh, cw = (b + f.pad_w - rw) / sw;
          conv_desc t{};
          t.nImg = f.nImg;
          t.nOfm = f.nIfm;
          t.nIfm = f.nOfm;
          t.ofh = Ha;
          t.ofw = Wb;
          t.kh = U;
          t.kw = V;
          t.stride_h = t.stride_w = 1;
          t.gemm_block = f.gemm_block;
          t.pad_h = U - 1 - ch;
          t.pad_w = V - 1 - cw;
          t.ifh = f.ofh;
          t.ifw = f.ofw;
          if (t.pad_h < 0 || t.pad_w < 0)
            throw ConfigError("backward data: this stride / padding combination needs a negative phase "
                              "padding (unsupported)");
          if (sh == 1 && sw == 1) validate_desc(t);  // the plain transposed conv is a valid layer
          conv_plan* c = create_plan(t, mode, device, recipe);
          kids.push_back(c);
          c->bwd_data = true;
          c->fwd = f;
          c->ph_a = int(a);
          c->ph_b = int(b);
          c->ph_rho_h = int(rh);
          c->ph_rho_w = int(rw);
          if (sh > 1 || sw > 1) {
            c->out_sh = int(sh);
            c->out_sw = int(sw);
            c->out_H = f.ifh;
            c->out_W = f.ifw;
          }
          DeviceGuard guard(device);
          const cudaError_t e = cudaMalloc(&c->wtrans, size_t(f.nOfm) * f.nIfm * U * V * sizeof(float));
          if (e != cudaSuccess) throw RuntimeError(std::string("cudaMalloc: ") + cudaGetErrorString(e));
        }
      if (sh == 1 && sw == 1) {
        *out = kids.at(0);
        return;
      }
      // strided: a parent plan holding the phases; its descriptor is the whole transposed
      // layer (dY in, dX out: the sizes conv_fwd / conv_fwd_host check and stage)
      auto* P = new conv_plan();
      P->d = f;
      P->d.nOfm = f.nIfm;
      P->d.nIfm = f.nOfm;
      P->d.ofh = f.ifh;
      P->d.ofw = f.ifw;
      P->d.ifh = f.ofh;
      P->d.ifw = f.ofw;
      P->kd = P->d;
      P->mode = mode;
      P->device = device;
      P->num_sms = kids.empty() ? 0 : kids[0]->num_sms;
      P->bwd_data = true;
      P->fwd = f;
      P->user_flt_elems = f.nOfm * f.nIfm * f.kh * f.kw;
      P->phase_plans = kids;
      P->zero_phases = zeros;
      std::string id;
      for (const conv_plan* c : kids)
        id += (id.empty() ? "" : " | ") + std::string("phase ") + std::to_string(c->ph_a) + "," +
              std::to_string(c->ph_b) + ": " + c->sched.recipe_id;
      for (const auto& z : zeros)
        id += (id.empty() ? "" : " | ") + std::string("phase ") + std::to_string(z.first) + "," +
              std::to_string(z.second) + ": zero";
      P->sched.recipe_id = id;
      *out = P;
    } catch (...) {
      cleanup();
      throw;
    }
  });
}

int conv_plan_create_bwd_weight(const conv_desc* d_in, int mode, int device, const char* recipe,
                                conv_plan** out) {
  return guarded([&] {
    if (!d_in || !out) throw ConfigError("null argument");
    *out = nullptr;
    conv_desc f = *d_in;
    validate_desc(f);
    if (f.gemm_block != 16) throw ConfigError("backward weight: gemm_block must be 16");
    if (mode == PSCONV_MODE_F16X2) throw ConfigError("backward weight: tf32 / 3xtf32 modes only");
    if (mode != PSCONV_MODE_3XTF32 && mode != PSCONV_MODE_TF32)
      throw ConfigError("unknown mode " + std::to_string(mode));
    (void)wgrad_geom(f, mode, 148, recipe);  // recipe / geometry errors before any device call
    int ndev = 0;
    CUDA_OK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw ConfigError("invalid device " + std::to_string(device));
    cudaDeviceProp prop;
    CUDA_OK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
      throw RuntimeError("psconv kernels are built for sm_100a; device is sm_" + std::to_string(prop.major) +
                         std::to_string(prop.minor));
    const WgradParams g = wgrad_geom(f, mode, prop.multiProcessorCount, recipe);
    auto* P = new conv_plan();
    P->d = f;
    P->kd = f;
    P->fwd = f;
    P->mode = mode;
    P->device = device;
    P->num_sms = prop.multiProcessorCount;
    P->bwd_weight = true;
    P->wg = g;
    P->sched.recipe_id = wgrad_recipe(g);
    DeviceGuard guard(device);
    cudaError_t e = cudaMalloc(&P->wg_ws, size_t(g.units) * 128 * g.bn * sizeof(float));
    if (e == cudaSuccess && g.tma) {
      const int copies = mode == PSCONV_MODE_3XTF32 ? 2 : 1;  // hi (raw) | lo
      e = cudaMalloc(&P->wg_x32, size_t(copies) * g.N * g.Cb2 * 32 * g.H * g.W * sizeof(float));
      if (e == cudaSuccess)
        e = cudaMalloc(&P->wg_y32, size_t(copies) * g.N * g.Kb2 * 32 * g.P * g.Q * sizeof(float));
    }
    if (e != cudaSuccess) {
      cudaFree(P->wg_ws);
      cudaFree(P->wg_x32);
      cudaFree(P->wg_y32);
      delete P;
      throw RuntimeError(std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    P->wg.ws = P->wg_ws;
    *out = P;
  });
}

int conv_wgrad_describe(const conv_desc* d_in, int mode, int num_sms, const char* recipe, char* buf, size_t len) {
  return guarded([&] {
    if (!d_in || !buf || !len) throw ConfigError("null argument");
    conv_desc f = *d_in;
    validate_desc(f);
    if (mode != PSCONV_MODE_3XTF32 && mode != PSCONV_MODE_TF32) throw ConfigError("backward weight: tf32 / 3xtf32 modes only");
    const WgradParams g = wgrad_geom(f, mode, num_sms > 0 ? num_sms : 148, recipe);
    const std::string t = wgrad_recipe(g) + " tiles:" + std::to_string(g.tiles) + " units:" +
                          std::to_string(g.units) + " stage_bytes:" + std::to_string(g.stage_bytes);
    const size_t n = std::min(t.size(), len - 1);
    std::memcpy(buf, t.data(), n);
    buf[n] = 0;
  });
}

int conv_bwd_weight(const conv_plan* P, const float* x, const float* dy, float* dw, void* stream) {
  return guarded([&] {
    if (!P || !x || !dy || !dw) throw ConfigError("null argument");
    if (!P->bwd_weight) throw ConfigError("not a backward-weight plan (conv_plan_create_bwd_weight)");
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(dw)) & 15)
      throw ConfigError("tensor pointers must be 16-byte aligned");
    DeviceGuard guard(P->device);
    launch_wgrad(P, x, dy, dw, static_cast<cudaStream_t>(stream));
  });
}

void conv_plan_destroy(conv_plan* p) {
  if (!p) return;
  for (conv_plan* c : p->phase_plans) conv_plan_destroy(c);
  if (p->pipe) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    auto* h = p->pipe;
    for (int i = 0; i < conv_plan::HostPipe::kSlots; ++i) {
      cudaFree(h->din[i]);
      cudaFree(h->dout[i]);
      cudaEventDestroy(h->h2d[i]);
      cudaEventDestroy(h->conv[i]);
      cudaEventDestroy(h->d2h[i]);
    }
    cudaFree(h->dflt);
    cudaEventDestroy(h->start);
    cudaEventDestroy(h->flt);
    cudaEventDestroy(h->end);
    if (h->sin) cudaStreamDestroy(h->sin);
    if (h->sout) cudaStreamDestroy(h->sout);
    delete h;
    cudaSetDevice(prev);
  }
  if (p->flt_pack || p->wg_ws) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    cudaFree(p->flt_pack);
    cudaFree(p->wfold);
    cudaFree(p->xfold);
    cudaFree(p->split_ctr);
    cudaFree(p->split_ws);
    cudaFree(p->absmax);
    cudaFree(p->wg_ws);
    cudaFree(p->wg_x32);
    cudaFree(p->wg_y32);
    cudaFree(p->wtrans);
    cudaSetDevice(prev);
  }
  delete p;
}

const char* conv_plan_recipe(const conv_plan* p) { return p ? p->sched.recipe_id.c_str() : ""; }

int64_t conv_plan_emit(const conv_plan* p, char* buf, size_t len) {
  int64_t need = -1;
  const int rc = guarded([&] {
    if (!p) throw ConfigError("null plan");
    if (!p->phase_plans.empty() || !p->zero_phases.empty())
      throw ConfigError("a strided backward-data plan is one transposed conv per output phase: no single driver nest");
    if (p->bwd_weight) throw ConfigError("a backward-weight plan has no forward driver nest");
    const std::string txt = emit_driver(p->d, p->sched);
    need = static_cast<int64_t>(txt.size());
    if (buf && len) {
      const size_t n = txt.size() < len - 1 ? txt.size() : len - 1;
      std::memcpy(buf, txt.data(), n);
      buf[n] = 0;
    }
  });
  return rc == PSCONV_OK ? need : -rc;
}

int conv_plan_launches(const conv_plan* p) {
  if (!p) return 0;
  if (p->bwd_weight) return 2;  // wgrad kernel + split reduction
  if (!p->phase_plans.empty() || !p->zero_phases.empty()) {
    int n = int(p->zero_phases.size());
    for (const conv_plan* c : p->phase_plans) n += conv_plan_launches(c);
    return n;
  }
  return 2 + (p->bwd_data ? 1 : 0);  // (backward data: filter transform +) filter prepack + conv
}

int conv_fwd_ex(const conv_plan* P, const float* in, const float* flt, float* out, const float* bias,
                int64_t img_begin, int64_t img_count, void* stream, unsigned flags) {
  return guarded([&] {
    if (!P) throw ConfigError("null plan");
    const bool prepacked = (flags & PSCONV_FLAG_PREPACKED) != 0;
    if (!in || !out || (!flt && !prepacked)) throw ConfigError("null tensor pointer");
    if (prepacked && !P->prepacked) throw ConfigError("PSCONV_FLAG_PREPACKED without conv_plan_prepack");
    if (prepacked) flt = in;  // unused; keeps the alignment check below simple
    if ((flags & PSCONV_FLAG_RELU) && (flags & PSCONV_FLAG_ACCUMULATE))
      throw ConfigError("PSCONV_FLAG_RELU cannot be combined with PSCONV_FLAG_ACCUMULATE");
    if (bias && (reinterpret_cast<uintptr_t>(bias) & 3)) throw ConfigError("bias must be 4-byte aligned");
    const conv_desc& d = P->d;
    if (img_begin < 0 || img_count < 0 || img_begin + img_count > d.nImg)
      throw ConfigError("image range [" + std::to_string(img_begin) + ", " +
                        std::to_string(img_begin + img_count) + ") outside nImg=" +
                        std::to_string(d.nImg));
    if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(flt) |
         reinterpret_cast<uintptr_t>(out)) & 15)
      throw ConfigError("tensor pointers must be 16-byte aligned");
    if (img_count == 0) return;
    if (P->bwd_weight) throw ConfigError("a backward-weight plan runs through conv_bwd_weight");
    DeviceGuard guard(P->device);
    const int64_t in_img = d.nIfm * d.ifh * d.ifw, out_img = d.nOfm * d.ofh * d.ofw;
    launch_range(P, in + img_begin * in_img, flt, out + img_begin * out_img, img_count,
                 static_cast<cudaStream_t>(stream), flags, bias);
  });
}

int conv_fwd(const conv_plan* P, const float* in, const float* flt, float* out, int64_t img_begin,
             int64_t img_count, void* stream, unsigned flags) {
  return conv_fwd_ex(P, in, flt, out, nullptr, img_begin, img_count, stream, flags);
}

int conv_plan_prepack(conv_plan* P, const float* flt, void* stream) {
  return guarded([&] {
    if (!P || !flt) throw ConfigError("null argument");
    if (reinterpret_cast<uintptr_t>(flt) & 15) throw ConfigError("filter must be 16-byte aligned");
    if (P->bwd_weight) throw ConfigError("a backward-weight plan has no filter to prepack");
    DeviceGuard guard(P->device);
    for (conv_plan* c : P->phase_plans) {  // strided backward data: every phase's filter
      launch_prepack(c, flt, static_cast<cudaStream_t>(stream));
      c->prepacked = true;
    }
    if (P->phase_plans.empty() && P->zero_phases.empty()) launch_prepack(P, flt, static_cast<cudaStream_t>(stream));
    P->prepacked = true;
  });
}

int conv_fwd_host(const conv_plan* P, const float* h_in, const float* h_flt, float* h_out,
                  int64_t img_begin, int64_t img_count, void* stream, unsigned flags) {
  return guarded([&] {
    if (!P) throw ConfigError("null plan");
    const bool prepacked = (flags & PSCONV_FLAG_PREPACKED) != 0;
    const bool accumulate = (flags & PSCONV_FLAG_ACCUMULATE) != 0;
    if (!h_in || !h_out || (!h_flt && !prepacked)) throw ConfigError("null tensor pointer");
    if (prepacked && !P->prepacked) throw ConfigError("PSCONV_FLAG_PREPACKED without conv_plan_prepack");
    const conv_desc& d = P->d;
    if (img_begin < 0 || img_count < 0 || img_begin + img_count > d.nImg)
      throw ConfigError("image range outside nImg");
    if (img_count == 0) return;
    if (P->bwd_weight) throw ConfigError("a backward-weight plan runs through conv_bwd_weight");
    const int64_t in_img = d.nIfm * d.ifh * d.ifw, out_img = d.nOfm * d.ofh * d.ofw;
    DeviceGuard guard(P->device);
    if (!P->pipe) {  // ~32 MB of input per chunk, kSlots buffers
      auto* h = new conv_plan::HostPipe();
      P->pipe = h;
      int64_t chunk_mb = 32;
      if (const char* e = std::getenv("PSCONV_HOST_CHUNK_MB")) chunk_mb = std::max(1, std::atoi(e));
      h->chunk = std::max<int64_t>(1, std::min<int64_t>(d.nImg, (chunk_mb << 20) / (in_img * 4)));
      for (int i = 0; i < conv_plan::HostPipe::kSlots; ++i) {
        CUDA_OK(cudaMalloc(&h->din[i], h->chunk * in_img * sizeof(float)));
        CUDA_OK(cudaMalloc(&h->dout[i], h->chunk * out_img * sizeof(float)));
        CUDA_OK(cudaEventCreateWithFlags(&h->h2d[i], cudaEventDisableTiming));
        CUDA_OK(cudaEventCreateWithFlags(&h->conv[i], cudaEventDisableTiming));
        CUDA_OK(cudaEventCreateWithFlags(&h->d2h[i], cudaEventDisableTiming));
      }
      // the caller's filter (KCRS16c16k of d): for a fold:C plan this is the unfolded
      // filter, larger than the folded operand count flt_elems
      CUDA_OK(cudaMalloc(&h->dflt, P->user_flt_elems * sizeof(float)));
      CUDA_OK(cudaEventCreateWithFlags(&h->start, cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&h->flt, cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&h->end, cudaEventDisableTiming));
      CUDA_OK(cudaStreamCreateWithFlags(&h->sin, cudaStreamNonBlocking));
      CUDA_OK(cudaStreamCreateWithFlags(&h->sout, cudaStreamNonBlocking));
    }
    auto* h = P->pipe;
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    // everything starts after the caller's prior work on `stream`
    CUDA_OK(cudaEventRecord(h->start, cs));
    CUDA_OK(cudaStreamWaitEvent(h->sin, h->start, 0));
    CUDA_OK(cudaStreamWaitEvent(h->sout, h->start, 0));
    unsigned kflags = flags;
    if (!prepacked) {
      CUDA_OK(cudaMemcpyAsync(h->dflt, h_flt, P->user_flt_elems * sizeof(float), cudaMemcpyHostToDevice, h->sin));
      CUDA_OK(cudaEventRecord(h->flt, h->sin));
      CUDA_OK(cudaStreamWaitEvent(cs, h->flt, 0));
    }
    // Chunk schedule: full chunks, with a ramp of 1/8, 1/4, 1/2 chunks at both ends
    // when there are enough images -- the first copy-in and the last copy-out are
    // the only copies not overlapped with the opposite direction (PCIe is duplex)
    std::vector<int64_t> sizes;
    {
      const int64_t c = h->chunk;
      int64_t left = img_count;
      std::vector<int64_t> ramp;
      if (img_count >= 4 * c && c >= 8) ramp = {c / 8, c / 4, c / 2};
      for (int64_t r : ramp) sizes.push_back(r), left -= r;
      std::vector<int64_t> tail(ramp.rbegin(), ramp.rend());
      for (int64_t r : tail) left -= r;
      while (left > 0) sizes.push_back(std::min(c, left)), left -= sizes.back();
      for (int64_t r : tail) sizes.push_back(r);
    }
    constexpr int kS = conv_plan::HostPipe::kSlots;
    int64_t c0 = img_begin;
    for (size_t i = 0; i < sizes.size(); ++i) {
      const int sl = int(i % kS);
      const int64_t cn = sizes[i];
      // copy in once the kernel kS chunks back has read this slot
      if (i >= kS) CUDA_OK(cudaStreamWaitEvent(h->sin, h->conv[sl], 0));
      CUDA_OK(cudaMemcpyAsync(h->din[sl], h_in + c0 * in_img, cn * in_img * sizeof(float),
                              cudaMemcpyHostToDevice, h->sin));
      if (accumulate) {  // `+=`: bring the current output chunk in as well
        if (i >= kS) CUDA_OK(cudaStreamWaitEvent(h->sin, h->d2h[sl], 0));
        CUDA_OK(cudaMemcpyAsync(h->dout[sl], h_out + c0 * out_img, cn * out_img * sizeof(float),
                                cudaMemcpyHostToDevice, h->sin));
      }
      CUDA_OK(cudaEventRecord(h->h2d[sl], h->sin));
      CUDA_OK(cudaStreamWaitEvent(cs, h->h2d[sl], 0));
      if (i >= kS && !accumulate) CUDA_OK(cudaStreamWaitEvent(cs, h->d2h[sl], 0));
      launch_range(P, h->din[sl], h->dflt, h->dout[sl], cn, cs, kflags);
      kflags |= PSCONV_FLAG_PREPACKED;  // the filter is repacked once, by the first chunk
      CUDA_OK(cudaEventRecord(h->conv[sl], cs));
      CUDA_OK(cudaStreamWaitEvent(h->sout, h->conv[sl], 0));
      CUDA_OK(cudaMemcpyAsync(h_out + c0 * out_img, h->dout[sl], cn * out_img * sizeof(float),
                              cudaMemcpyDeviceToHost, h->sout));
      CUDA_OK(cudaEventRecord(h->d2h[sl], h->sout));
      c0 += cn;
    }
    CUDA_OK(cudaEventRecord(h->end, h->sout));
    CUDA_OK(cudaStreamWaitEvent(cs, h->end, 0));
  });
}

int gemm_pack_b(const float* b, float* out, int64_t K, int64_t N, void* stream) {
  return guarded([&] {
    if (!b || !out) throw ConfigError("null argument");
    if (K <= 0 || N <= 0 || K % 16 || N % 16) throw ConfigError("gemm_pack_b: K and N must be positive multiples of 16");
    gemm_pack_b_kernel<<<grid_for(K * N), 256, 0, static_cast<cudaStream_t>(stream)>>>(b, out, K, N);
    CUDA_OK(cudaGetLastError());
  });
}

int conv_fill_input(const conv_desc* d_in, uint64_t seed, int64_t c_logical, float* in,
                    int64_t img_begin, int64_t img_count, void* stream) {
  return guarded([&] {
    if (!d_in || !in) throw ConfigError("null argument");
    conv_desc d = *d_in;
    validate_desc(d);
    if (c_logical <= 0 || c_logical > d.nIfm) c_logical = d.nIfm;
    if (img_begin < 0 || img_count < 0 || img_begin + img_count > d.nImg)
      throw ConfigError("image range outside nImg");
    const int64_t n = img_count * d.nIfm * d.ifh * d.ifw;
    if (n == 0) return;
    fill_input_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        in + img_begin * d.nIfm * d.ifh * d.ifw, seed, n, img_begin, int(d.nIfm / 16),
        int(d.ifh), int(d.ifw), int(c_logical));
    CUDA_OK(cudaGetLastError());
  });
}

int conv_fill_filter(const conv_desc* d_in, uint64_t seed, int64_t c_logical, float* flt,
                     void* stream) {
  return guarded([&] {
    if (!d_in || !flt) throw ConfigError("null argument");
    conv_desc d = *d_in;
    validate_desc(d);
    if (c_logical <= 0 || c_logical > d.nIfm) c_logical = d.nIfm;
    const int64_t n = d.nOfm * d.nIfm * d.kh * d.kw;
    fill_filter_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        flt, seed, n, int(d.nIfm / 16), int(d.kh), int(d.kw), int(c_logical));
    CUDA_OK(cudaGetLastError());
  });
}

int conv_pack_input(const conv_desc* d_in, const float* nchw, int64_t c_logical, float* out,
                    void* stream) {
  return guarded([&] {
    if (!d_in || !nchw || !out) throw ConfigError("null argument");
    conv_desc d = *d_in;
    validate_desc(d);
    if (c_logical <= 0 || c_logical > d.nIfm) c_logical = d.nIfm;
    const int64_t n = d.nImg * d.nIfm * d.ifh * d.ifw;
    pack_input_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        nchw, out, n, int(d.nIfm / 16), int(d.ifh), int(d.ifw), int(c_logical));
    CUDA_OK(cudaGetLastError());
  });
}

int conv_pack_filter(const conv_desc* d_in, const float* kcrs, int64_t c_logical, float* out,
                     void* stream) {
  return guarded([&] {
    if (!d_in || !kcrs || !out) throw ConfigError("null argument");
    conv_desc d = *d_in;
    validate_desc(d);
    if (c_logical <= 0 || c_logical > d.nIfm) c_logical = d.nIfm;
    const int64_t n = d.nOfm * d.nIfm * d.kh * d.kw;
    pack_filter_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        kcrs, out, n, int(d.nIfm / 16), int(d.kh), int(d.kw), int(c_logical));
    CUDA_OK(cudaGetLastError());
  });
}

int conv_unpack_output(const conv_desc* d_in, const float* nkpq16k, float* nkpq, void* stream) {
  return guarded([&] {
    if (!d_in || !nkpq16k || !nkpq) throw ConfigError("null argument");
    conv_desc d = *d_in;
    validate_desc(d);
    const int64_t n = d.nImg * d.nOfm * d.ofh * d.ofw;
    unpack_output_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        nkpq16k, nkpq, n, int(d.nOfm / 16), int(d.ofh * d.ofw));
    CUDA_OK(cudaGetLastError());
  });
}

}  // extern "C"
