// Backward-weight kernel: pixel-major implicit GEMM on tcgen05 with
// MN-major tf32 operands gathered straight from the activation layouts.
//
//   dW[k][c][r][s] = sum_{n,p,q} dY[n][k][p][q] * X[n][c][p*sh + r - ph][q*sw + s - pw]
//
// For every tap (r, s) this is a GEMM over the pixels (n, p, q): the reduction index is the
// pixel, so both operands are "MN-major" -- one pixel = one reduction row of 32 channels
// (two 16-channel blocks of NCHW16c / NKPQ16k side by side, 128 B). kind::tf32 accepts
// MN-major operands only in the SWIZZLE_128B_BASE32B smem layout (4-row atoms of 128-B
// rows, 32-B chunks XOR-ed with the row; tools/probe_mn.cu). TMA cannot build it from 64-B
// channel blocks: a box whose inner dimension (64 B) is narrower than the 128-B swizzle
// span is stored one inner row per 128-B smem row, half empty, and a second box cannot start
// 64 B in (misaligned; tools/probe_tma_sw32.cu). So producer warps gather the operands
// with 16-byte cp.async copies, each placed at its swizzled position (out-of-image pixels and
// channels past C / K: zero fill through src-size 0), one cp.async group per stage; a
// producer thread signals a stage after its own copies of it completed (wait_group) and a
// proxy fence -- the MMAs read it through the async proxy.
//
// Stage = a Qb x Pb pixel box of one image: rows = Qb * Pb reduction rows (multiple of 8).
//   X side:  ntap taps x cn channels = ntap * cn / 32 MN groups (tap-shifted windows)
//   dY side: kn channels = kn / 32 MN groups
// Every MN group is `rows` 128-B rows (LBO = rows * 128 B, SBO = 512 B: 4-row atoms).
//
// Tile = 128 (M) x bn (N) accumulator in TMEM:
//   swap 0: M = 128 output channels k (dY), N = ntap taps x cn input channels (X)
//   swap 1: M = ntap x cn = 128 (X: taps x input channels), N = kn output channels (dY)
//           (layers with K < 128, e.g. ResNet-50's K = 64 convs)
// Work unit = (pixel split, tile); units are split-major so the CTAs running at one time
// share a pixel range (its X / dY slice is read from HBM once, the other tiles hit L2).
// Each unit writes its 128 x bn partial to a workspace; wgrad_reduce_kernel adds the splits
// in split order (bitwise reproducible) and scatters into KCRS16c16k.
//
// Warp roles: 0-3 epilogue (TMEM lane quadrant = warp; TMEM -> registers -> workspace),
// 4 TMEM owner + MMA issuer, 5.. producers (kWgProdWarps). 3xTF32: the producers also write lo = x -
// trunc_tf32(x) of every chunk they copied into the stage's lo half; the MMAs D += A_hi B_hi
// + A_lo B_hi + A_hi B_lo (kind::tf32 truncates fp32 operands, so A_hi / B_hi are the raw
// tiles), accumulated in chunks of `chunk_k8` K=8 steps (the TMEM accumulation error grows
// with the chain length) that the epilogue sums in fp32 registers;
// double-buffered accumulators keep the MMA busy meanwhile.
#pragma once
#include <cuda.h>
#include <cstdint>

#include "sm100_ptx.cuh"

namespace psconv {

constexpr int kWgMaxStages = 8;
constexpr int kWgProdWarps = 8;  // producer warps (cp.async gatherers)

struct WgradParams {
  int N, Cb, Kb, H, W, P, Q, R, S, sh, sw, ph, pw;
  int swap;                         // see above
  int kn, cn, ntap, bn;             // channels / taps per tile, MMA N
  int tiles_k, tiles_c, tiles_t, tiles;
  int Qb, Pb, rows;                 // pixel box per stage (rows = Qb * Pb, multiple of 8)
  int tiles_q, tiles_p;             // boxes per image
  int nstage;                       // N * tiles_p * tiles_q pixel stages
  int splits, units, stage_per_split;
  int stages;                       // ring depth
  int x_bytes, y_bytes;             // per stage (hi), X region first
  int stage_bytes;                  // x + y (x2 for 3xTF32: hi | lo)
  int chunk_k8;                     // 3xTF32: K=8 steps per accumulation chunk (0: whole unit)
  int debug;                        // profiling (PSCONV_DEBUG): 1 skip copies, 2 skip MMAs
  int tma;                          // 1: TMA path over the relaid X / dY (else cp.async gather)
  int pair;                         // TMA path, sw 0, one tap: CTA pairs (cta_group::2, M = 256): the
                                    // two CTAs hold the output channels 2kp*128.. / (2kp+1)*128.. and
                                    // one half each of the input channels (cn / 2); tile index
                                    // ((kp * tiles_t + tt) * tiles_c + ct) * 2 + (kt & 1)
  // tap fold (recipe pp:C, few-channel layers such as the ResNet stem): the kernel runs the
  // 1x1 wgrad of X' = the layer's (tap, channel) window per output pixel (fc real channels per
  // tap, R*S*fc folded channels padded to 32) against dY; o* is the original layer
  int fc, oCb, oR, oS, oH, oW, osh, osw, oph, opw;
  int Cb2, Kb2;                     // TMA path: 32-channel blocks of the relaid X / dY
  const float* x;                   // NCHW16c forward input
  const float* dy;                  // NKPQ16k output gradient
  float* ws;                        // partials [unit][128][bn]
};

namespace ptx {
// MN-major SWIZZLE_128B_BASE32B descriptor (layout type 1): lbo = MN-group pitch, sbo = the
// pitch of 4-row reduction atoms (512 B when contiguous)
__device__ __forceinline__ uint64_t smem_desc_mn32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (1ull << 61);
}
template <int BN, int M = 128>
__host__ __device__ constexpr uint32_t idesc_tf32_mn() {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | (static_cast<uint32_t>(BN >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
// 16-byte global -> shared copy; src_bytes = 0 zero-fills the destination
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
}  // namespace ptx

template <int BN, bool SPLIT3, bool TMA = false, bool PAIR = false>
struct WgCfg {
  // 4 epilogue + 1 MMA + producer warps (the TMA path: one producer warp)
  static constexpr int kThreads = 32 * (5 + (TMA ? 1 : kWgProdWarps));
  static constexpr int kAccCols = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  static constexpr uint32_t kTmemCols = 2 * kAccCols;  // two accumulators (power of 2, >= 64)
};

__device__ __forceinline__ void wg_tile_coords(const WgradParams& p, int tile, int& kt, int& tt, int& ct) {
  int rest = tile, bit = 0;
  if (p.pair) {
    bit = tile & 1;
    rest = tile >> 1;
  }
  ct = rest % p.tiles_c;
  tt = (rest / p.tiles_c) % p.tiles_t;
  kt = rest / (p.tiles_c * p.tiles_t);
  if (p.pair) kt = 2 * kt + bit;
}
__host__ __device__ __forceinline__ int wg_tile_index(const WgradParams& p, int kt, int tt, int ct) {
  return p.pair ? (((kt >> 1) * p.tiles_t + tt) * p.tiles_c + ct) * 2 + (kt & 1) : (kt * p.tiles_t + tt) * p.tiles_c + ct;
}

__device__ __forceinline__ void wg_stage_coords(const WgradParams& p, int g, int& n, int& p0, int& q0) {
  const int per_img = p.tiles_p * p.tiles_q;
  n = g / per_img;
  const int r = g - n * per_img;
  p0 = (r / p.tiles_q) * p.Pb;
  q0 = (r % p.tiles_q) * p.Qb;
}

// The producer thread's share of one stage: its chunk column k8 (half = k8 / 4 selects the
// 16-channel block of the 32-channel group, c16 = k8 % 4 the 16-B piece of it) of rows
// row0 + kRowStep * m, in every MN group of the stage. The per-row pixel offsets live in a
// shared-memory table (built once per CTA), the per-tap shifts in another (per unit); per
// (row, tap) one bounds test and one pointer, then a pointer step + cp.async per block pair.
// Compact loops on purpose: an unrolled version stalled on instruction fetch (ncu: BSYNC
// no_instruction) and ran at ~0.16 IPC per producer warp.
struct WgRowTab {
  int xoff;  // X: (pi * sh * W + qi * sw) * 16 floats from the box origin
  int xhw;   // X: (pi * sh) << 16 | qi * sw
  int yoff;  // dY: (pi * Q + qi) * 16
  int ypq;   // dY: pi << 16 | qi
};
struct WgTapTab {
  int off;  // (r * W + s) * 16 floats
  int rs;   // r << 16 | s
};

template <int PW>
struct WgProducer {
  static constexpr int kRowStep = PW * 4;  // 8 chunk columns per 128-B row
  int k8, row0;
  uint32_t doff0;  // byte offset of the chunk inside its MN group at m = 0 (row & 3 is the
                   // same for every m: the row step is a multiple of 4, one swizzle phase)

  __device__ __forceinline__ void init(int tid) {
    k8 = tid & 7;
    row0 = tid >> 3;
    const int chunk32 = (k8 >> 1) ^ (row0 & 3);  // logical 32-B chunk (half*2 + c16/2), swizzled
    doff0 = static_cast<uint32_t>(row0 * 128 + chunk32 * 32 + (k8 & 1) * 16);
  }

  // issue the stage's copies into the slot at shared address `sb`
  __device__ __forceinline__ void issue(const WgradParams& p, const WgRowTab* rows, const WgTapTab* taps, uint32_t sb,
                                        int n, int p0, int q0, int kt, int ct) const {
    const uint32_t grp = static_cast<uint32_t>(p.rows) * 128u;
    const int half = k8 >> 2, c16 = k8 & 3;
    const int npx = p.cn / 32, npy = p.kn / 32;
    // block pairs j whose block (first + 2 j) exists; past C / K: zeros
    const int cb0 = ct * (p.cn / 16) + half, kb0 = kt * (p.kn / 16) + half;
    const int jx = max(0, min(npx, (p.Cb - cb0 + 1) / 2)), jy = max(0, min(npy, (p.Kb - kb0 + 1) / 2));
    const int64_t xpair = static_cast<int64_t>(2) * p.H * p.W * 16;  // floats between block pairs
    const int64_t ypair = static_cast<int64_t>(2) * p.P * p.Q * 16;
    const int hb = p0 * p.sh - p.ph, wb = q0 * p.sw - p.pw;  // input origin of the box (tap 0, 0)
    const float* xs = p.x + ((static_cast<int64_t>(n) * p.Cb + cb0) * p.H + hb) * p.W * 16 + wb * 16 + c16 * 4;
    const float* ys = p.dy + ((static_cast<int64_t>(n) * p.Kb + kb0) * p.P + p0) * p.Q * 16 + q0 * 16 + c16 * 4;
    const int pmax = p.P - p0, qmax = p.Q - q0;
    const uint32_t ybase = sb + static_cast<uint32_t>(p.x_bytes);
#pragma unroll 1
    for (int row = row0, m = 0; row < p.rows; row += kRowStep, ++m) {
      const WgRowTab rt = rows[row];
      const uint32_t dm = doff0 + static_cast<uint32_t>(m * kRowStep * 128);
      const int hr = hb + (rt.xhw >> 16), wr = wb + (rt.xhw & 0xFFFF);
#pragma unroll 1
      for (int t = 0; t < p.ntap; ++t) {
        const WgTapTab tp = taps[t];
        const int h = hr + (tp.rs >> 16), w = wr + (tp.rs & 0xFFFF);
        const bool ok = static_cast<unsigned>(h) < static_cast<unsigned>(p.H) &&
                        static_cast<unsigned>(w) < static_cast<unsigned>(p.W);
        const float* src = ok ? xs + (rt.xoff + tp.off) : p.x;
        const int64_t step = ok ? xpair : 0;
        const uint32_t d = sb + static_cast<uint32_t>(t * npx) * grp + dm;
        // independent addresses per copy: a running pointer made every copy wait for the
        // previous cp.async to read its operands (ncu: long scoreboard on the increment)
#pragma unroll 4
        for (int j = 0; j < npx; ++j)
          ptx::cp_async16(d + j * grp, src + j * step, (ok && j < jx) ? 16u : 0u);
      }
      const bool ok = (rt.ypq >> 16) < pmax && (rt.ypq & 0xFFFF) < qmax;
      const float* src = ok ? ys + rt.yoff : p.dy;
      const int64_t step = ok ? ypair : 0;
      const uint32_t d = ybase + dm;
#pragma unroll 4
      for (int j = 0; j < npy; ++j) ptx::cp_async16(d + j * grp, src + j * step, (ok && j < jy) ? 16u : 0u);
    }
  }

  // 3xTF32: lo = x - trunc_tf32(x) of this thread's chunks of the (landed) stage
  __device__ __forceinline__ void split(const WgradParams& p, uint8_t* slot) const {
    const uint32_t grp = static_cast<uint32_t>(p.rows) * 128u;
    const int groups = p.ntap * (p.cn / 32) + p.kn / 32;
    const uint32_t lo = static_cast<uint32_t>(p.x_bytes + p.y_bytes);
#pragma unroll 1
    for (int row = row0, m = 0; row < p.rows; row += kRowStep, ++m) {
      uint32_t o = doff0 + static_cast<uint32_t>(m * kRowStep * 128);
#pragma unroll 2
      for (int g = 0; g < groups; ++g, o += grp) {
        const float4 v = *reinterpret_cast<const float4*>(slot + o);
        float4 l;
        l.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
        l.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
        l.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
        l.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
        *reinterpret_cast<float4*>(slot + lo + o) = l;
      }
    }
  }
};

// TMA path (recipe tma:1): X and dY relaid once per call into 32-channel blocks
// ([N][C/32][H][W][32], wgrad_relayout_kernel; 3xTF32: + the lo halves), so one pixel's 32
// channels are 128 contiguous bytes -- a TMA box with a 128-B inner dimension lands dense in the
// SWIZZLE_128B_ATOM_32B layout, one box per tap (X) / per stage (dY), multicast-free, ~2x the
// L2->SM rate of the cp.async gather.
template <int BN, bool SPLIT3, bool TMA = false, bool PAIR = false>
__global__ void __launch_bounds__(WgCfg<BN, SPLIT3, TMA, PAIR>::kThreads, 1)
    wgrad_sm100(const __grid_constant__ WgradParams p, const __grid_constant__ CUtensorMap tm_x,
                const __grid_constant__ CUtensorMap tm_xlo, const __grid_constant__ CUtensorMap tm_y,
                const __grid_constant__ CUtensorMap tm_ylo) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  using Cfg = WgCfg<BN, SPLIT3, TMA, PAIR>;
  static_assert(!PAIR || TMA, "CTA pairs run on the TMA path");
  constexpr uint32_t kIdesc = ptx::idesc_tf32_mn<BN, PAIR ? 256 : 128>();
  constexpr int CS = PAIR ? 2 : 1;
  const int rank = PAIR ? static_cast<int>(blockIdx.x & 1) : 0;
  const bool leader = rank == 0;
  // PAIR: the cluster takes CTA-level units 2 uc and 2 uc + 1 (the two output-channel halves
  // of one pair tile, same pixel range)
  const int ustart = PAIR ? static_cast<int>(blockIdx.x >> 1) * 2 + rank : static_cast<int>(blockIdx.x);
  const int ustep = static_cast<int>(gridDim.x);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int kStages = p.stages;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * p.stage_bytes);
  uint64_t* full = bars;                     // stage landed (+ split): every producer thread
  uint64_t* empty = bars + kWgMaxStages;     // MMAs done with the slot
  uint64_t* acc_full = bars + 2 * kWgMaxStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  // per-row pixel offsets of the box (256 max) and the unit's tap shifts (9 max x 2 buffers)
  WgRowTab* rowtab = reinterpret_cast<WgRowTab*>(smem + kStages * p.stage_bytes + 256);
  WgTapTab* taptab = reinterpret_cast<WgTapTab*>(rowtab + 256);
  const int warp = threadIdx.x >> 5;
  for (int row = threadIdx.x; row < p.rows; row += blockDim.x) {
    const int pi = row / p.Qb, qi = row - (row / p.Qb) * p.Qb;
    WgRowTab t;
    t.xoff = (pi * p.sh * p.W + qi * p.sw) * 16;
    t.xhw = ((pi * p.sh) << 16) | (qi * p.sw);
    t.yoff = (pi * p.Q + qi) * 16;
    t.ypq = (pi << 16) | qi;
    rowtab[row] = t;
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], TMA ? 1 : 32 * kWgProdWarps);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&acc_full[a], 1);
      ptx::mbar_init(&acc_empty[a], 4 * CS);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 4) {
    if (PAIR)
      ptx::tmem_alloc_pair(tmem_slot, Cfg::kTmemCols);
    else
      ptx::tmem_alloc(tmem_slot, Cfg::kTmemCols);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (PAIR) ptx::cluster_sync_all();  // both CTAs' barriers initialised, TMEM allocated
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ptx::griddep_launch_dependents();

  const int per_split = p.stage_per_split;
  // chunks per unit: 3xTF32 splits the reduction into accumulation chunks of chunk_k8 K=8
  // steps (whole stages); TF32 accumulates the unit in one chunk
  const int k8_stage = p.rows / 8;
  const int chunk_st = (SPLIT3 && p.chunk_k8 > 0) ? max(1, p.chunk_k8 / k8_stage) : (1 << 30);

  if (TMA && warp == 5) {
    // ------------------------------------------------------------ producer (TMA)
    if (ptx::elect_one()) {
      ptx::prefetch_tmap(&tm_x);
      ptx::prefetch_tmap(&tm_y);
    }
    ptx::griddep_wait();
    __syncwarp();
    const uint32_t tx = static_cast<uint32_t>(p.x_bytes + p.y_bytes) * (SPLIT3 ? 2u : 1u) * CS;
    const uint32_t lo = static_cast<uint32_t>(p.x_bytes + p.y_bytes);
    const uint32_t tap_bytes = static_cast<uint32_t>(p.cn / CS) * p.rows * 4;
    // PAIR: both CTAs' boxes complete on the LEADER's full barrier (it expects both shares)
    const uint32_t full_leader = PAIR ? ptx::mapa(&full[0], 0) : 0u;
    int stage = 0;
    uint32_t phase = 0;
    for (int u = ustart; u < p.units; u += ustep) {
      const int split = u / p.tiles;
      int kt, tt, ct;
      wg_tile_coords(p, u - split * p.tiles, kt, tt, ct);
      const int g0 = split * per_split, g1 = min(p.nstage, g0 + per_split);
      const int xcb = ct * (p.cn / 32) + rank * (p.cn / 64);  // this CTA's input-channel groups
      for (int g = g0; g < g1; ++g) {
        int n, p0, q0;
        wg_stage_coords(p, g, n, p0, q0);
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        if (p.debug & 1) {  // profiling: no loads, the stage is "full" at once
          if (leader && ptx::elect_one()) ptx::mbar_arrive(&full[stage]);
        } else if (ptx::elect_one()) {
          uint8_t* sb = smem + stage * p.stage_bytes;
          if (leader) ptx::mbar_expect_tx(&full[stage], tx);
          const uint32_t fb = full_leader + 8u * stage;
          for (int t = 0; t < p.ntap; ++t) {
            // taps past R*S (a partial last tap group) load the last tap again; the reduce
            // kernel never reads those accumulator rows / columns
            const int tap = min(tt * p.ntap + t, p.R * p.S - 1);
            const int r = tap / p.S, sx = tap - r * p.S;
            const int wq = q0 * p.sw + sx - p.pw, hp = p0 * p.sh + r - p.ph;
            if (PAIR) {
              ptx::tma_load_5d_cb(sb + t * tap_bytes, &tm_x, fb, 0, wq, hp, xcb, n);
              if (SPLIT3) ptx::tma_load_5d_cb(sb + lo + t * tap_bytes, &tm_xlo, fb, 0, wq, hp, xcb, n);
            } else {
              ptx::tma_load_5d(sb + t * tap_bytes, &tm_x, &full[stage], 0, wq, hp, xcb, n);
              if (SPLIT3) ptx::tma_load_5d(sb + lo + t * tap_bytes, &tm_xlo, &full[stage], 0, wq, hp, xcb, n);
            }
          }
          if (PAIR) {
            ptx::tma_load_5d_cb(sb + p.x_bytes, &tm_y, fb, 0, q0, p0, kt * (p.kn / 32), n);
            if (SPLIT3) ptx::tma_load_5d_cb(sb + lo + p.x_bytes, &tm_ylo, fb, 0, q0, p0, kt * (p.kn / 32), n);
          } else {
            ptx::tma_load_5d(sb + p.x_bytes, &tm_y, &full[stage], 0, q0, p0, kt * (p.kn / 32), n);
            if (SPLIT3) ptx::tma_load_5d(sb + lo + p.x_bytes, &tm_ylo, &full[stage], 0, q0, p0, kt * (p.kn / 32), n);
          }
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (!TMA && warp >= 5) {
    // ------------------------------------------------------------ producers (cp.async)
    WgProducer<kWgProdWarps> pr;
    pr.init(threadIdx.x - 160);
    int tt_cur = -1, tbuf = 0;
    ptx::griddep_wait();  // X / dY come from earlier kernels in the stream (PDL)
    const uint32_t s0 = ptx::smem_u32(smem);
    // a stage is signalled once `lag` younger stages are in flight (cp.async groups)
    const int lag = kStages > 3 ? 3 : kStages - 1;
    int stage = 0, pending = 0, sig_stage = 0;
    uint32_t phase = 0;
    auto signal_oldest = [&]() {
      if (SPLIT3) pr.split(p, smem + sig_stage * p.stage_bytes);
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(&full[sig_stage]);
      if (++sig_stage == kStages) sig_stage = 0;
    };
    for (int u = ustart; u < p.units; u += ustep) {
      const int split = u / p.tiles;
      int kt, tt, ct;
      wg_tile_coords(p, u - split * p.tiles, kt, tt, ct);
      const int g0 = split * per_split, g1 = min(p.nstage, g0 + per_split);
      if (tt != tt_cur) {  // the unit's taps (double-buffered: the other warps may still read)
        tt_cur = tt;
        tbuf ^= 1;
        const int i = threadIdx.x - 160;
        if (i < p.ntap) {
          // taps past R*S (a partial last tap group) copy the last tap again; the reduce
          // kernel never reads those accumulator rows / columns
          const int tap = min(tt * p.ntap + i, p.R * p.S - 1);
          const int r = tap / p.S, sx = tap - r * p.S;
          WgTapTab tp;
          tp.off = (r * p.W + sx) * 16;
          tp.rs = (r << 16) | sx;
          taptab[tbuf * 16 + i] = tp;
        }
        ptx::named_bar(1, 32 * kWgProdWarps);
      }
      for (int g = g0; g < g1; ++g) {
        int n, p0, q0;
        wg_stage_coords(p, g, n, p0, q0);
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        if (!(p.debug & 1))
          pr.issue(p, rowtab, taptab + tbuf * 16, s0 + static_cast<uint32_t>(stage * p.stage_bytes), n, p0, q0, kt,
                   ct);
        ptx::cp_async_commit();
        if (++pending > lag) {
          if (lag == 3)
            ptx::cp_async_wait<3>();
          else if (lag == 2)
            ptx::cp_async_wait<2>();
          else
            ptx::cp_async_wait<1>();
          signal_oldest();
          --pending;
        }
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    ptx::cp_async_wait<0>();
    while (pending-- > 0) signal_oldest();
  } else if (warp == 4 && leader) {
    // ------------------------------------------------------------ MMA issuer (PAIR: the leader
    // issues M = 256 MMAs over both CTAs' A rows and B halves)
    const uint32_t lbo = static_cast<uint32_t>(p.rows) * 128u;
    const uint32_t s0 = ptx::smem_u32(smem);
    const uint32_t a_off = p.swap ? 0u : static_cast<uint32_t>(p.x_bytes);
    const uint32_t b_off = p.swap ? static_cast<uint32_t>(p.x_bytes) : 0u;
    const uint32_t lo_off = static_cast<uint32_t>(p.x_bytes + p.y_bytes);
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int u = ustart; u < p.units; u += ustep) {
      const int split = u / p.tiles;
      const int g0 = split * per_split, g1 = min(p.nstage, g0 + per_split);
      int in_chunk = 0;
      for (int g = g0; g < g1; ++g) {
        if (in_chunk == 0) {  // a fresh accumulator (chunk) begins (PAIR: both CTAs drained it)
          if (PAIR)
            ptx::mbar_wait_cluster(&acc_empty[acc], acc_phase ^ 1);
          else
            ptx::mbar_wait(&acc_empty[acc], acc_phase ^ 1);
          ptx::tc_fence_after();
        }
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const bool first = in_chunk == 0;
        const bool last = ++in_chunk == chunk_st || g + 1 == g1;
        if (ptx::elect_one()) {
          const uint32_t base = s0 + static_cast<uint32_t>(stage * p.stage_bytes);
          const uint32_t d = tmem_base + static_cast<uint32_t>(acc * Cfg::kAccCols);
          const int nk8 = (p.debug & 2) ? 0 : k8_stage;
          // descriptors built once per stage; a K=8 step is +1024 B = +64 in the 16-B address
          // field (no carry out of it: smem offsets < 256 KB)
          uint64_t ad = ptx::smem_desc_mn32(base + a_off, lbo, 512), bd = ptx::smem_desc_mn32(base + b_off, lbo, 512);
          const uint64_t lo16 = lo_off >> 4;
          uint32_t accum = first ? 0u : 1u;
          for (int j = 0; j < nk8; ++j, ad += 64, bd += 64) {
            if (PAIR) {
              ptx::mma_tf32_pair(d, ad, bd, kIdesc, accum);
              if (SPLIT3) {
                ptx::mma_tf32_pair(d, ad + lo16, bd, kIdesc, 1u);
                ptx::mma_tf32_pair(d, ad, bd + lo16, kIdesc, 1u);
              }
            } else {
              ptx::mma_tf32(d, ad, bd, kIdesc, accum);
              if (SPLIT3) {
                ptx::mma_tf32(d, ad + lo16, bd, kIdesc, 1u);
                ptx::mma_tf32(d, ad, bd + lo16, kIdesc, 1u);
              }
            }
            accum = 1u;
          }
          if (PAIR) {
            ptx::mma_commit_pair(&empty[stage]);
            if (last) ptx::mma_commit_pair(&acc_full[acc]);
          } else {
            ptx::mma_commit(&empty[stage]);
            if (last) ptx::mma_commit(&acc_full[acc]);
          }
        }
        __syncwarp();
        if (last) {
          in_chunk = 0;
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------ epilogue (warps 0-3)
    const int row = warp * 32 + (threadIdx.x & 31);
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(warp * 32) << 16);
    // accumulator drained: PAIR's second CTA arrives on the leader's barrier
    const uint32_t acc_empty_leader = PAIR ? ptx::mapa(&acc_empty[0], 0) : 0u;
    auto release = [&](int a) {
      ptx::tc_fence_before();
      __syncwarp();
      if (ptx::elect_one()) {  // one arrival per warp
        if (PAIR && !leader)
          ptx::mbar_arrive_remote(acc_empty_leader + 8u * a);
        else
          ptx::mbar_arrive(&acc_empty[a]);
      }
      __syncwarp();
    };
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = ustart; u < p.units; u += ustep) {
      const int split = u / p.tiles;
      const int g0 = split * per_split, g1 = min(p.nstage, g0 + per_split);
      float* dst = p.ws + (static_cast<int64_t>(u) * 128 + row) * p.bn;
      if constexpr (SPLIT3 && BN <= 128) {
        const int nchunks = (g1 - g0 + chunk_st - 1) / chunk_st;
        float sum[BN];
#pragma unroll
        for (int i = 0; i < BN; ++i) sum[i] = 0.f;
        for (int c = 0; c < nchunks; ++c) {
          ptx::mbar_wait_sleep(&acc_full[acc], acc_phase);
          ptx::tc_fence_after();
#pragma unroll
          for (int c0 = 0; c0 < BN; c0 += 32) {
            uint32_t v[32];
            ptx::tmem_ld32(lane_base + acc * Cfg::kAccCols + c0, v);
            ptx::tmem_wait_ld();
            ptx::reg_fence(v);
#pragma unroll
            for (int i = 0; i < 32; ++i) sum[c0 + i] += __uint_as_float(v[i]);
          }
          release(acc);
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 4)
          *reinterpret_cast<float4*>(dst + c0) = make_float4(sum[c0], sum[c0 + 1], sum[c0 + 2], sum[c0 + 3]);
      } else {
        // one chunk per unit (TF32): stream the accumulator to the workspace in 32-column pieces
        ptx::mbar_wait_sleep(&acc_full[acc], acc_phase);
        ptx::tc_fence_after();
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t v[32];
          ptx::tmem_ld32(lane_base + acc * Cfg::kAccCols + c0, v);
          ptx::tmem_wait_ld();
          ptx::reg_fence(v);
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(dst + c0 + i) =
                make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                            __uint_as_float(v[i + 3]));
        }
        release(acc);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (PAIR) ptx::cluster_sync_all();  // no CTA leaves while the pair still uses it
  if (warp == 4) {
    ptx::tc_fence_after();
    if (PAIR)
      ptx::tmem_dealloc_pair(tmem_base, Cfg::kTmemCols);
    else
      ptx::tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
#endif
}

// TMA path: NCHW16c (or NKPQ16k) -> [N][C/32][H][W][32] (an odd last block's partner is
// zero); lo != nullptr also writes lo = x - trunc_tf32(x) in the same layout. One thread per
// 16-B piece of the output.
__global__ void wgrad_relayout_kernel(const float* __restrict__ in, float* __restrict__ out, float* __restrict__ lo,
                                      int Cb, int Cb2, int64_t HW, int64_t n_pieces) {
  ptx::griddep_wait();
  ptx::griddep_launch_dependents();
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n_pieces; e += int64_t(gridDim.x) * blockDim.x) {
    const int j = int(e & 7);  // 16-B piece of the 128-B pixel row
    const int64_t t = e >> 3;  // (n, cb2, pixel)
    const int64_t px = t % HW;
    const int64_t nc = t / HW;
    const int cb2 = int(nc % Cb2);
    const int64_t n = nc / Cb2;
    const int cb = 2 * cb2 + (j >> 2);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (cb < Cb) v = __ldg(reinterpret_cast<const float4*>(in + ((n * Cb + cb) * HW + px) * 16) + (j & 3));
    reinterpret_cast<float4*>(out)[e] = v;
    if (lo) {
      float4 l;
      l.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
      l.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
      l.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
      l.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
      reinterpret_cast<float4*>(lo)[e] = l;
    }
  }
}

// Tap fold (recipe pp:C): out[n][cb2][p][q][32] holds folded channel c' = cb2 * 32 + j =
// (r * S + s) * C + c of output pixel (p, q): X[n][c][p*sh + r - ph][q*sw + s - pw] (0 outside
// the image and for c' >= R*S*C); lo != nullptr also writes the 3xTF32 lo halves. A block folds
// kFoldQ output pixels of one output row: it stages the R input rows of its window (the first
// ceil(C/4) 16-B pieces of each pixel, zero outside the image) in shared memory with coalesced
// loads, then every thread assembles its pixel's folded 16-B pieces from there. (Earlier
// versions gathered straight from global memory: 2.1-2.4 ms on the ResNet stem at N = 256,
// re-reading X 4.5x from DRAM or starved of warps by a per-thread row buffer.)
constexpr int kFoldQ = 64;
__global__ void __launch_bounds__(kFoldQ) wgrad_fold_kernel(const __grid_constant__ WgradParams g,
                                                            const float* __restrict__ in, float* __restrict__ out,
                                                            float* __restrict__ lo, int64_t n_rows) {
  extern __shared__ float4 ftile[];  // [R][win][c4s], then the folded-channel offset table
  ptx::griddep_wait();
  ptx::griddep_launch_dependents();
  const int c4s = (g.fc + 3) / 4;  // 16-B pieces per pixel holding the real channels
  const int win = (kFoldQ - 1) * g.osw + g.oS;
  const int T = g.oR * g.oS * g.fc;
  // folded channel -> float offset in the tile relative to the thread's first window pixel
  // (-1: a padding channel), computed once per block (no divisions in the gather loop)
  int* ctab = reinterpret_cast<int*>(ftile + g.oR * win * c4s);
  for (int cf = threadIdx.x; cf < g.Cb2 * 32; cf += kFoldQ) {
    int o = -1;
    if (cf < T) {
      const int t = cf / g.fc, c = cf - t * g.fc;
      const int r = t / g.oS, sx = t - r * g.oS;
      o = (r * win + sx) * c4s * 4 + c;
    }
    ctab[cf] = o;
  }
  const int64_t PQ = int64_t(g.P) * g.Q;
  const int qtiles = (g.Q + kFoldQ - 1) / kFoldQ;
  for (int64_t b = blockIdx.x; b < n_rows * qtiles; b += gridDim.x) {
    const int qt = int(b % qtiles);
    const int64_t np = b / qtiles;
    const int pp = int(np % g.P);
    const int64_t n = np / g.P;
    const int q0 = qt * kFoldQ;
    const int w0 = q0 * g.osw - g.opw, h0 = pp * g.osh - g.oph;
    __syncthreads();
    for (int i = threadIdx.x; i < g.oR * win * c4s; i += kFoldQ) {
      const int c4 = i % c4s, wi = (i / c4s) % win, r = i / (c4s * win);
      const int h = h0 + r, w = w0 + wi;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (h >= 0 && h < g.oH && w >= 0 && w < g.oW)
        v = __ldg(reinterpret_cast<const float4*>(in + ((n * g.oCb * g.oH + h) * g.oW + w) * 16) + c4);
      ftile[i] = v;
    }
    __syncthreads();
    const int q = q0 + int(threadIdx.x);
    const int nq = g.Q - q0 < kFoldQ ? g.Q - q0 : kFoldQ;  // pixels of this block
    const float* tile = reinterpret_cast<const float*>(ftile) + threadIdx.x * g.osw * c4s * 4;
    float* stage = reinterpret_cast<float*>(ctab + g.Cb2 * 32);  // [kFoldQ][36]: one 32-channel group
    const int64_t pq0 = int64_t(pp) * g.Q + q0;
    for (int g2 = 0; g2 < g.Cb2; ++g2) {
      if (q < g.Q) {
#pragma unroll 2
        for (int k = 0; k < 8; ++k) {
          const int4 ct = reinterpret_cast<const int4*>(ctab)[g2 * 8 + k];
          reinterpret_cast<float4*>(stage + threadIdx.x * 36)[k] =
              make_float4(ct.x >= 0 ? tile[ct.x] : 0.f, ct.y >= 0 ? tile[ct.y] : 0.f, ct.z >= 0 ? tile[ct.z] : 0.f,
                          ct.w >= 0 ? tile[ct.w] : 0.f);
        }
      }
      __syncthreads();
      // the group's nq pixel rows are contiguous in out: coalesced 16-B stores
      float4* dst = reinterpret_cast<float4*>(out) + ((n * g.Cb2 + g2) * PQ + pq0) * 8;
      float4* dlo = lo ? reinterpret_cast<float4*>(lo) + ((n * g.Cb2 + g2) * PQ + pq0) * 8 : nullptr;
      for (int i = threadIdx.x; i < nq * 8; i += kFoldQ) {
        float4 v = reinterpret_cast<const float4*>(stage + (i >> 3) * 36)[i & 7];
        dst[i] = v;
        if (dlo) {
          v.x -= __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
          v.y -= __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
          v.z -= __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
          v.w -= __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
          dlo[i] = v;
        }
      }
      __syncthreads();
    }
  }
}

// dW (KCRS16c16k) = the split partials of every tile added in split order. One 256-thread
// block per 16 x 16 (k, c) block of one tap: it reads the partials along their contiguous
// dimension (64-B segments) and writes the block's 1 KB of dW contiguously (through a shared
// transpose when the partial rows are output channels).
__global__ void __launch_bounds__(256) wgrad_reduce_kernel(const __grid_constant__ WgradParams p, float* __restrict__ dw) {
  __shared__ float tr[16][17];
  ptx::griddep_wait();
  // (tap fold: dW of the original layer; its channel c of tap t is folded channel t * fc + c)
  const int oCb = p.fc ? p.oCb : p.Cb, RS = p.fc ? p.oR * p.oS : p.R * p.S;
  const int64_t nblk = int64_t(p.Kb) * oCb * RS;
  const int64_t tile_elems = int64_t(128) * p.bn;
  const int t = threadIdx.x;
  // read roles: swap 0 -> rows are k (contiguous c): (k16, c16) = (t / 16, t % 16);
  //             swap 1 -> rows are c (contiguous k): (c16, k16) = (t / 16, t % 16)
  const int k16 = p.swap ? (t & 15) : (t >> 4), c16 = p.swap ? (t >> 4) : (t & 15);
  for (int64_t b = blockIdx.x; b < nblk; b += gridDim.x) {
    int64_t r = b;
    const int tap0 = int(r % RS);
    r /= RS;
    const int cb = int(r % oCb);
    const int kb = int(r / oCb);
    const int k = kb * 16 + k16;
    int c = cb * 16 + c16, tap = tap0;
    float s = 0.f;
    bool zero = false;
    if (p.fc) {
      if (c >= p.fc) {  // padded channels of the few-channel layer
        zero = true;
      } else {
        c = tap * p.fc + c;
        tap = 0;
      }
    }
    if (!zero) {
      const int tt = tap / p.ntap, tl = tap - tt * p.ntap, ct = c / p.cn, cl = c - ct * p.cn;
      const int kt = k / p.kn, kl = k - kt * p.kn;
      const int tile = wg_tile_index(p, kt, tt, ct);
      const int xi = tl * p.cn + cl;  // X-side index within the tile (taps x channels)
      const int64_t off = p.swap ? int64_t(xi) * p.bn + kl : int64_t(kl) * p.bn + xi;
      const float* src = p.ws + int64_t(tile) * tile_elems + off;
      for (int sp = 0; sp < p.splits; ++sp) s += src[int64_t(sp) * p.tiles * tile_elems];
    }
    float* blk = dw + b * 256;  // [16c][16k] of (kb, cb, tap0)
    if (p.swap) {
      blk[t] = s;  // t = c16 * 16 + k16: the block's own order
    } else {
      __syncthreads();
      tr[k16][c16] = s;
      __syncthreads();
      blk[t] = tr[t & 15][t >> 4];  // (c16, k16) = (t / 16, t % 16)
    }
  }
}

}  // namespace psconv
