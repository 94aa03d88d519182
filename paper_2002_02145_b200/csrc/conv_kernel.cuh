// Blocked direct-convolution forward on sm_100a tensor cores.
//
// The reference nest (ConvPreset::build, include/nestrank/presets.hpp:60-127;
// paper Fig. 5) is
//   for img, ofm_tile, ifm_tile, oj, kj, ki:            <- outer (driver) loops
//     gemm_microkernel(&out[img][ofm_tile][oj][0][0],   <- band (oi, ofm, ifm)
//                      &flt[ofm_tile][ifm_tile][kj][ki][0][0],
//                      &in[img][ifm_tile][oj*sh+kj][ki][0])
// Here the same contraction is one implicit GEMM per launch:
//   M = pixels (img, oj, oi)   -> 128-row tiles = TMA box [16c][Qb][Pb][Nb][kps blocks]
//   N = output channels        -> BN = 16 * (ofm_tile block count)
//   K = (ifm_tile, kj, ki, ifm)-> one k-step = one (ifm_tile,kj,ki) triple =
//                                 16 channels = two tcgen05 K=8 tf32 MMAs
// i.e. each k-step is exactly the reference microkernel call batch-reduced
// over 128 (or, for a CTA pair, 256) output pixels and BN output channels.
//
// Warp roles (persistent CTA, one per SM):
//   warp 0      TMA producer: A box (NCHW16c, padding = TMA OOB zero fill,
//               stride = TMA element strides) + this CTA's rows of the B block
//               (filter prepacked K-major [C*R*S/16][K][16c])
//   warp 1      TMEM owner; MMA issuer (single CTA, or the pair's leader);
//               in the pair's second CTA: forwards "stage ready" to the leader
//   warps 2-5   epilogue: tcgen05.ld -> registers -> SW64 staging tiles in smem ->
//               one TMA tensor store (or reduce-add for `+=`) per 16-channel block (NKPQ16k)
//   warps 6-9   (3xTF32 only) splitter: A -> lo = A - tf32(A) in shared memory
//
// PAIR (cluster of 2, tcgen05.mma.cta_group::2, M = 256): the two SMs of a
// pair work on two 128-pixel tiles with the same BN output channels; each CTA
// stages its own A tile and HALF of the B block, and the leader issues one
// M=256 MMA that reads A from both SMs and B halves from both. Measured on B200
// (r01 model fit) the single-CTA kernel is bound by ~128 B/cycle/SM of shared
// memory traffic (tensor-core operand reads + TMA writes + splitter); the pair
// halves the B share of both, so the loop becomes MMA-bound.
//
// Numerics (measured on B200, tools/probe2.cu): kind::tf32 reads fp32 operands
// by truncating the 13 low mantissa bits, so A_hi is the raw fp32 tile and only
// A_lo = x - trunc(x) is materialised. The tensor-core accumulation into TMEM
// loses ~2^-25 of the running sum per MMA (error grows linearly with the MMA
// chain), so in 3xTF32 mode the reduction is split into chunks of
// `chunk_stages` pipeline stages: each chunk restarts its TMEM accumulator and the
// epilogue adds the chunks in fp32 (round-to-nearest) into a TMEM running sum.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>

#include "sm100_ptx.cuh"

namespace psconv {

struct ConvParams {
  int img_count, Cb, H, W, Kb, P, Q, R, S, sh, sw, ph, pw;
  int Qb, Pb, Nb;                 // M-tile box in output pixels (Qb*Pb*Nb <= 128)
  int tiles_q, tiles_p, tiles_n;  // M-tile grid
  int tiles_k;                    // N tiles (K / BN)
  int mtiles, mgroups, groups;    // M tiles; groups of CS M tiles; groups * tiles_k
  int m_order;                    // 0: img outer of oj, 1: oj outer of img (oi innermost)
  int k_outer;                    // 1: ofm_tile outer of the pixel loops (recipe order)
  int m_block;                    // > 0: grouped raster, blocks of m_block M groups x all N
                                  // tiles (N outer inside a block) so concurrent CTAs share
                                  // A rows and B columns in L2 (GEMM-like shapes)
  int ksteps;                     // Cb*R*S
  int kps;                        // k-steps per pipeline stage (input-channel blocks per TMA box)
  int cbg;                        // extent of the channel-block counter (Cb / kps or Cb)
  int stages;                     // pipeline stages in the ring (<= kMaxStages)
  int stage_bytes;                // [A x kps | A_lo x kps (3x) | B x kps | B_lo x kps (3x)]
  int ring_bytes;                 // stages * stage_bytes rounded up to 1 KB
  int a_pitch;                    // bytes between the kps A tiles of a stage
  int b128;                       // filter rows hold 2 channel blocks (128 B, SWIZZLE_128B)
  int tmem_a;                     // 3xTF32, BN <= 128: A_hi / A_lo live in TMEM (the splitter
                                  // writes them with tcgen05.st, the MMAs read A from TMEM):
                                  // no A_lo round trip through smem, no smem reads of A by
                                  // the three MMAs per K-half
  int a_slots, a_slot_col;        // TMEM A ring: slots of 32 columns (hi 16 | lo 16) from col
  // halo mode (stride-1 R x S > 1): the M tile is Pb whole output rows of one
  // image laid out at the padded input pitch hw = Q + S - 1 (columns q >= Q
  // are junk rows); one TMA box loads the input halo (hr = Pb + R - 1 rows of
  // hw pixels) per channel block ONCE, and the R*S shifted operands are read
  // in place at row offset kj*hw + ki (any 64-B row start is legal for the
  // SW64 descriptor, tools/probe_shift.cu). A ring: `stages` x `stage_bytes`
  // (kps halo tiles, a_tile bytes apart); B ring: hb_stages x hb_stage_bytes
  // (one (kj, ki) filter box over the kps blocks) at hb_ring_off.
  int halo, hw, hr, a_tile;
  int hb_stages, hb_stage_bytes, hb_ring_off;
  int tc;                         // halo tap concat (TF32, 3x3, bn == K <= 64): per filter row kj
                                  // one N = 3 bn MMA of the shared A rows (halo pitch hw = 32:
                                  // one output row per epilogue warp) into D = [D_0|D_1|D_2];
                                  // out[r] = D_0[r] + D_1[r+1] + D_2[r+2] (warp shuffles)
  int b_res;                      // halo: the CTA's whole filter slice (R*S*cbg boxes of
                                  // hb_stage_bytes at hb_ring_off) loaded once and kept
                                  // resident (one N tile); no B ring
  int cb_group;                   // 1: a stage = kps channel blocks at one (kj, ki), one B box
                                  // spanning them; 0: kps consecutive k-steps, one box each
  int a_boxes;                    // A boxes per coordinate step: 1 (spans the step's blocks;
                                  // a_pitch = box rows x 64 or 8 KB) or kps (one per block, 8 KB)
  int nst;                        // stages per tile = ceil(ksteps / kps)
  int a_lo_off, b_off, b_lo_off;  // region offsets inside a stage
  int chunk_stages;               // stages per TMEM accumulation chunk
  int ksplit;                     // split-K: work units per tile (reduction split into ksplit
                                  // stage ranges of split_stages); 1 = whole tiles
  int split_stages;
  int split_from;                 // tiles [0, split_from) are whole units; later tiles split
  int units;                      // split_from + (groups - split_from) * ksplit
  // Split tiles combine deterministically without any CTA waiting on a CTA that may not
  // be resident: every unit of a split tile takes a ticket (split_ctr[2t], relaxed atomic)
  // when its partial is ready; the first ksplit-1 units write their partial to their slot
  // of split_ws and count themselves done (split_ctr[2t+1], release); the last ticket
  // holder -- whose peers have all taken tickets, i.e. are running their epilogue --
  // waits for the done count, adds the partials in split order ((p0 + p1) + p2 ...) and
  // stores the tile once, then zeroes both counters for the next launch. The workspace and
  // counters are plan-owned (sized at conv_plan_create); no output memset, no atomics on
  // the output, bitwise reproducible.
  int* split_ctr;                 // [2 * split tiles * CS] {tickets, done}
  float* split_ws;                // [split tiles * CS][ksplit][128 x BN] partials
  int tile_chunks;                // accumulation chunks of a whole tile (ksplit == 1)
  int kord[3];                    // stage order outer->inner over {0 ifm group, 1 kj, 2 ki}
  int tap_dw;                     // input columns between consecutive ki taps (1; G for the
                                  // (c,s)-folded input, conv_fwd.cu fold)
  int egroups;                    // host dispatch: epilogue warp groups (kernel template EG)
  int ostages;                    // output staging blocks of 8 KB after the ring: kOutStages, or
                                  // kMaxOutStages (recipe os:8, output-heavy layers: the store warp
                                  // then hands a slot back only when half the slots' stores are
                                  // still reading, so TMA store latency overlaps the next rounds)
  int ncat;                       // 3xTF32, BN <= 64, not halo: filter rows [B_hi;B_lo] per
                                  // N tile; per K half one N = 2 BN MMA A_hi x [B_hi;B_lo]
                                  // (-> D1 | D2) + one N = BN MMA A_lo x B_hi (-> D1);
                                  // the epilogue adds D1 + D2. 45 + 64 instead of 3 x 45
                                  // cycles per K half at BN = 64 (tools/probe_mma_pair.cu)
  const unsigned* absmax_a;        // f16x2: |max| bits of the input range (power-of-two
  const unsigned* absmax_b;        // operand scales; the epilogue unscales) and the filter
  int accumulate;                 // out += conv
  const float* bias;              // fused epilogue: + bias[k] (nullptr: none)
  int relu;                       // fused epilogue: max(., 0) (not with accumulate)
  int debug;                      // profiling only (PSCONV_DEBUG): 1 skip A loads, 2 skip MMA, 4 skip stores, 32 skip B loads
  float* out;                     // output at image img_begin
  long long out_img_stride;       // Kb*P*Q*16 floats
  unsigned long long* trace;      // profiling only (PSCONV_DEBUG & 8): CTA 0 stage timestamps
};
constexpr int kTraceStages = 128;
// trace buffer layout (CTA 0): [producer 4 x S][MMA 4 x S][events 8][splitter 2 x S][epilogue 2 x 32]
constexpr int kTraceSplit = 8 * kTraceStages + 8;
constexpr int kTraceEpi = kTraceSplit + 2 * kTraceStages;
constexpr int kTraceEpiR = kTraceEpi + 64;   // per epilogue round (first 16): 5 timestamps
constexpr int kTraceWords = kTraceEpiR + 80;
// CTA-0 clock trace (PSCONV_DEBUG=8) is compiled in only with -DPSCONV_TRACE
// (tools/build_variant.sh): the instrumented loops measured 5% slower on cfg5.
#ifdef PSCONV_TRACE
constexpr bool kTrace = true;
#else
constexpr bool kTrace = false;
#endif
constexpr int kHaloB = 8;
  // halo mode: B-ring barriers follow 8 A-ring slots

// Shared-memory plan (per CTA, one CTA per SM): a ring of `stages` pipeline
// stages inside kStageBudget, then two output staging blocks, then barriers.
// A stage carries `kps` k-steps loaded by ONE TMA box per operand (the box
// spans kps input-channel blocks): the producer and MMA threads are single
// warps whose per-stage work (barrier wait, expect_tx, TMA issue, commit,
// coordinate update) measured ~270 cycles on B200 (tools/conv_times.py with
// PSCONV_DEBUG=7 on cfg1), which exceeded the 64-cycle MMA time of a BN=64
// k-step; grouping amortises it over kps k-steps.
constexpr int kOutStageBytes = 128 * 64;  // one 128-pixel x 16-channel output block
constexpr int kOutStages = 4;             // staging blocks: two rounds of 32 channels in flight
constexpr int kMaxOutStages = 16;         // recipe os:8 / 12 / 16 (ConvParams::ostages): more rounds, the
                                          // store warp keeps half of them reading smem at a time
constexpr int kStageBudget = 227 * 1024 - kOutStages * kOutStageBytes - 2048 - 1024;
constexpr int kMaxStages = 16;

template <int BN, bool SPLIT3, bool PAIR, int EG = 1>
struct KernelCfg {
  static constexpr int kCS = PAIR ? 2 : 1;
  static constexpr int kBRows = BN / kCS;     // B rows staged per CTA
  static constexpr int kABytes = 128 * 64;    // 128 pixels x 16 fp32 channels
  static constexpr int kBBytes = kBRows * 64; // kBRows output channels x 16 input channels
  static constexpr int kOutStageBytes = psconv::kOutStageBytes;
  // TMEM (per CTA: 128 lanes x BN columns per accumulator)
  static constexpr int kAccBufs = (SPLIT3 && BN == 256) ? 1 : 2;
  // 3xTF32 at BN <= 64 (N-concat, ConvParams::ncat): an accumulator buffer is
  // [D1 | D2], 2 x BN columns (A_hi x [B_hi;B_lo] in one N = 2 BN MMA)
  static constexpr int kAccW = (SPLIT3 && BN <= 64) ? 2 * BN : BN;
  static constexpr int kSumCol = kAccBufs * kAccW;
  static constexpr int kColsNeeded = kAccBufs * kAccW + (SPLIT3 ? BN : 0);
  // 3xTF32 at BN <= 128 takes all 512 columns: the rest hold the TMEM A ring
  static constexpr int kTmemCols = (SPLIT3 && BN <= 128) ? 512
                                   : kColsNeeded <= 32    ? 32
                                   : kColsNeeded <= 64  ? 64
                                   : kColsNeeded <= 128 ? 128
                                   : kColsNeeded <= 256 ? 256
                                                        : 512;
  // two epilogue warp groups (4 warps each, one per TMEM lane quadrant) drain
  // alternate 32-column rounds: TF32 warps 2-5 and 6-9; 3xTF32 warps 2-5 and
  // 10-13 (the splitter is 6-9)
  static constexpr int kEpiGroups = EG;
  // + one store warp: issues the epilogue's TMA stores from the staging slots the
  // epilogue warps fill (mbarrier handshakes), so no epilogue warp waits on a store issue
  static constexpr int kThreads = (SPLIT3 ? 320 : 192) + (kEpiGroups - 1) * 128 + 32;
  static constexpr int kStoreWarp = kThreads / 32 - 1;
  static constexpr int kBarBytes = 1024;
  static constexpr int kSmemBytes =
      kStageBudget + kOutStages * kOutStageBytes + kBarBytes + 1024;  // upper bound (+align slack)
  static constexpr int smem_bytes(int ring_bytes, int ostages = kOutStages) {
    return ring_bytes + ostages * kOutStageBytes + kBarBytes + 1024;
  }
  static constexpr int kDrainW = BN < 32 ? BN : 32;  // epilogue TMEM load width (columns)
  static_assert(BN == 16 || BN == 32 || BN == 64 || BN == 128 || BN == 256, "BN");
  static_assert(kBRows >= 8, "B rows per CTA must be whole 8-row swizzle atoms");
  static_assert(2 * (kABytes + kBBytes) * (SPLIT3 ? 2 : 1) <= kStageBudget, "two stages of one k-step");
  static_assert(kSmemBytes <= 227 * 1024, "smem");
  static_assert(4 * kMaxStages * 8 + 4 * 8 + 8 + 2 * kMaxOutStages * 8 + kMaxOutStages * 4 <= kBarBytes,
                "barriers");  // full/split/empty/aslot + acc + tmem slot/ticket + staging slots
  static_assert(kColsNeeded <= 512, "TMEM");
  // 3xTF32's splitter needs a CTA-local "A landed" signal; pairing it would need
  // a cluster-scope release per k-step (MEMBAR.GPU, measured ~3x slower).
  static_assert(!(PAIR && SPLIT3), "CTA pair is used for TF32 only");
};

struct TileCoord {
  int tn, tp, tq, tk;
  bool live;  // false: padding tile of the last pair group (no stores)
};

__device__ __forceinline__ TileCoord decode_group(const ConvParams& p, int g, int rank, int CS) {
  TileCoord c;
  int mg;
  if (p.m_block > 0) {
    const int per = p.m_block * p.tiles_k;
    const int b = g / per;
    const int base = b * p.m_block;
    const int gm = min(p.m_block, p.mgroups - base);
    const int r = g - b * per;
    c.tk = r / gm;
    mg = base + (r - c.tk * gm);
  } else if (p.k_outer) {
    c.tk = g / p.mgroups;
    mg = g - c.tk * p.mgroups;
  } else {
    mg = g / p.tiles_k;
    c.tk = g - mg * p.tiles_k;
  }
  const int m = mg * CS + rank;
  c.live = m < p.mtiles;
  c.tq = m % p.tiles_q;
  const int rest = m / p.tiles_q;
  if (p.m_order == 0) {
    c.tp = rest % p.tiles_p;
    c.tn = rest / p.tiles_p;  // may exceed tiles_n for padding tiles -> TMA OOB zeros
  } else {
    c.tn = rest % p.tiles_n;
    c.tp = rest / p.tiles_n;
  }
  return c;
}

// lo = x - trunc_tf32(x) over n4 float4s (128 splitter threads), loads batched
// 4 deep for ILP
__device__ __forceinline__ void split_lo(const float4* a, float4* alo, int n4, int tid) {
#ifdef PSCONV_SPLIT_SIMPLE
#pragma unroll 4
  for (int idx = tid; idx < n4; idx += 128) {
    const float4 x = a[idx];
    float4 lo;
    lo.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
    lo.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
    lo.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
    lo.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
    alo[idx] = lo;
  }
  return;
#endif
  for (int base = tid; base < n4; base += 512) {
    float4 x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (base + i * 128 < n4) x[i] = a[base + i * 128];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (base + i * 128 < n4) {
        float4 lo;
        lo.x = x[i].x - __uint_as_float(__float_as_uint(x[i].x) & 0xFFFFE000u);
        lo.y = x[i].y - __uint_as_float(__float_as_uint(x[i].y) & 0xFFFFE000u);
        lo.z = x[i].z - __uint_as_float(__float_as_uint(x[i].z) & 0xFFFFE000u);
        lo.w = x[i].w - __uint_as_float(__float_as_uint(x[i].w) & 0xFFFFE000u);
        alo[base + i * 128] = lo;
      }
    }
  }
}

// f16x2 scale: 2^(14 - e) for |max| in [2^e, 2^(e+1)), so scaled operands stay
// below 2^15 (fp16 max 65504) and keep the most precision in hi / lo
__device__ __forceinline__ float pow2_scale(unsigned absmax_bits) {
  if ((absmax_bits & 0x7FFFFFFFu) == 0) return 1.f;
  int se = 14 - (static_cast<int>((absmax_bits >> 23) & 0xFFu) - 127);
  se = se > 127 ? 127 : (se < -126 ? -126 : se);
  return __uint_as_float(static_cast<uint32_t>(se + 127) << 23);
}

// f16x2 splitter: each 64-B fp32 row (16 channels, SW64 layout) of the stage's A
// tiles -> a 64-B row of fp16 [hi 0..15 | lo 0..15] at the same offset of the out
// region (same swizzle phase), x * s = hi + lo (both round-to-nearest). Each thread
// walks its row's logical chunks (physical = logical ^ phase): conflict-free.
__device__ __forceinline__ void split_f16(const uint8_t* a, uint8_t* out, int rows, int tid, float s) {
  for (int r = tid; r < rows; r += 128) {
    const uint32_t ph = (static_cast<uint32_t>(r) >> 1) & 3u;
    float4 x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = *reinterpret_cast<const float4*>(a + r * 64 + ((k ^ ph) << 4));
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float v[4] = {x[k].x * s, x[k].y * s, x[k].z * s, x[k].w * s};
#pragma unroll
      for (int e = 0; e < 4; e += 2) {
        const __half2 h = __floats2half2_rn(v[e], v[e + 1]);
        const float2 hf = __half22float2(h);
        const __half2 l = __floats2half2_rn(v[e] - hf.x, v[e + 1] - hf.y);
        hi[k * 2 + e / 2] = *reinterpret_cast<const uint32_t*>(&h);
        lo[k * 2 + e / 2] = *reinterpret_cast<const uint32_t*>(&l);
      }
    }
    uint8_t* o = out + r * 64;
    *reinterpret_cast<uint4*>(o + ((0u ^ ph) << 4)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(o + ((1u ^ ph) << 4)) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
    *reinterpret_cast<uint4*>(o + ((2u ^ ph) << 4)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    *reinterpret_cast<uint4*>(o + ((3u ^ ph) << 4)) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
  }
}

// Halo-mode producer (warp 0; warp-uniform loop, one elected lane issues).
// Per M tile and input-channel group: one halo box into the A ring, then one
// filter box per (kj, ki) tap into the B ring.
// split-K work unit u -> (tile group, stage range [ib, ie))
enum : int { kEpiStore = 0, kEpiFused = 1, kEpiSplit = 2 };
struct Unit {
  int g, ib, ie, sp;  // sp: split index, -1 for a whole tile
};
// SPLITK: the launch splits its tail tiles (EPI == kEpiSplit); otherwise every
// unit is a whole tile
template <bool SPLITK>
__device__ __forceinline__ Unit decode_unit(const ConvParams& p, int u) {
  Unit w;
  if (!SPLITK || u < p.split_from) {  // whole tiles: no divisions on the producer's per-tile path
    w.g = u;
    w.ib = 0;
    w.ie = p.nst;
    w.sp = -1;
    return w;
  }
  const int v = u - p.split_from;
  const int t = v / p.ksplit;
  w.g = p.split_from + t;
  w.sp = v - t * p.ksplit;
  w.ib = w.sp * p.split_stages;
  w.ie = min(p.nst, w.ib + p.split_stages);
  return w;
}

template <int BN, bool SPLIT3, bool PAIR>
__device__ __forceinline__ void halo_producer(const ConvParams& p, uint8_t* smem, uint64_t* full,
                                              uint64_t* empty, int cluster, int nclusters, int rank,
                                              bool leader, const CUtensorMap* tmap_in,
                                              const CUtensorMap* tmap_flt, const CUtensorMap* tmap_flt_lo) {
  using Cfg = KernelCfg<BN, SPLIT3, PAIR>;
  constexpr int CS = Cfg::kCS;
  const bool skip_a = (p.debug & 1) != 0;
  const uint32_t a_tx = (skip_a ? 0u : static_cast<uint32_t>(p.kps * p.hr * p.hw * 64)) * CS;
  // one B box (a tap, or with tap concat a filter row of S taps) over kps blocks, both CTAs
  const uint32_t b_tx = static_cast<uint32_t>(p.hb_stage_bytes) * CS;
  const bool hncat = SPLIT3 && BN <= 64 && p.ncat != 0;  // 3xTF32 N-concat filter rows
  const uint32_t full_leader = PAIR ? ptx::mapa(&full[0], 0) : 0u;
  const int taps = p.tc ? p.R : p.R * p.S;
  const int brows = p.tc ? p.S * Cfg::kBRows : Cfg::kBRows;  // B rows of one CTA's box
  int as = 0, bs = 0, gs = 0;
  uint32_t aph = 0, bph = 0;
  if (p.b_res) {
    // resident filter slice: every (channel group, tap) box once, one barrier
    // (PAIR: each CTA loads its BN/2 rows, completing on the leader's barrier)
    const int k0 = rank * brows;  // single N tile (tiles_k == 1)
    if (ptx::elect_one()) {
      if (!PAIR || leader) ptx::mbar_expect_tx(&full[kHaloB], b_tx * p.cbg * taps);
      for (int cg = 0; cg < p.cbg; ++cg)
        for (int t = 0; t < taps; ++t) {
          uint8_t* sb = smem + p.hb_ring_off + (cg * taps + t) * p.hb_stage_bytes;
          const int cb = cg * p.kps;
          if (!PAIR) {
            // (N-concat: one box of [B_hi; B_lo] rows per block, conv_fwd.cu)
            ptx::tma_load_4d(sb, tmap_flt, &full[kHaloB], 0, hncat ? 2 * k0 : k0, t, cb >> p.b128);
            if (SPLIT3 && !hncat)
              ptx::tma_load_4d(sb + p.b_lo_off, tmap_flt_lo, &full[kHaloB], 0, k0, t, cb >> p.b128);
          } else {
            ptx::tma_load_4d_cb(sb, tmap_flt, full_leader + 8u * kHaloB, 0, k0, t, cb >> p.b128);
          }
        }
    }
    __syncwarp();
  }
  for (int g = cluster; g < p.groups; g += nclusters) {
    const TileCoord tc = decode_group(p, g, rank, CS);
    const int hp = tc.tp * p.Pb - p.ph;
    const int wq = tc.tq * p.Qb - p.pw;  // (whole rows: tq = 0; tap concat: Qb-wide column tiles)
    const int n0 = tc.tn;
    const int k0 = tc.tk * BN * (p.tc ? p.S : 1) + rank * brows;
    for (int cg = 0; cg < p.cbg; ++cg) {
      const int cb = cg * p.kps;
      ptx::mbar_wait(&empty[as], aph ^ 1);
      if (ptx::elect_one()) {
        uint8_t* sa = smem + as * p.stage_bytes;
        if (!PAIR) {
          ptx::mbar_expect_tx(&full[as], a_tx);
          if (!skip_a) ptx::tma_load_5d(sa, tmap_in, &full[as], 0, wq, hp, n0, cb);
        } else {
          if (leader) ptx::mbar_expect_tx(&full[as], a_tx);
          if (!skip_a) ptx::tma_load_5d_cb(sa, tmap_in, full_leader + 8u * as, 0, wq, hp, n0, cb);
        }
      }
      __syncwarp();
      if (++as == p.stages) {
        as = 0;
        aph ^= 1;
      }
      for (int t = 0; t < taps && !p.b_res; ++t) {
        const int bi = kHaloB + bs;
        const bool tr = kTrace && p.trace != nullptr && blockIdx.x == 0 && gs < kTraceStages;
        if (tr) p.trace[gs * 4 + 0] = clock64();
        ptx::mbar_wait(&empty[bi], bph ^ 1);
        if (tr) p.trace[gs * 4 + 1] = clock64();
        if (ptx::elect_one()) {
          uint8_t* sb = smem + p.hb_ring_off + bs * p.hb_stage_bytes;
          if (!PAIR) {
            ptx::mbar_expect_tx(&full[bi], b_tx);
            ptx::tma_load_4d(sb, tmap_flt, &full[bi], 0, hncat ? 2 * k0 : k0, t, cb >> p.b128);
            if (SPLIT3 && !hncat)
              ptx::tma_load_4d(sb + p.b_lo_off, tmap_flt_lo, &full[bi], 0, k0, t, cb >> p.b128);
          } else {
            if (leader) ptx::mbar_expect_tx(&full[bi], b_tx);
            ptx::tma_load_4d_cb(sb, tmap_flt, full_leader + 8u * bi, 0, k0, t, cb >> p.b128);
          }
        }
        __syncwarp();
        if (tr) p.trace[gs * 4 + 2] = clock64();
        ++gs;
        if (++bs == p.hb_stages) {
          bs = 0;
          bph ^= 1;
        }
      }
    }
  }
}

// Lean halo-mode MMA issuer for 3x3 taps with one accumulation chunk per tile:
// per (tile, channel group) one elected thread issues all 9 x KPS x 2 (x3 in
// 3xTF32) MMAs with compile-time tap offsets (A: kj*hw + ki rows into the halo
// tile). BRES: the filter is resident (box t of the group); otherwise the
// thread waits for each tap's B-ring stage and releases it by a commit. The
// generic issuer's per-tap bookkeeping (~200-400 cycles per tap, measured with
// the clock trace) starves the tensor core at N = 64 (48-cycle MMAs).
// TC (tap concat, TF32, bn <= 64): per filter row kj ONE MMA of N = 3 bn over the three
// ki taps' filter rows [W(kj,0); W(kj,1); W(kj,2)] with the A rows shifted by kj*hw only:
// D_ki[r] = sum x[r + kj*hw] W(kj, ki), and the epilogue forms out[r] = sum_ki D_ki[r + ki].
// N = 192 runs at the full tensor rate (96 cycles per K = 8) where three N = 64 MMAs take
// 3 x 45-48 (tools/probe_mma_rate.cu).
template <int BN, bool SPLIT3, bool PAIR, int KPS, bool BRES, bool TC = false>
__device__ __forceinline__ void halo_mma_fast(const ConvParams& p, uint8_t* smem, uint64_t* full,
                                             uint64_t* split_full, uint64_t* empty, uint64_t* acc_full,
                                             uint64_t* acc_empty, uint32_t tmem_base, int cluster,
                                             int nclusters, uint32_t idesc) {
  using Cfg = KernelCfg<BN, SPLIT3, PAIR>;
  constexpr int kAccBufs = Cfg::kAccBufs;
  constexpr int kTaps = TC ? 3 : 9;                   // MMA groups per channel group
  constexpr int kAccW = TC ? 3 * BN : Cfg::kAccW;     // accumulator columns per buffer
  constexpr uint32_t kIdescTC = ptx::idesc_tf32_m128<(3 * BN <= 256 ? 3 * BN : BN), 128 * Cfg::kCS>();
  const uint64_t adesc0 = ptx::smem_desc_sw64(ptx::smem_u32(smem), 16, 512);
  const uint64_t bdesc0 = p.b128 ? ptx::smem_desc_sw128(ptx::smem_u32(smem), 16, 1024) : adesc0;
  const bool hncat = SPLIT3 && BN <= 64 && p.ncat != 0;  // [B_hi; B_lo] rows per block
  const uint32_t bblk = static_cast<uint32_t>(Cfg::kBBytes * (hncat ? 2 : 1) * (TC ? 3 : 1)) >> 4;
  const uint32_t b_even = p.b128 ? 4u : bblk;
  const uint32_t b_odd = p.b128 ? (2u * bblk - 4u) : bblk;
  constexpr uint32_t kIdesc2 = ptx::idesc_tf32_m128<(BN <= 128 ? 2 * BN : BN), 128 * Cfg::kCS>();
  const uint32_t a_tile = static_cast<uint32_t>(p.a_tile) >> 4;
  const uint32_t alo_off = static_cast<uint32_t>(p.a_lo_off) >> 4;
  const uint32_t blo_off = static_cast<uint32_t>(p.b_lo_off) >> 4;
  const uint32_t hw4 = static_cast<uint32_t>(p.hw) * 4u;  // one row = 64 B = 4 desc units
  const uint32_t bstep = static_cast<uint32_t>(p.hb_stage_bytes) >> 4;
  const uint32_t bres = static_cast<uint32_t>(p.hb_ring_off) >> 4;
  const uint32_t astage = static_cast<uint32_t>(p.stage_bytes) >> 4;
  const bool skip_mma = (p.debug & 2) != 0;
  if (BRES) {
    ptx::mbar_wait(&full[kHaloB], 0);  // resident filter slice landed (both CTAs')
    ptx::tc_fence_after();
  }
  int as = 0, cit = 0, bs = 0;
  uint32_t aph = 0, bph = 0;
  for (int g = cluster; g < p.groups; g += nclusters, ++cit) {
    const int buf = kAccBufs == 1 ? 0 : (cit & 1);
    const uint32_t acc_phase = (kAccBufs == 1 ? cit : (cit >> 1)) & 1;
    if (PAIR)
      ptx::mbar_wait_cluster(&acc_empty[buf], acc_phase ^ 1);
    else
      ptx::mbar_wait(&acc_empty[buf], acc_phase ^ 1);
    const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(buf * kAccW);
    for (int cg = 0; cg < p.cbg; ++cg) {
      const int gs = cit * p.cbg + cg;
      const bool tr = kTrace && p.trace != nullptr && blockIdx.x == 0 && gs < kTraceStages;
      if (tr) p.trace[4 * kTraceStages + gs * 4 + 0] = clock64();
      ptx::mbar_wait(&full[as], aph);  // PAIR: both CTAs' halos landed
      if (tr) p.trace[4 * kTraceStages + gs * 4 + 3] = clock64();
      if (SPLIT3) ptx::mbar_wait(&split_full[as], aph);
      ptx::tc_fence_after();
      if (tr) p.trace[4 * kTraceStages + gs * 4 + 1] = clock64();
      if (ptx::elect_one()) {
        const uint64_t a0 = adesc0 + static_cast<uint32_t>(as) * astage;
        const uint64_t b0 = bdesc0 + bres + static_cast<uint32_t>(BRES ? cg * kTaps : 0) * bstep;
        uint32_t acc_in = cg == 0 ? 0u : 1u;
        int ts = bs;
        uint32_t tph = bph;
#pragma unroll
        for (int t = 0; t < kTaps; ++t) {
          uint64_t da = TC ? a0 + static_cast<uint32_t>(t) * hw4
                           : a0 + static_cast<uint32_t>(t / 3) * hw4 + static_cast<uint32_t>(t % 3) * 4u;
          uint64_t db = b0 + static_cast<uint32_t>(BRES ? t : ts) * bstep;
          if (!BRES) {
            ptx::mbar_wait(&full[kHaloB + ts], tph);  // this tap's filter box landed
            ptx::tc_fence_after();
          }
#pragma unroll
          for (int j = 0; j < KPS; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (!skip_mma) {
                if (TC && PAIR) {
                  ptx::mma_tf32_pair(d_tmem, da + h * 2, db + h * 2, kIdescTC, acc_in);  // -> D0|D1|D2
                } else if (TC) {
                  ptx::mma_tf32(d_tmem, da + h * 2, db + h * 2, kIdescTC, acc_in);
                } else if (SPLIT3 && hncat) {
                  ptx::mma_tf32(d_tmem, da + h * 2, db + h * 2, kIdesc2, acc_in);        // -> D1 | D2
                  ptx::mma_tf32(d_tmem, da + alo_off + h * 2, db + h * 2, idesc, 1u);   // A_lo B_hi
                } else if (SPLIT3) {
                  ptx::mma_tf32(d_tmem, da + alo_off + h * 2, db + h * 2, idesc, acc_in);
                  ptx::mma_tf32(d_tmem, da + h * 2, db + blo_off + h * 2, idesc, 1u);
                  ptx::mma_tf32(d_tmem, da + h * 2, db + h * 2, idesc, 1u);
                } else if (PAIR) {
                  ptx::mma_tf32_pair(d_tmem, da + h * 2, db + h * 2, idesc, acc_in);
                } else {
                  ptx::mma_tf32(d_tmem, da + h * 2, db + h * 2, idesc, acc_in);
                }
              }
              acc_in = 1u;
            }
            da += a_tile;
            db += (j & 1) ? b_odd : b_even;
          }
          if (!BRES) {  // release the tap's B stage once its MMAs completed
            if (PAIR)
              ptx::mma_commit_pair(&empty[kHaloB + ts]);
            else
              ptx::mma_commit(&empty[kHaloB + ts]);
            if (++ts == p.hb_stages) {
              ts = 0;
              tph ^= 1;
            }
          }
        }
        if (PAIR) {
          ptx::mma_commit_pair(&empty[as]);
          if (cg == p.cbg - 1) ptx::mma_commit_pair(&acc_full[buf]);
        } else {
          ptx::mma_commit(&empty[as]);
          if (cg == p.cbg - 1) ptx::mma_commit(&acc_full[buf]);
        }
      }
      __syncwarp();
      if (tr) p.trace[4 * kTraceStages + gs * 4 + 2] = clock64();
      if (!BRES)
        for (int t = 0; t < kTaps; ++t)  // warp-uniform copy of the B-ring position
          if (++bs == p.hb_stages) {
            bs = 0;
            bph ^= 1;
          }
      if (++as == p.stages) {
        as = 0;
        aph ^= 1;
      }
    }
  }
}

// Halo-mode MMA issuer (warp 1 of the single CTA / pair leader). Walks the same
// (channel group, tap) sequence; accumulation chunks are counted in taps.
template <int BN, bool SPLIT3, bool PAIR>
__device__ __forceinline__ void halo_mma(const ConvParams& p, uint8_t* smem, uint64_t* full,
                                         uint64_t* split_full, uint64_t* empty, uint64_t* acc_full,
                                         uint64_t* acc_empty, uint32_t tmem_base, int cluster,
                                         int nclusters, uint32_t idesc) {
  using Cfg = KernelCfg<BN, SPLIT3, PAIR>;
  constexpr int kAccBufs = Cfg::kAccBufs;
  const uint64_t adesc0 = ptx::smem_desc_sw64(ptx::smem_u32(smem), 16, 512);
  const uint64_t bdesc0 = p.b128 ? ptx::smem_desc_sw128(ptx::smem_u32(smem), 16, 1024) : adesc0;
  const bool hncat = SPLIT3 && BN <= 64 && p.ncat != 0;  // [B_hi; B_lo] rows per block
  const uint32_t bblk = static_cast<uint32_t>(Cfg::kBBytes * (hncat ? 2 : 1)) >> 4;
  const uint32_t b_even = p.b128 ? 4u : bblk;
  const uint32_t b_odd = p.b128 ? (2u * bblk - 4u) : bblk;
  constexpr uint32_t kIdesc2 = ptx::idesc_tf32_m128<(BN <= 128 ? 2 * BN : BN), 128 * Cfg::kCS>();
  const uint32_t a_tile = static_cast<uint32_t>(p.a_tile) >> 4;
  const uint32_t alo_off = static_cast<uint32_t>(p.a_lo_off) >> 4;
  const uint32_t blo_off = static_cast<uint32_t>(p.b_lo_off) >> 4;
  const int taps = p.R * p.S;
  const int kps = p.kps;
  const bool skip_mma = (p.debug & 2) != 0;
  int as = 0, bs = 0, cit = 0, gs = 0;
  uint32_t aph = 0, bph = 0;
  if (p.b_res) {
    ptx::mbar_wait(&full[kHaloB], 0);  // resident filter slice landed (both CTAs')
    ptx::tc_fence_after();
  }
  for (int g = cluster; g < p.groups; g += nclusters) {
    int tg = 0;  // tap index within the tile's reduction
    int cc = 0;  // taps into the current accumulation chunk
    int buf = 0;
    uint32_t d_tmem = tmem_base;
    for (int cg = 0; cg < p.cbg; ++cg) {
      ptx::mbar_wait(&full[as], aph);  // PAIR: both CTAs' halos landed
      if (SPLIT3) ptx::mbar_wait(&split_full[as], aph);
      int r = 0, sx = 0;
      for (int t = 0; t < taps; ++t, ++tg) {
        const bool chunk_start = cc == 0;
        const bool chunk_end = cc + 1 == p.chunk_stages || tg + 1 == p.nst;
        if (chunk_start) {
          buf = kAccBufs == 1 ? 0 : (cit & 1);
          const uint32_t acc_phase = (kAccBufs == 1 ? cit : (cit >> 1)) & 1;
          if (PAIR)
            ptx::mbar_wait_cluster(&acc_empty[buf], acc_phase ^ 1);
          else
            ptx::mbar_wait(&acc_empty[buf], acc_phase ^ 1);
          d_tmem = tmem_base + static_cast<uint32_t>(buf * Cfg::kAccW);
        }
        const int bi = kHaloB + bs;
        const bool tr = kTrace && p.trace != nullptr && blockIdx.x == 0 && gs < kTraceStages;
        if (tr) p.trace[4 * kTraceStages + gs * 4 + 0] = clock64();
        if (!p.b_res) {
          ptx::mbar_wait(&full[bi], bph);
          ptx::tc_fence_after();
        }
        if (tr) p.trace[4 * kTraceStages + gs * 4 + 1] = clock64();
        if (ptx::elect_one()) {
          uint64_t da = adesc0 + ((static_cast<uint32_t>(as * p.stage_bytes) +
                                   static_cast<uint32_t>(r * p.hw + sx) * 64u) >> 4);
          const int bslot = p.b_res ? cg * taps + t : bs;
          uint64_t db = bdesc0 + ((static_cast<uint32_t>(p.hb_ring_off + bslot * p.hb_stage_bytes)) >> 4);
          uint32_t acc_in = chunk_start ? 0u : 1u;
          for (int j = 0; j < kps && !skip_mma; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (SPLIT3 && hncat) {
                ptx::mma_tf32(d_tmem, da + h * 2, db + h * 2, kIdesc2, acc_in);        // -> D1 | D2
                ptx::mma_tf32(d_tmem, da + alo_off + h * 2, db + h * 2, idesc, 1u);   // A_lo B_hi
              } else if (SPLIT3) {
                ptx::mma_tf32(d_tmem, da + alo_off + h * 2, db + h * 2, idesc, acc_in);
                ptx::mma_tf32(d_tmem, da + h * 2, db + blo_off + h * 2, idesc, 1u);
                ptx::mma_tf32(d_tmem, da + h * 2, db + h * 2, idesc, 1u);
              } else if (PAIR) {
                ptx::mma_tf32_pair(d_tmem, da + h * 2, db + h * 2, idesc, acc_in);
              } else {
                ptx::mma_tf32(d_tmem, da + h * 2, db + h * 2, idesc, acc_in);
              }
              acc_in = 1u;
            }
            da += a_tile;
            db += (j & 1) ? b_odd : b_even;
          }
          if (PAIR) {
            if (!p.b_res) ptx::mma_commit_pair(&empty[bi]);
            if (t == taps - 1) ptx::mma_commit_pair(&empty[as]);
            if (chunk_end) ptx::mma_commit_pair(&acc_full[buf]);
          } else {
            if (!p.b_res) ptx::mma_commit(&empty[bi]);
            if (t == taps - 1) ptx::mma_commit(&empty[as]);
            if (chunk_end) ptx::mma_commit(&acc_full[buf]);
          }
        }
        __syncwarp();
        if (tr) p.trace[4 * kTraceStages + gs * 4 + 2] = clock64();
        ++gs;
        if (chunk_end) {
          ++cit;
          cc = 0;
        } else {
          ++cc;
        }
        if (++sx == p.S) {
          sx = 0;
          ++r;
        }
        if (++bs == p.hb_stages) {
          bs = 0;
          bph ^= 1;
        }
      }
      if (++as == p.stages) {
        as = 0;
        aph ^= 1;
      }
    }
  }
}

// EPI: the output path, each a separate instantiation (runtime checks in the
// per-block store loop cost 5-10% on epilogue-heavy layers, measured on l1 1x1
// 64->64 / 64->256): kEpiStore (store, or reduce-add for `+=`), kEpiFused
// (+ bias / ReLU), kEpiSplit (tail split-K units, flag-ordered partials)
// EG: epilogue warp groups (1, or 2 draining alternate 32-channel rounds; recipe eg:)
// F16 (with SPLIT3): the f16x2 mode -- the splitter writes scaled fp16 hi|lo rows
// of A, the filter rows hold fp16 hi|lo, three K=16 kind::f16 MMAs per k-step
template <int BN, bool SPLIT3, bool PAIR, int EPI, int EG, bool F16 = false>
__global__ void __launch_bounds__(KernelCfg<BN, SPLIT3, PAIR, EG>::kThreads, 1)
    conv_fwd_sm100(const __grid_constant__ ConvParams p, const __grid_constant__ CUtensorMap tmap_in,
                   const __grid_constant__ CUtensorMap tmap_flt,
                   const __grid_constant__ CUtensorMap tmap_flt_lo,
                   const __grid_constant__ CUtensorMap tmap_out) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  using Cfg = KernelCfg<BN, SPLIT3, PAIR, EG>;
  constexpr int CS = Cfg::kCS;
  const int kStages = p.stages;
  constexpr int kAccBufs = Cfg::kAccBufs;
  constexpr uint32_t kIdesc = ptx::idesc_tf32_m128<BN, 128 * CS>();
  constexpr uint32_t kIdescF16 = ptx::idesc_f16_m128<BN, 128 * CS>();
  // N-concat only exists at BN <= 64 (3xTF32): wider tiles fold the check away (a
  // runtime test in the MMA issue loop cost 9% on cfg5)
  const bool ncat = SPLIT3 && !F16 && BN <= 64 && p.ncat != 0;

  const long long t_entry = clock64();
  unsigned long long* ev = (kTrace && p.trace != nullptr && blockIdx.x == 0) ? p.trace + 8 * kTraceStages : nullptr;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B align the carve-out (SWIZZLE_64B atoms are 512 B). The offset is the
  // same in both CTAs of a pair, which the pair MMA relies on.
  // (pointer arithmetic on the __shared__ array, not an integer round trip: the compiler
  // keeps the shared address space and emits STS/LDS instead of generic ST.E/LD.E)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  auto stage_base = [&](int s) { return smem + s * p.stage_bytes; };

  uint8_t* out_stage = smem + p.ring_bytes;  // p.ostages x 8 KB (1024-B aligned)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.ring_bytes + p.ostages * Cfg::kOutStageBytes);
  uint64_t* full = bars;                         // own TMA landed (1 arrive + tx)
  uint64_t* split_full = bars + kMaxStages;      // own splitter done (count 128)
  uint64_t* empty = bars + 2 * kMaxStages;       // MMA consumed the stage (commit, pair: both CTAs)
  uint64_t* acc_full = bars + 3 * kMaxStages;    // chunk accumulator ready   [kAccBufs]
  uint64_t* acc_empty = acc_full + 2;            // chunk accumulator drained [kAccBufs] (4 warps x CS)
  uint64_t* aslot_empty = acc_empty + 2;         // TMEM A slot consumed by the MMA [kMaxStages]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aslot_empty + kMaxStages);
  volatile int* split_word = reinterpret_cast<volatile int*>(tmem_slot + 1);  // split-K ticket broadcast
  uint64_t* out_full = aslot_empty + kMaxStages + 1;  // staging slot filled (128 epilogue threads)
  uint64_t* out_free = out_full + kMaxOutStages;      // staging slot read by its TMA store (store warp)
  volatile int* out_skip = reinterpret_cast<volatile int*>(out_free + kMaxOutStages);  // slot holds no tile

  const int warp = threadIdx.x >> 5;
  const int rank = PAIR ? static_cast<int>(blockIdx.x & 1) : 0;
  const bool leader = rank == 0;
  const int cluster = blockIdx.x / CS;
  const int nclusters = gridDim.x / CS;
  const int nst = p.nst;  // pipeline stages per tile

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&split_full[s], 128);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < (p.halo ? p.hb_stages : 0); ++s) {  // halo B ring: barriers 8..
      ptx::mbar_init(&full[kHaloB + s], 1);
      ptx::mbar_init(&empty[kHaloB + s], 1);
    }
    for (int a = 0; a < kAccBufs; ++a) {
      ptx::mbar_init(&acc_full[a], 1);
      ptx::mbar_init(&acc_empty[a], 4 * EG * CS);
    }
    for (int a = 0; a < (p.tmem_a ? p.a_slots : 0); ++a) ptx::mbar_init(&aslot_empty[a], 1);
    for (int o = 0; o < kMaxOutStages; ++o) {
      ptx::mbar_init(&out_full[o], 128);
      ptx::mbar_init(&out_free[o], 1);
    }
    ptx::fence_mbar_init();
  }
  // tap concat needs 2 x 3 bn accumulator columns (bn 64: 384 -> 512)
  const uint32_t tmem_cols = (!SPLIT3 && BN <= 64 && p.tc) ? 512u : static_cast<uint32_t>(Cfg::kTmemCols);
  if (warp == 1) {
    if (PAIR)
      ptx::tmem_alloc_pair(tmem_slot, tmem_cols);
    else
      ptx::tmem_alloc(tmem_slot, tmem_cols);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (PAIR) ptx::cluster_sync_all();  // both CTAs' barriers initialised, TMEM allocated
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: the next kernel in the stream may be scheduled now -- its CTAs take an SM as soon
  // as ours leave it and run their prologue there; every global read or write it makes
  // waits in its griddepcontrol.wait for this grid's completion and memory flush
  ptx::griddep_launch_dependents();
  if (ev && threadIdx.x == 0) {
    ev[0] = t_entry;
    ev[1] = clock64();  // barriers initialised, TMEM allocated
  }

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // Warp-uniform loop (all lanes iterate, one elected lane issues): keeps the
    // coordinates in uniform registers; k-step coordinates advance
    // incrementally in the recipe's reduction order (no divisions).
    if (ptx::elect_one()) {
      ptx::prefetch_tmap(&tmap_in);
      ptx::prefetch_tmap(&tmap_flt);
      if (SPLIT3) ptx::prefetch_tmap(&tmap_flt_lo);
    }
    // all global-memory operands come from earlier kernels in the stream (PDL)
    ptx::griddep_wait();
    __syncwarp();
    if (p.halo) {
      halo_producer<BN, SPLIT3, PAIR>(p, smem, full, empty, cluster, nclusters, rank, leader,
                                      &tmap_in, &tmap_flt, &tmap_flt_lo);
    } else {
    // one box per operand per stage: A spans kps channel blocks (tensor map
    // dims [16c][W][H][img][Cb], so each block's rows land contiguously),
    // B spans the same kps blocks of the prepacked filter ([16c][K][R*S][Cb])
    const uint32_t a_step_bytes = static_cast<uint32_t>(p.Qb * p.Pb * p.Nb * 64);
    // PAIR: both CTAs' loads complete on the LEADER's full barrier (the leader
    // expects both shares); the second CTA never arrives on its own.
    const bool skip_a = (p.debug & 1) != 0;
    const bool skip_b = (p.debug & 32) != 0;  // profiling: what a resident filter would save
    const uint32_t tx1 =
        ((skip_a ? 0u : a_step_bytes) + (skip_b ? 0u : Cfg::kBBytes * (SPLIT3 && !F16 ? 2 : 1))) * CS;  // per k-step
    const uint32_t full_leader = PAIR ? ptx::mapa(&full[0], 0) : 0u;
    // cb_group: one coordinate step per stage, boxes span kps channel blocks;
    // otherwise kps coordinate steps per stage (the last stage may be partial)
    const int nsub = p.cb_group ? 1 : p.kps;
    const int tap_dw = p.tap_dw;
    const int cb_mul = p.cb_group ? p.kps : 1;
    const int d0 = p.kord[0], d1 = p.kord[1], d2 = p.kord[2];
    const int e1 = d1 == 0 ? p.cbg : (d1 == 1 ? p.R : p.S);
    const int e2 = d2 == 0 ? p.cbg : (d2 == 1 ? p.R : p.S);
    int stage = 0, gs = 0;
    uint32_t phase = 0;
    for (int u = cluster; u < p.units; u += nclusters) {
      const Unit un = decode_unit<EPI == kEpiSplit>(p, u);
      const TileCoord tc = decode_group(p, un.g, rank, CS);
      const int wq = tc.tq * p.Qb * p.sw - p.pw;
      const int hp = tc.tp * p.Pb * p.sh - p.ph;
      const int n0 = tc.tn * p.Nb;
      const int k0 = tc.tk * BN + rank * Cfg::kBRows;
      // reduction-loop counters (outer -> inner) at the unit's first coordinate step
      int v0 = 0, v1 = 0, v2 = 0;
      if (un.ib > 0) {
        const int t0 = p.cb_group ? un.ib : un.ib * p.kps;
        v2 = t0 % e2;
        v1 = (t0 / e2) % e1;
        v0 = t0 / (e2 * e1);
      }
      for (int it = un.ib; it < un.ie; ++it) {
        const int nk = min(p.kps, p.ksteps - it * p.kps);
        const bool tr = kTrace && p.trace != nullptr && blockIdx.x == 0 && gs < kTraceStages;
        if (tr) p.trace[gs * 4 + 0] = clock64();
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        if (tr) p.trace[gs * 4 + 1] = clock64();
        uint8_t* sb = stage_base(stage);
        const bool issuer = ptx::elect_one();
        if (issuer && (!PAIR || leader)) ptx::mbar_expect_tx(&full[stage], tx1 * nk);
        for (int j = 0; j < nsub && j < nk; ++j) {
          const int cb = (d0 == 0 ? v0 : (d1 == 0 ? v1 : v2)) * cb_mul;
          const int r = d0 == 1 ? v0 : (d1 == 1 ? v1 : v2);
          const int s = d0 == 2 ? v0 : (d1 == 2 ? v1 : v2);
          const int rs = r * p.S + s;
          const int tw = s * tap_dw;  // input column of tap ki (tap dilation of the fold)
          if (issuer) {
            uint8_t* sa = sb + j * p.a_boxes * p.a_pitch;
            uint8_t* sbb = sb + p.b_off + j * Cfg::kBBytes * (ncat ? 2 : 1);
            if (!PAIR) {
              if (!skip_a)
                for (int i = 0; i < p.a_boxes; ++i)
                  ptx::tma_load_5d(sa + i * p.a_pitch, &tmap_in, &full[stage], 0, wq + tw, hp + r, n0, cb + i);
              // (ncat: one box of [B_hi;B_lo] rows of the N tile)
              if (!skip_b) ptx::tma_load_4d(sbb, &tmap_flt, &full[stage], 0, ncat ? 2 * k0 : k0, rs, cb >> p.b128);
              if (SPLIT3 && !F16 && !ncat && !skip_b)
                ptx::tma_load_4d(sbb - p.b_off + p.b_lo_off, &tmap_flt_lo, &full[stage], 0, k0, rs,
                                 cb >> p.b128);
            } else {
              const uint32_t fb = full_leader + 8u * stage;
              if (!skip_a)
                for (int i = 0; i < p.a_boxes; ++i)
                  ptx::tma_load_5d_cb(sa + i * p.a_pitch, &tmap_in, fb, 0, wq + tw, hp + r, n0, cb + i);
              if (!skip_b) ptx::tma_load_4d_cb(sbb, &tmap_flt, fb, 0, k0, rs, cb >> p.b128);
            }
          }
          if (++v2 == e2) {
            v2 = 0;
            if (++v1 == e1) {
              v1 = 0;
              ++v0;
            }
          }
        }
        __syncwarp();
        if (tr) p.trace[gs * 4 + 2] = clock64();
        ++gs;
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    }  // !halo
  } else if (warp == 1 && leader && p.halo) {
    // 3x3, one chunk per tile: the lean issuer (resident filter or B ring)
    const bool fast = p.R == 3 && p.S == 3 && p.chunk_stages >= p.nst && (p.debug & 16) == 0;
#define PSCONV_HALO_FAST(K, R)                                                                         \
  halo_mma_fast<BN, SPLIT3, PAIR, K, R>(p, smem, full, split_full, empty, acc_full, acc_empty, tmem_base, \
                                        cluster, nclusters, kIdesc)
#define PSCONV_HALO_TC(K, R)                                                                                 \
  halo_mma_fast<BN, SPLIT3, PAIR, K, R, true>(p, smem, full, split_full, empty, acc_full, acc_empty, tmem_base, \
                                              cluster, nclusters, kIdesc)
    bool issued = false;
    if constexpr (!SPLIT3 && BN <= 64) {
      if (p.tc) {  // tap concat: always the lean issuer (3x3, one chunk)
        if (p.b_res && p.kps == 4) PSCONV_HALO_TC(4, true);
        else if (p.b_res && p.kps == 2) PSCONV_HALO_TC(2, true);
        else if (p.b_res) PSCONV_HALO_TC(1, true);
        else if (p.kps == 4) PSCONV_HALO_TC(4, false);
        else if (p.kps == 2) PSCONV_HALO_TC(2, false);
        else PSCONV_HALO_TC(1, false);
        issued = true;
      }
    }
    if (issued) {
    } else if (fast && p.b_res && p.kps == 4) PSCONV_HALO_FAST(4, true);
    else if (fast && p.b_res && p.kps == 2) PSCONV_HALO_FAST(2, true);
    else if (fast && p.b_res && p.kps == 1) PSCONV_HALO_FAST(1, true);
    else if (fast && p.kps == 4) PSCONV_HALO_FAST(4, false);
    else if (fast && p.kps == 2) PSCONV_HALO_FAST(2, false);
    else if (fast && p.kps == 1) PSCONV_HALO_FAST(1, false);
#undef PSCONV_HALO_FAST
#undef PSCONV_HALO_TC
    else
      halo_mma<BN, SPLIT3, PAIR>(p, smem, full, split_full, empty, acc_full, acc_empty, tmem_base,
                                 cluster, nclusters, kIdesc);
  } else if (warp == 1 && leader) {
    // ------------------------------------------------------------ MMA issuer
    // Warp-uniform loop; one elected lane issues tcgen05.mma / commit.
    // Descriptors: A and B are K-major SW64 (64-B rows, 8-row groups 512 B
    // apart); K half h (channels 8h..8h+7) starts 32 B (2 x 16 B) into the row.
    const uint64_t desc0 = ptx::smem_desc_sw64(ptx::smem_u32(smem), 16, 512);
    // B: SW64 rows of one channel block, or (b128) SW128 rows of a block pair:
    // k-step j of the pair sits 64 B into the row, 8-row atoms 1024 B apart
    const uint64_t bdesc0 = p.b128 ? ptx::smem_desc_sw128(ptx::smem_u32(smem), 16, 1024) : desc0;
    const uint32_t bstep = static_cast<uint32_t>(Cfg::kBBytes * (ncat ? 2 : 1)) >> 4;  // B of one k-step
    const uint32_t b_even = p.b128 ? 4u : bstep;                 // after an even j
    const uint32_t b_odd = p.b128 ? (2u * bstep - 4u) : bstep;
    constexpr uint32_t kIdesc2 = ptx::idesc_tf32_m128<(BN <= 128 ? 2 * BN : BN), 128 * CS>();
    const uint32_t stage_desc = static_cast<uint32_t>(p.stage_bytes) >> 4;
    const uint32_t a_step = static_cast<uint32_t>(p.a_pitch) >> 4;  // next k-step's A tile
    const uint32_t alo_off = static_cast<uint32_t>(p.a_lo_off) >> 4;
    const uint32_t b_off = static_cast<uint32_t>(p.b_off) >> 4;
    const uint32_t blo_off = static_cast<uint32_t>(p.b_lo_off) >> 4;
    const int kps = p.kps;
    const bool skip_mma = (p.debug & 2) != 0;
    int stage = 0, gs = 0;
    int aslot = 0;  // TMEM A ring position (3xTF32 tmem_a)
    uint32_t phase = 0;
    int cit = 0;  // chunk counter across tiles -> accumulator buffer / phase
    for (int u = cluster; u < p.units; u += nclusters) {
      const Unit un = decode_unit<EPI == kEpiSplit>(p, u);
      const int unchunks =
          EPI != kEpiSplit || un.sp < 0 ? p.tile_chunks : (un.ie - un.ib + p.chunk_stages - 1) / p.chunk_stages;
      for (int c = 0; c < unchunks; ++c, ++cit) {
        const int buf = kAccBufs == 1 ? 0 : (cit & 1);
        const uint32_t acc_phase = (kAccBufs == 1 ? cit : (cit >> 1)) & 1;
        if (PAIR)
          ptx::mbar_wait_cluster(&acc_empty[buf], acc_phase ^ 1);
        else
          ptx::mbar_wait(&acc_empty[buf], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(buf * Cfg::kAccW);
        const int it0 = un.ib + c * p.chunk_stages;
        const int it_end = min(un.ie, it0 + p.chunk_stages);
        for (int it = it0; it < it_end; ++it) {
          const bool tr = kTrace && p.trace != nullptr && blockIdx.x == 0 && gs < kTraceStages;
          if (tr) p.trace[4 * kTraceStages + gs * 4 + 0] = clock64();
          ptx::mbar_wait(&full[stage], phase);  // PAIR: both CTAs' loads landed
          if (tr) p.trace[4 * kTraceStages + gs * 4 + 3] = clock64();
          if (SPLIT3) ptx::mbar_wait(&split_full[stage], phase);
          ptx::tc_fence_after();
          if (tr) p.trace[4 * kTraceStages + gs * 4 + 1] = clock64();
          const int nk = min(kps, p.ksteps - it * kps);  // partial last stage (cb_group = 0)
          if (ptx::elect_one()) {
            uint64_t da = desc0 + static_cast<uint64_t>(stage) * stage_desc;
            uint64_t db = bdesc0 + static_cast<uint64_t>(stage) * stage_desc + b_off;
            uint32_t acc_in = it == it0 ? 0u : 1u;
            int aslot_j = aslot;  // (state lives outside the elected lane: any lane may be elected)
            for (int j = 0; j < nk && (!skip_mma || p.tmem_a); ++j) {
              if constexpr (SPLIT3 && BN <= 128) {
                if (p.tmem_a) {  // A_hi / A_lo from the TMEM slot of this k-step
                  const uint32_t ah = tmem_base + static_cast<uint32_t>(p.a_slot_col + aslot_j * 32);
                  const uint64_t db_lo = db - b_off + blo_off;
                  if constexpr (F16) {  // A_hi at ah, A_lo at ah + 8; B_hi / B_lo = the row's K halves
                    if (!skip_mma) {
                      ptx::mma_f16_ts(d_tmem, ah + 8, db, kIdescF16, acc_in);  // A_lo B_hi (small first)
                      ptx::mma_f16_ts(d_tmem, ah, db + 2, kIdescF16, 1u);      // A_hi B_lo
                      ptx::mma_f16_ts(d_tmem, ah, db, kIdescF16, 1u);          // A_hi B_hi
                    }
                    acc_in = 1u;
                    ptx::mma_commit(&aslot_empty[aslot_j]);
                    if (++aslot_j == p.a_slots) aslot_j = 0;
                    da += a_step;
                    db += (j & 1) ? b_odd : b_even;
                    continue;
                  }
#ifdef PSCONV_DBG_PRINT
                  if (blockIdx.x == 0)
                    printf("mma it=%d j=%d stage=%d aslot=%d ah=%u db=%llx dblo=%llx acc_in=%u d=%u\n", it, j, stage, aslot_j,
                           ah, (unsigned long long)db, (unsigned long long)db_lo, acc_in, d_tmem);
#endif
                  if (ncat) {
#pragma unroll
                    for (int h = 0; h < 2 && !skip_mma; ++h) {
                      ptx::mma_tf32_ts(d_tmem, ah + h * 8, db + h * 2, kIdesc2, acc_in);  // -> D1 | D2
                      ptx::mma_tf32_ts(d_tmem, ah + 16 + h * 8, db + h * 2, kIdesc, 1u);  // A_lo B_hi -> D1
                      acc_in = 1u;
                    }
                  } else {
#pragma unroll
                    for (int h = 0; h < 2 && !skip_mma; ++h) {
                      ptx::mma_tf32_ts(d_tmem, ah + 16 + h * 8, db + h * 2, kIdesc, acc_in);  // small terms first
                      ptx::mma_tf32_ts(d_tmem, ah + h * 8, db_lo + h * 2, kIdesc, 1u);
                      ptx::mma_tf32_ts(d_tmem, ah + h * 8, db + h * 2, kIdesc, 1u);
                      acc_in = 1u;
                    }
                  }
                  ptx::mma_commit(&aslot_empty[aslot_j]);
                  if (++aslot_j == p.a_slots) aslot_j = 0;
                  da += a_step;
                  db += (j & 1) ? b_odd : b_even;
                  continue;
                }
              }
              if constexpr (F16) {  // one K = 16 step: A (hi|lo) and B (hi|lo) rows, lo at +32 B
                const uint64_t da16 = da + alo_off;
                ptx::mma_f16(d_tmem, da16 + 2, db, kIdescF16, acc_in);  // A_lo B_hi (small terms first)
                ptx::mma_f16(d_tmem, da16, db + 2, kIdescF16, 1u);      // A_hi B_lo
                ptx::mma_f16(d_tmem, da16, db, kIdescF16, 1u);          // A_hi B_hi
                acc_in = 1u;
                da += a_step;
                db += (j & 1) ? b_odd : b_even;
                continue;
              }
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                if (ncat) {
                  ptx::mma_tf32(d_tmem, da + h * 2, db + h * 2, kIdesc2, acc_in);        // -> D1 | D2
                  ptx::mma_tf32(d_tmem, da + alo_off + h * 2, db + h * 2, kIdesc, 1u);  // A_lo B_hi -> D1
                } else if (SPLIT3) {
                  const uint64_t da_lo = da + alo_off + h * 2;
                  const uint64_t db_lo = db - b_off + blo_off + h * 2;
                  ptx::mma_tf32(d_tmem, da_lo, db + h * 2, kIdesc, acc_in);  // small terms first
                  ptx::mma_tf32(d_tmem, da + h * 2, db_lo, kIdesc, 1u);
                  ptx::mma_tf32(d_tmem, da + h * 2, db + h * 2, kIdesc, 1u);
                } else if (PAIR) {
                  ptx::mma_tf32_pair(d_tmem, da + h * 2, db + h * 2, kIdesc, acc_in);
                } else {
                  ptx::mma_tf32(d_tmem, da + h * 2, db + h * 2, kIdesc, acc_in);
                }
                acc_in = 1u;
              }
              da += a_step;
              db += (j & 1) ? b_odd : b_even;
            }
            if (PAIR)
              ptx::mma_commit_pair(&empty[stage]);
            else
              ptx::mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (SPLIT3 && p.tmem_a) aslot = (aslot + nk) % p.a_slots;  // warp-uniform ring position
          if (tr) p.trace[4 * kTraceStages + gs * 4 + 2] = clock64();
          ++gs;
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (ptx::elect_one()) {
          if (PAIR)
            ptx::mma_commit_pair(&acc_full[buf]);
          else
            ptx::mma_commit(&acc_full[buf]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // second CTA of a pair: its loads complete on the leader's barrier and the
    // leader issues the pair MMAs; nothing to do here.
  } else if (warp == Cfg::kStoreWarp) {
    // ------------------------------------------------------------ store warp
    // Walks the epilogue's rounds in the same order (units, last chunk, 32-channel rounds
    // of both groups): waits for a staging slot to be filled, issues its TMA tensor
    // store(s) (reduce-add for `+=`), waits until the store has read the slot and hands it
    // back. Slots of split-K writer units carry no tile (out_skip).
    constexpr int DW = Cfg::kDrainW;
    constexpr int kBlk = DW / 16;
    const int kRounds = p.ostages / EG / kBlk;  // staging slots per epilogue group
    // os:8 -- deferred hand-back: up to `depth` (half the slots) bulk groups keep reading smem
    // while the epilogue fills the other half; a slot returns once `depth` younger groups are
    // committed (cp.async.bulk.wait_group.read depth). Default staging: one group at a time.
    const int depth = p.ostages > kOutStages ? (kRounds * EG) / 2 : 0;
    uint64_t fifo = 0u;  // committed slots, oldest in the low nibble
    int pending = 0;
    if (ptx::elect_one()) {
      ptx::prefetch_tmap(&tmap_out);
      int ost[2] = {0, 0};
      uint32_t oph[2] = {0u, 0u};
      const bool reduce = p.accumulate != 0;
      for (int u = cluster; u < p.units; u += nclusters) {
        const Unit un = decode_unit<EPI == kEpiSplit>(p, u);
        const TileCoord tc = decode_group(p, un.g, rank, CS);
        if (!tc.live) continue;
        const int q0 = tc.tq * p.Qb, p0 = tc.tp * p.Pb, n0 = tc.tn * p.Nb;
        const int kb0 = tc.tk * (BN / 16);
        for (int j = 0; j < BN / DW; ++j) {
          const int g = EG == 2 ? (j & 1) : 0;
          const int slot = g * kRounds + ost[g];
          ptx::mbar_wait(&out_full[slot], oph[g]);
          if (!out_skip[slot] && !(p.debug & 4)) {
            const uint8_t* st = out_stage + slot * (kBlk * Cfg::kOutStageBytes);
#pragma unroll
            for (int blk = 0; blk < kBlk; ++blk) {
              const int kb = kb0 + j * kBlk + blk;
              if (reduce)
                ptx::tma_reduce_add_5d(&tmap_out, st + blk * Cfg::kOutStageBytes, 0, q0, p0, kb, n0);
              else
                ptx::tma_store_5d(&tmap_out, st + blk * Cfg::kOutStageBytes, 0, q0, p0, kb, n0);
            }
            ptx::bulk_commit();
            if (depth == 0) {
              ptx::bulk_wait_read<0>();  // the slot's bytes are in flight to global memory
              ptx::mbar_arrive(&out_free[slot]);
            } else {
              fifo |= static_cast<uint64_t>(slot) << (4 * pending);
              if (++pending > depth) {
                switch (depth) {  // (an immediate operand)
                  case 1: ptx::bulk_wait_read<1>(); break;
                  case 2: ptx::bulk_wait_read<2>(); break;
                  case 3: ptx::bulk_wait_read<3>(); break;
                  case 4: ptx::bulk_wait_read<4>(); break;
                  case 6: ptx::bulk_wait_read<6>(); break;
                  default: ptx::bulk_wait_read<8>(); break;
                }
                while (pending > depth) {
                  ptx::mbar_arrive(&out_free[fifo & 15u]);
                  fifo >>= 4;
                  --pending;
                }
              }
            }
          } else {
            // a slot without a store (split-K writer unit): no younger group will push the
            // pending ones out, so drain them here (else the epilogue could wait on them forever)
            if (pending > 0) {
              ptx::bulk_wait_read<0>();
              for (; pending > 0; --pending, fifo >>= 4) ptx::mbar_arrive(&out_free[fifo & 15u]);
            }
            ptx::mbar_arrive(&out_free[slot]);
          }
          if (++ost[g] == kRounds) {
            ost[g] = 0;
            oph[g] ^= 1u;
          }
        }
      }
      if (ev) ev[5] = clock64();  // last store issued
      ptx::bulk_wait_all();       // stores complete before smem is released
      if (ev) ev[6] = clock64();
    }
    __syncwarp();
  } else if (warp < 6 || (EG == 2 && warp >= (SPLIT3 ? 10 : 6))) {
    // ------------------------------------------------------------ epilogue
    constexpr int DW = Cfg::kDrainW;
    constexpr int kGroups = EG;
    const int egrp = warp < 6 ? 0 : 1;  // rounds j = egrp, egrp + kGroups, ...
    // Output path: each 16-channel block of the 128-pixel tile is staged in
    // shared memory (SWIZZLE_64B image of the TMA box, conflict-free 16-B
    // writes) and written by one TMA tensor store (full lines; pixels outside
    // the layer are clipped by TMA; `+=` semantics via TMA reduce-add).
    const int lane = threadIdx.x & 31;
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = quad * 32 + lane;
    // first thread of each group: traces, the split-K ticket
    const bool store_thread = threadIdx.x == (egrp == 0 ? 64 : (SPLIT3 ? 320 : 192));
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(quad * 32) << 16);
    const uint32_t acc_empty_leader = PAIR ? ptx::mapa(&acc_empty[0], 0) : 0u;
    // staged row of this lane: the tile row itself, or (halo) its pixel
    // (pr, q) = (row / hw, row % hw) packed at pitch Q; junk lanes (q >= Q or
    // pr >= Pb) stage nothing
    int srow = row;
    bool row_valid = true;
    if (p.halo) {
      // (staging pitch = the tile's Qb columns: Q for whole-row tiles, 33 - kw with tap concat)
      const int pr = row / p.hw, q = row - pr * p.hw;
      row_valid = q < p.Qb && pr < p.Pb;
      srow = pr * p.Qb + q;
    }
    const uint32_t row_off = static_cast<uint32_t>(srow) * 64u;
    const uint32_t row_swz = (static_cast<uint32_t>(srow) >> 1) & 3u;  // SW64: chunk ^= bits[7:8]
    int ostage = 0;      // this group's staging slot (round robin over kRounds)
    uint32_t oph = 0u;   // its phase (toggles when ostage wraps)
    float out_scale = 1.f;
    if constexpr (F16) {
      ptx::griddep_wait();
      out_scale = 1.f / (pow2_scale(*p.absmax_a) * pow2_scale(*p.absmax_b));
    }
    int cit = 0;
    [[maybe_unused]] int rtrace = 0;  // epilogue rounds traced (PSCONV_TRACE builds)
    for (int u = cluster; u < p.units; u += nclusters) {
      const Unit un = decode_unit<EPI == kEpiSplit>(p, u);
      const int unchunks =
          EPI != kEpiSplit || un.sp < 0 ? p.tile_chunks : (un.ie - un.ib + p.chunk_stages - 1) / p.chunk_stages;
      const TileCoord tc = decode_group(p, un.g, rank, CS);
      // split tile: ticket -> write the partial to the workspace, or (last ticket)
      // combine all partials in split order and store the tile (ConvParams::split_ctr)
      const bool split = EPI == kEpiSplit && un.sp >= 0 && tc.live;
      const int stile = split ? (un.g - p.split_from) * CS + rank : 0;
      int* const ctr = split ? p.split_ctr + 2 * stile : nullptr;
      float4* const ws = split ? reinterpret_cast<float4*>(p.split_ws) + static_cast<long long>(stile) * p.ksplit * (32 * BN)
                               : nullptr;
      bool fixer = false;
      for (int c = 0; c < unchunks; ++c, ++cit) {
        const int buf = kAccBufs == 1 ? 0 : (cit & 1);
        const uint32_t acc_phase = (kAccBufs == 1 ? cit : (cit >> 1)) & 1;
        const bool last = c == unchunks - 1;
#ifdef PSCONV_EPI_SLEEP
        ptx::mbar_wait_sleep(&acc_full[buf], acc_phase);
#else
        ptx::mbar_wait(&acc_full[buf], acc_phase);
#endif
        if (ev && store_thread && cit == 0) ev[4] = clock64();
        if (ev && threadIdx.x == 64 && cit < 32) p.trace[kTraceEpi + 2 * cit] = clock64();
        ptx::tc_fence_after();
        if (EPI == kEpiSplit && split && last) {
          // the unit's partial is complete: take a ticket; the last holder waits until the
          // other ksplit-1 units (all past their own ticket, so running) have written theirs
          if (threadIdx.x == 64) {
            const int t = ptx::atom_add_relaxed_gpu(ctr, 1);
            if (t == p.ksplit - 1)
              while (ptx::ld_acquire_gpu(ctr + 1) != p.ksplit - 1) {
              }
            *split_word = t;
          }
          ptx::named_bar(3, 128 * kGroups);
          fixer = *split_word == p.ksplit - 1;
          if (fixer) ptx::fence_acq_rel_gpu();
        }
        constexpr bool kTcCap = !SPLIT3 && BN <= 64;  // tap concat instantiations
        const int accw = (kTcCap && p.tc) ? 3 * BN : Cfg::kAccW;
        const uint32_t tacc = lane_base + static_cast<uint32_t>(buf * accw);
        const uint32_t tsum = lane_base + static_cast<uint32_t>(Cfg::kSumCol);
#pragma unroll 1
        for (int j = egrp; j < BN / DW; j += kGroups) {
          const bool rtr = ev && threadIdx.x == 64 && rtrace < 16;
          if (rtr) p.trace[kTraceEpiR + 5 * rtrace] = clock64();
          uint32_t v[DW];
          if constexpr (DW == 32) ptx::tmem_ld32(tacc + j * 32, v);
          else ptx::tmem_ld16(tacc + j * 16, v);
          // tap concat: D = [D_0 | D_1 | D_2] (ki taps); out[r] = D_0[r] + D_1[r+1] + D_2[r+2]
          // -- one output row per warp (halo pitch 32), so the row shifts are warp shuffles
          // (lanes 30-31 read their own values: junk columns)
          [[maybe_unused]] uint32_t t1[kTcCap ? DW : 1], t2[kTcCap ? DW : 1];
          if constexpr (kTcCap) {
            if (p.tc) {
              if constexpr (DW == 32) {
                ptx::tmem_ld32(tacc + BN + j * 32, t1);
                ptx::tmem_ld32(tacc + 2 * BN + j * 32, t2);
              } else {
                ptx::tmem_ld16(tacc + BN + j * 16, t1);
                ptx::tmem_ld16(tacc + 2 * BN + j * 16, t2);
              }
            }
          }
          if constexpr (Cfg::kAccW == 2 * BN) {
            if (ncat) {  // D1 + D2 (A_hi B_lo in its own accumulator)
              uint32_t v2[DW];
              if constexpr (DW == 32) ptx::tmem_ld32(tacc + BN + j * 32, v2);
              else ptx::tmem_ld16(tacc + BN + j * 16, v2);
              ptx::tmem_wait_ld();
              ptx::reg_fence(v);
              ptx::reg_fence(v2);
#pragma unroll
              for (int i = 0; i < DW; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) + __uint_as_float(v2[i]));
            }
          }
          if (SPLIT3 && c > 0) {
            uint32_t sacc[DW];
            if constexpr (DW == 32) ptx::tmem_ld32(tsum + j * 32, sacc);
            else ptx::tmem_ld16(tsum + j * 16, sacc);
            ptx::tmem_wait_ld();
            ptx::reg_fence(v);
            ptx::reg_fence(sacc);
#pragma unroll
            for (int i = 0; i < DW; ++i)
              v[i] = __float_as_uint(__uint_as_float(sacc[i]) + __uint_as_float(v[i]));
          } else {
            ptx::tmem_wait_ld();
            ptx::reg_fence(v);
          }
          if constexpr (kTcCap) {
            if (p.tc) {
              ptx::reg_fence(t1);
              ptx::reg_fence(t2);
#pragma unroll
              for (int i = 0; i < DW; ++i)
                v[i] = __float_as_uint(__uint_as_float(v[i]) +
                                       __uint_as_float(__shfl_down_sync(0xFFFFFFFFu, t1[i], 1)) +
                                       __uint_as_float(__shfl_down_sync(0xFFFFFFFFu, t2[i], 2)));
            }
          }
          if (rtr) p.trace[kTraceEpiR + 5 * rtrace + 1] = clock64();
          if (!last) {
            if constexpr (DW == 32) ptx::tmem_st32(tsum + j * 32, v);
            else ptx::tmem_st16(tsum + j * 16, v);
          } else if (tc.live) {
            bool store_round = true;  // false: a split-K writer unit (partial in the workspace)
            // fused epilogue on the finished sum: + bias[k], ReLU (the same
            // value for all lanes: broadcast loads through L1)
            if constexpr (F16) {  // undo the operand scales (exact powers of two)
#pragma unroll
              for (int i = 0; i < DW; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * out_scale);
            }
            if constexpr (EPI == kEpiSplit) {
              if (split) {
                // workspace slot layout per round: [DW/4][128 rows] float4s (coalesced per warp)
                const int wbase = j * (DW / 4) * 128 + row;
                // every unit writes its partial (the last ticket too: its sum then reads only
                // the workspace, in split order, and its registers stay free)
#pragma unroll
                for (int c4 = 0; c4 < DW / 4; ++c4)
                  __stcg(ws + un.sp * (32 * BN) + wbase + c4 * 128,
                         make_float4(__uint_as_float(v[4 * c4]), __uint_as_float(v[4 * c4 + 1]),
                                     __uint_as_float(v[4 * c4 + 2]), __uint_as_float(v[4 * c4 + 3])));
                if (!fixer) store_round = false;  // the slot is handed over empty
#pragma unroll 1
                for (int sp = 0; sp < (store_round ? p.ksplit : 0); ++sp) {  // v accumulates (own partial re-read)
#pragma unroll
                  for (int c4 = 0; c4 < DW / 4; ++c4) {
                    const float4 x = __ldcg(ws + sp * (32 * BN) + wbase + c4 * 128);
                    const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                      v[4 * c4 + e] = __float_as_uint(sp == 0 ? xs[e] : __uint_as_float(v[4 * c4 + e]) + xs[e]);
                  }
                }
              }
            }
            if constexpr (EPI == kEpiFused) {
            if (p.bias != nullptr) {
              const float* bj = p.bias + tc.tk * BN + j * DW;
#pragma unroll
              for (int i = 0; i < DW; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) + __ldg(bj + i));
            }
            if (p.relu) {
#pragma unroll
              for (int i = 0; i < DW; ++i) v[i] = __float_as_uint(fmaxf(__uint_as_float(v[i]), 0.f));
            }
            }
            // one staging round = the DW/16 blocks of this TMEM load: one
            // barrier pair and one bulk group per round, kOutStages/(DW/16)
            // rounds in flight
            constexpr int kBlk = DW / 16;
            const int kRounds = p.ostages / kGroups / kBlk;  // per group
            const int slot = egrp * kRounds + ostage;
            uint8_t* st = out_stage + slot * (kBlk * Cfg::kOutStageBytes);
            ptx::mbar_wait(&out_free[slot], oph ^ 1u);  // the slot's previous store has read it
            if (rtr) p.trace[kTraceEpiR + 5 * rtrace + 2] = clock64();
            if (row_valid && store_round) {
#pragma unroll
              for (int blk = 0; blk < kBlk; ++blk) {
#pragma unroll
                for (int c4 = 0; c4 < 4; ++c4) {
                  const int b = blk * 16 + 4 * c4;
                  const uint32_t off = row_off + ((static_cast<uint32_t>(c4) ^ row_swz) << 4);
                  *reinterpret_cast<uint4*>(st + blk * Cfg::kOutStageBytes + off) =
                      make_uint4(v[b + 0], v[b + 1], v[b + 2], v[b + 3]);
                }
              }
            }
            ptx::fence_proxy_async_smem();
            if (store_thread) out_skip[slot] = store_round ? 0 : 1;
            ptx::mbar_arrive(&out_full[slot]);  // the store warp issues the TMA store(s)
            if (rtr) p.trace[kTraceEpiR + 5 * rtrace + 3] = clock64();
            if (++ostage == kRounds) {
              ostage = 0;
              oph ^= 1u;
            }
            if (rtr) p.trace[kTraceEpiR + 5 * rtrace + 4] = clock64();
          }
          if (kTrace) ++rtrace;
        }
        if (!last) ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (ev && threadIdx.x == 64 && cit < 32) p.trace[kTraceEpi + 2 * cit + 1] = clock64();
        if (ptx::elect_one()) {
          if (PAIR && !leader)
            ptx::mbar_arrive_remote(acc_empty_leader + 8u * buf);
          else
            ptx::mbar_arrive(&acc_empty[buf]);
        }
        __syncwarp();
      }
      if (EPI == kEpiSplit && split) {
        if (!fixer) {  // partial written by every epilogue thread -> count this unit done
          __threadfence();
          ptx::named_bar(3, 128 * kGroups);
          if (threadIdx.x == 64) ptx::red_release_gpu_add(ctr + 1, 1);
        } else {  // tile stored; reset the counters for the next launch (stream-ordered)
          ptx::named_bar(3, 128 * kGroups);
          if (threadIdx.x == 64) {
            ctr[0] = 0;
            ctr[1] = 0;
          }
        }
      }
    }
  } else if (SPLIT3 && warp < 10) {
    // ------------------------------------------------------------ splitter
    // lo = x - trunc_tf32(x), exact in fp32 (the MMA reads x itself as hi).
    const int tid = threadIdx.x - 192;
    float a_scale = 1.f;
    if constexpr (F16) {
      ptx::griddep_wait();  // the input |max| comes from the preceding kernel
      a_scale = pow2_scale(*p.absmax_a);
    }
    int stage = 0;
    uint32_t phase = 0;
    if (p.halo) {
      // one split per halo tile (kps blocks x hr*hw rows), reused by all R*S taps
      const int n4 = (p.kps * p.a_tile) >> 4;
      for (int g = cluster; g < p.groups; g += nclusters)
        for (int cg = 0; cg < p.cbg; ++cg) {
          ptx::mbar_wait(&full[stage], phase);
          split_lo(reinterpret_cast<const float4*>(stage_base(stage)),
                   reinterpret_cast<float4*>(stage_base(stage) + p.a_lo_off), n4, tid);
          ptx::fence_proxy_async_smem();
          ptx::mbar_arrive(&split_full[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
    } else if (SPLIT3 && BN <= 128 && p.tmem_a) {
      // TMEM A: each thread owns one pixel row (TMEM lane = warp quadrant x 32 +
      // lane), reads its 16 channels from the swizzled smem tile and writes
      // hi = x (the MMA truncates) and lo = x - trunc(x) into a 32-column slot
      const int lane = threadIdx.x & 31;
      const int quad = (threadIdx.x >> 5) & 3;
      const int row = quad * 32 + lane;
      const uint32_t row_off = static_cast<uint32_t>(row) * 64u;
      const uint32_t row_swz = (static_cast<uint32_t>(row) >> 1) & 3u;
      const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(quad * 32) << 16);
      int slot = 0;
      uint32_t sph = 0;
      int gs = 0;
      for (int u = cluster; u < p.units; u += nclusters) {
        const Unit un = decode_unit<EPI == kEpiSplit>(p, u);
        for (int it = un.ib; it < un.ie; ++it, ++gs) {
          const bool tr = kTrace && p.trace != nullptr && blockIdx.x == 0 && tid == 0 && gs < kTraceStages;
          ptx::mbar_wait(&full[stage], phase);
          if (tr) p.trace[kTraceSplit + 2 * gs] = clock64();
          const int nk = min(p.kps, p.ksteps - it * p.kps);
          for (int j = 0; j < nk; ++j) {
            ptx::mbar_wait(&aslot_empty[slot], sph ^ 1);  // the MMAs of slot's last use retired
            ptx::tc_fence_after();
            const uint8_t* a = stage_base(stage) + j * p.a_pitch + row_off;
            if constexpr (F16) {
              // f16x2: the slot's first 16 columns = [hi halves 0..15 | lo halves 0..15],
              // two halves per 32-bit column (the kind::f16 A-from-TMEM layout)
              uint32_t v[16];
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) {
                const float4 x = *reinterpret_cast<const float4*>(a + ((static_cast<uint32_t>(c4) ^ row_swz) << 4));
                const float xs[4] = {x.x * a_scale, x.y * a_scale, x.z * a_scale, x.w * a_scale};
#pragma unroll
                for (int e = 0; e < 4; e += 2) {
                  const __half2 h = __floats2half2_rn(xs[e], xs[e + 1]);
                  const float2 hf = __half22float2(h);
                  const __half2 l = __floats2half2_rn(xs[e] - hf.x, xs[e + 1] - hf.y);
                  v[c4 * 2 + e / 2] = *reinterpret_cast<const uint32_t*>(&h);
                  v[8 + c4 * 2 + e / 2] = *reinterpret_cast<const uint32_t*>(&l);
                }
              }
              ptx::tmem_st16(lane_base + static_cast<uint32_t>(p.a_slot_col + slot * 32), v);
              if (++slot == p.a_slots) {
                slot = 0;
                sph ^= 1;
              }
              continue;
            }
            uint32_t hi[16], lo[16];
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              const uint4 x = *reinterpret_cast<const uint4*>(a + ((static_cast<uint32_t>(c4) ^ row_swz) << 4));
              const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                hi[c4 * 4 + e] = xs[e];
                lo[c4 * 4 + e] = __float_as_uint(__uint_as_float(xs[e]) -
                                                 __uint_as_float(xs[e] & 0xFFFFE000u));
              }
            }
            const uint32_t col = lane_base + static_cast<uint32_t>(p.a_slot_col + slot * 32);
#ifdef PSCONV_DBG_PRINT
            if (blockIdx.x == 0 && (row == 0 || row == 1))
              printf("split it=%d j=%d stage=%d slot=%d row=%d col=%u a0=%f a1=%f lo0=%e sb_off=%d\n", it, j, stage, slot, row,
                     col, __uint_as_float(hi[0]), __uint_as_float(hi[1]), __uint_as_float(lo[0]),
                     int(stage_base(stage) - smem));
#endif
            ptx::tmem_st16(col, hi);
            ptx::tmem_st16(col + 16, lo);
            if (++slot == p.a_slots) {
              slot = 0;
              sph ^= 1;
            }
          }
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
          ptx::mbar_arrive(&split_full[stage]);
          if (tr) p.trace[kTraceSplit + 2 * gs + 1] = clock64();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    } else {
    int gs = 0;
    for (int u = cluster; u < p.units; u += nclusters) {
      const Unit un = decode_unit<EPI == kEpiSplit>(p, u);
      for (int it = un.ib; it < un.ie; ++it, ++gs) {
        const bool tr = kTrace && p.trace != nullptr && blockIdx.x == 0 && tid == 0 && gs < kTraceStages;
        ptx::mbar_wait(&full[stage], phase);
        if (tr) p.trace[kTraceSplit + 2 * gs] = clock64();
        // A tiles of the stage: kps x a_pitch bytes (packed box image, or 8 KB
        // tiles); the lo region mirrors it (offsets are multiples of 512 B, so
        // the swizzle phase matches). Loads are batched 4 deep for ILP.
        const float4* a = reinterpret_cast<const float4*>(stage_base(stage));
        float4* alo = reinterpret_cast<float4*>(stage_base(stage) + p.a_lo_off);
        const int n4 = (min(p.kps, p.ksteps - it * p.kps) * p.a_pitch) >> 4;
        if constexpr (F16)
          split_f16(reinterpret_cast<const uint8_t*>(a), reinterpret_cast<uint8_t*>(alo), n4 >> 2, tid, a_scale);
        else
          split_lo(a, alo, n4, tid);
        ptx::fence_proxy_async_smem();
        ptx::mbar_arrive(&split_full[stage]);
        if (tr) p.trace[kTraceSplit + 2 * gs + 1] = clock64();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (PAIR) ptx::cluster_sync_all();  // no CTA leaves while the pair still uses it
  if (ev && threadIdx.x == 0) ev[7] = clock64();
  if (warp == 1) {
    ptx::tc_fence_after();
    if (PAIR)
      ptx::tmem_dealloc_pair(tmem_base, tmem_cols);
    else
      ptx::tmem_dealloc(tmem_base, tmem_cols);
  }
#endif
}

}  // namespace psconv
