// Few-channel convolution forward (the ResNet-50 stem: C = 3 real channels in a
// 16-channel block, 7x7, stride 2) on sm_100a tensor cores, "parity-plane tap
// pairs" (recipe pp:C, C <= 4 real input channels).
//
// The reference nest is the same Fig. 5 nest as conv_kernel.cuh (presets.hpp:60-127);
// only the operand staging differs. With C <= 4, one tap's input channels are
// 16 B (4 fp32; channels >= C are zero in the caller's layout, and the packed
// filter zeroes them). A tcgen05 kind::tf32 MMA of K = 8 reads its A operand as
// two 16-B K halves LBO bytes apart (SWIZZLE_NONE K-major layout), so one MMA
// contracts TWO taps of 4 channels when the two taps' operand rows sit at a
// constant distance. That holds over parity planes of the input:
//   plane[pr][pc][i][j] = in[h0 + s*i + pr][w0 + s*j + pc]   (s = stride, TMA
//   element strides s, 16-B pixels = channels 0..3)
// tap (kj, ki) = (s*u + pr, s*v + pc) of output pixel (py, qx) of the tile is
//   plane[pr][pc][py + u][qx + v]
// so for a tile of Qb = 8 columns x 16 rows, the A operand of a tap is 16
// core-matrix groups (py) of 8 contiguous 16-B rows (qx), SBO = plane pitch --
// the planes themselves are the operand (no im2col, no folded copy). Taps are
// sorted by their plane address and paired: LBO = address difference. R*S taps
// -> ceil(R*S/2) MMAs per tile (7x7: 25), versus 49 16-channel k-steps of the
// plain kernel (or the fold pass + 14 k-steps of fold:C).
//
// Per tile the producer loads s*s plane boxes (for the stem 4 x 11 x 19 pixels
// x 16 B = 13.4 KB, every input pixel's 16 B read once per tile); the filter,
// prepacked per MMA as [kh][8-row group][8][16 B] blocks (pp_pack_filter), stays
// resident in shared memory. Roles: warp 0 TMA producer, warp 1 TMEM owner + MMA
// issuer, warps 2-5 epilogue (tcgen05.ld -> SW64 staging -> TMA store, as in
// conv_kernel.cuh), warps 6-9 (3xTF32) lo = x - trunc(x) of the planes.
#pragma once
#include <cstdint>
#include <cuda.h>

#include "sm100_ptx.cuh"

namespace psconv {

constexpr int kPpMaxMma = 32;  // R*S <= 64 taps

struct PpParams {
  int img_count, P, Q, s, ph, pw;
  int tiles_q, tiles_p, tiles_k, groups;
  int nmma;                     // MMAs (tap pairs) per tile
  int planes;                   // s * s
  int plane_bytes;              // PR * PC * 16 rounded up to 128
  int pitch;                    // PC * 16 (SBO of the A operand)
  int box_bytes;                // bytes one plane box delivers (PR * PC * 16)
  int stage_bytes;              // planes * plane_bytes (x2 with the lo planes in 3xTF32)
  int lo_off;                   // lo planes inside a stage
  int stages;
  int b_bytes;                  // resident filter (hi); lo follows in 3xTF32
  int a_off[kPpMaxMma];         // first tap's operand offset inside the plane region
  int a_lbo[kPpMaxMma];         // second tap - first tap (bytes, > 0)
  const float* bpack;           // packed filter in global memory (hi | lo)
  int accumulate;               // out += conv (TMA reduce-add)
};

template <int BN, bool SPLIT3>
struct PpCfg {
  static constexpr int kThreads = SPLIT3 ? 320 : 192;
  static constexpr int kOutBytes = 128 * 64;  // one 128-pixel x 16-channel staging block
  static constexpr int kOutBlocks = 4;        // two 32-channel rounds in flight
  // one MMA's B block: BN rows x 8 tf32 ([kh][BN/8][8][16 B]); 3xTF32 N-concat: 2 BN
  // rows, B_hi then B_lo, so A_hi x [B_hi;B_lo] is ONE N = 2 BN MMA (-> D1 | D2) and
  // A_lo x B_hi an N = BN MMA on the block's first half (-> D1); the epilogue adds D2
  static constexpr int kBRowsMma = SPLIT3 ? 2 * BN : BN;
  static constexpr int kMmaBBytes = kBRowsMma * 32;
  static constexpr int kAccW = SPLIT3 ? 2 * BN : BN;  // accumulator columns per buffer
  static constexpr int kTmemCols = 2 * kAccW < 32 ? 32 : 2 * kAccW;
  static_assert(BN == 64 || BN == 128, "BN");
};

template <int BN, bool SPLIT3>
__global__ void __launch_bounds__(PpCfg<BN, SPLIT3>::kThreads, 1)
    conv_pp_sm100(const __grid_constant__ PpParams p, const __grid_constant__ CUtensorMap tmap_in,
                  const __grid_constant__ CUtensorMap tmap_out) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  using Cfg = PpCfg<BN, SPLIT3>;
  constexpr uint32_t kIdesc = ptx::idesc_tf32_m128<BN, 128>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // (pointer arithmetic on the __shared__ array, not an integer round trip: the compiler
  // keeps the shared address space and emits STS/LDS instead of generic ST.E/LD.E)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  // [ring: stages x stage_bytes][resident B (hi | lo)][out staging][barriers]
  const int ring = (p.stages * p.stage_bytes + 1023) / 1024 * 1024;
  uint8_t* bres = smem + ring;
  const int bres_bytes = (p.b_bytes * (SPLIT3 ? 2 : 1) + 1023) / 1024 * 1024;
  uint8_t* out_stage = bres + bres_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(out_stage + Cfg::kOutBlocks * Cfg::kOutBytes);
  uint64_t* full = bars;                 // [16] planes landed
  uint64_t* split_full = bars + 16;      // [16] lo planes written (3xTF32)
  uint64_t* empty = bars + 32;           // [16] MMAs done with the stage
  uint64_t* acc_full = bars + 48;        // [2]
  uint64_t* acc_empty = bars + 50;       // [2]
  uint64_t* b_full = bars + 52;          // resident filter landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 53);

  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&split_full[s], 128);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&acc_full[a], 1);
      ptx::mbar_init(&acc_empty[a], 4);
    }
    ptx::mbar_init(b_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, Cfg::kTmemCols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ptx::griddep_launch_dependents();  // PDL: see conv_fwd_sm100
  const int tiles_pq = p.tiles_q * p.tiles_p;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (ptx::elect_one()) {
      ptx::prefetch_tmap(&tmap_in);
      ptx::griddep_wait();  // the packed filter / input come from earlier kernels (PDL)
      const uint32_t btot = static_cast<uint32_t>(p.b_bytes * (SPLIT3 ? 2 : 1));
      ptx::mbar_expect_tx(b_full, btot);
      for (uint32_t o = 0; o < btot; o += 32768u)
        ptx::bulk_load(bres + o, reinterpret_cast<const uint8_t*>(p.bpack) + o, min(32768u, btot - o), b_full);
      int stage = 0;
      uint32_t phase = 0;
      for (int g = blockIdx.x; g < p.groups; g += gridDim.x) {
        const int m = g / p.tiles_k;
        const int tq = m % p.tiles_q, tp = (m / p.tiles_q) % p.tiles_p, n = m / tiles_pq;
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        ptx::mbar_expect_tx(&full[stage], static_cast<uint32_t>(p.planes * p.box_bytes));
        uint8_t* sb = smem + stage * p.stage_bytes;
        const int w0 = tq * 8 * p.s - p.pw, h0 = tp * 16 * p.s - p.ph;
        for (int pl = 0; pl < p.planes; ++pl)
          ptx::tma_load_5d(sb + pl * p.plane_bytes, &tmap_in, &full[stage], 0, w0 + pl % p.s, h0 + pl / p.s, n, 0);
        if (++stage == p.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    ptx::mbar_wait(b_full, 0);
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint32_t bbase = ptx::smem_u32(bres);
    constexpr uint32_t kBLbo = (Cfg::kBRowsMma / 8) * 128;  // B block: [kh][rows/8 groups][8 rows][16 B]
    constexpr uint32_t kIdesc2 = ptx::idesc_tf32_m128<(SPLIT3 ? 2 * BN : BN), 128>();
    int stage = 0, t = 0;
    uint32_t phase = 0;
    for (int g = blockIdx.x; g < p.groups; g += gridDim.x, ++t) {
      const int tk = g % p.tiles_k;
      const int buf = t & 1;
      ptx::mbar_wait(&acc_empty[buf], ((t >> 1) & 1) ^ 1);
      ptx::mbar_wait(&full[stage], phase);
      if (SPLIT3) ptx::mbar_wait(&split_full[stage], phase);
      ptx::tc_fence_after();
      if (ptx::elect_one()) {
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(buf * Cfg::kAccW);
        const uint32_t a0 = sbase + static_cast<uint32_t>(stage * p.stage_bytes);
        const uint32_t b0 = bbase + static_cast<uint32_t>(tk * p.nmma * Cfg::kMmaBBytes);
        for (int i = 0; i < p.nmma; ++i) {
          const uint32_t ao = a0 + static_cast<uint32_t>(p.a_off[i]);
          const uint32_t lbo = static_cast<uint32_t>(p.a_lbo[i]);
          const uint64_t da = ptx::smem_desc_none(ao, lbo, static_cast<uint32_t>(p.pitch));
          const uint64_t db = ptx::smem_desc_none(b0 + static_cast<uint32_t>(i * Cfg::kMmaBBytes), kBLbo, 128u);
          if (SPLIT3) {
            const uint64_t da_lo =
                ptx::smem_desc_none(ao + static_cast<uint32_t>(p.lo_off), lbo, static_cast<uint32_t>(p.pitch));
            ptx::mma_tf32(d_tmem, da, db, kIdesc2, i > 0 ? 1u : 0u);  // A_hi x [B_hi;B_lo] -> D1 | D2
            ptx::mma_tf32(d_tmem, da_lo, db, kIdesc, 1u);            // A_lo x B_hi -> D1
          } else {
            ptx::mma_tf32(d_tmem, da, db, kIdesc, i > 0 ? 1u : 0u);
          }
        }
        ptx::mma_commit(&empty[stage]);
        ptx::mma_commit(&acc_full[buf]);
      }
      __syncwarp();
      if (++stage == p.stages) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ epilogue
    const int lane = threadIdx.x & 31;
    const int quad = warp & 3;
    const int row = quad * 32 + lane;  // = py * 8 + qx = the TMA output box row
    const bool store_thread = threadIdx.x == 64;
    const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(quad * 32) << 16);
    const uint32_t row_off = static_cast<uint32_t>(row) * 64u;
    const uint32_t row_swz = (static_cast<uint32_t>(row) >> 1) & 3u;  // SW64 staging
    if (store_thread) ptx::prefetch_tmap(&tmap_out);
    int ostage = 0, t = 0;
    for (int g = blockIdx.x; g < p.groups; g += gridDim.x, ++t) {
      const int tk = g % p.tiles_k, m = g / p.tiles_k;
      const int tq = m % p.tiles_q, tp = (m / p.tiles_q) % p.tiles_p, n = m / tiles_pq;
      const int buf = t & 1;
      ptx::mbar_wait(&acc_full[buf], (t >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t tacc = lane_base + static_cast<uint32_t>(buf * Cfg::kAccW);
#pragma unroll 1
      for (int j = 0; j < BN / 32; ++j) {
        uint32_t v[32];
        ptx::tmem_ld32(tacc + j * 32, v);
        if constexpr (SPLIT3) {  // D1 + D2
          uint32_t v2[32];
          ptx::tmem_ld32(tacc + BN + j * 32, v2);
          ptx::tmem_wait_ld();
          ptx::reg_fence(v);
          ptx::reg_fence(v2);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) + __uint_as_float(v2[i]));
        }
        ptx::tmem_wait_ld();
        ptx::reg_fence(v);
        uint8_t* st = out_stage + ostage * (2 * Cfg::kOutBytes);
        if (store_thread) ptx::bulk_wait_read<1>();  // this round's two blocks read out
        ptx::named_bar(1, 128);
#pragma unroll
        for (int blk = 0; blk < 2; ++blk)
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const int b = blk * 16 + 4 * c4;
            const uint32_t off = row_off + ((static_cast<uint32_t>(c4) ^ row_swz) << 4);
            *reinterpret_cast<uint4*>(st + blk * Cfg::kOutBytes + off) = make_uint4(v[b], v[b + 1], v[b + 2], v[b + 3]);
          }
        ptx::fence_proxy_async_smem();
        ptx::named_bar(1, 128);
        if (store_thread) {
          const int kb0 = tk * (BN / 16) + j * 2;
          if (p.accumulate) {
            ptx::tma_reduce_add_5d(&tmap_out, st, 0, tq * 8, tp * 16, kb0, n);
            ptx::tma_reduce_add_5d(&tmap_out, st + Cfg::kOutBytes, 0, tq * 8, tp * 16, kb0 + 1, n);
          } else {
            ptx::tma_store_5d(&tmap_out, st, 0, tq * 8, tp * 16, kb0, n);
            ptx::tma_store_5d(&tmap_out, st + Cfg::kOutBytes, 0, tq * 8, tp * 16, kb0 + 1, n);
          }
          ptx::bulk_commit();
        }
        ostage ^= 1;
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (ptx::elect_one()) ptx::mbar_arrive(&acc_empty[buf]);
      __syncwarp();
    }
    if (store_thread) ptx::bulk_wait_all();
  } else if (SPLIT3) {
    // ------------------------------------------------------------ splitter (planes -> lo planes)
    const int tid = threadIdx.x - 192;
    const int n4 = (p.planes * p.plane_bytes) >> 4;
    int stage = 0;
    uint32_t phase = 0;
    for (int g = blockIdx.x; g < p.groups; g += gridDim.x) {
      ptx::mbar_wait(&full[stage], phase);
      const float4* a = reinterpret_cast<const float4*>(smem + stage * p.stage_bytes);
      float4* lo = reinterpret_cast<float4*>(smem + stage * p.stage_bytes + p.lo_off);
      for (int i = tid; i < n4; i += 128) {
        const float4 x = a[i];
        float4 l;
        l.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
        l.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
        l.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
        l.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
        lo[i] = l;
      }
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(&split_full[stage]);
      if (++stage == p.stages) {
        stage = 0;
        phase ^= 1;
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
#endif
}

}  // namespace psconv
