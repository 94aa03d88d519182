// Schedule selector: the PolyScientist ranking step (paper §4, reference
// pipeline.hpp:61-92 rank_variants -> costrank.hpp:19-40 cost/rank_by_cost)
// re-expressed for B200.
//
// The reference costs a variant by exact per-dependence working sets placed
// greedily in a cache hierarchy (reuse.hpp:29-82, cachefit.hpp:157-183). That
// engine materialises every iteration point (intset.hpp:295-307) and cannot
// run at BASELINE sizes (~2,000 s / ~700 GB per variant for
// cfg1), so here each candidate is costed in closed form:
//   t = max(tensor-pipe time, L2->SMEM operand time, HBM time) + fixed costs
// where the working set that decides HBM re-reads is the L2 footprint of the
// tiles co-resident on the 148 SMs (the GPU analogue of Alg. 1's WS at the
// level the persistent scheduler's rasterisation order controls).
// Candidates are the reference's recipe space (the four loop orders of
// samples/variants/conv_orders.cfg, the oj row tile) crossed with the GPU tile
// axes (BN, pixel box); ranking is ascending cost with ties broken by id, as
// in rank_by_cost (costrank.hpp:31-40).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <tuple>

#include "internal.hpp"

namespace psconv {

namespace {
#ifndef EPI_FIX
#define EPI_FIX 800.0
#endif
#ifndef EPI_ROUND
#define EPI_ROUND 700.0
#endif
#ifndef EPI_TC
#define EPI_TC 1000.0
#endif
#ifndef EPI_EG
#define EPI_EG 1.2
#endif
#ifndef EPI_PAIR
#define EPI_PAIR 1.3
#endif

// B200 machine model. Peaks: defaults from an earlier pod's MEASURED_PEAKS.json;
// the Python layer loads this pod's file at import (conv_select_set_machine:
// HBM copy GB/s, tf32 = bf16 / 2); the rest are modelling constants (DESIGN.md
// §4) fitted to r01 measurements.
struct Machine {
  double sms = 148;
  double hbm_gbs = 6538.9;
  double l2_gbs = 20000.0;       // aggregate L2 slice read bandwidth (not binding in r01 data)
  double tf32_tflops = 811.4;    // dense tf32 tensor peak (derived)
  double l2_bytes = 100e6;       // usable share of the 126 MB L2
  double launch_us = 4.0;        // launch + prologue (TMEM alloc, barrier init)
  double tile_fill_us = 0.6;     // pipeline fill of the first k-steps of a tile
  double clock_ghz = 1.6;        // SM clock under sustained tensor load (power-capped)
  double port_bytes_per_cycle = 110.0;  // ~0.85 x 128 B/cycle L2->SMEM per SM
  double kstep_sync_cyc = 30.0;  // mbarrier round trips per k-step
  double drain_round_trip_cyc = 100.0;  // one 32-column TMEM drain step
  double row_requests_per_cycle = 0.75;  // TMA rows per cycle per SM, all SMs loading
};
Machine kB200{};  // set once, before any ranking (conv_select_set_machine)

struct Geo {
  int64_t N, C, K, H, W, P, Q, R, S, Cb, Kb;
};
Geo geo(const conv_desc& d) {
  return Geo{d.nImg, d.nIfm, d.nOfm, d.ifh, d.ifw, d.ofh, d.ofw, d.kh, d.kw, d.nIfm / 16, d.nOfm / 16};
}

// Paper's four §2 orders (reference samples/variants/conv_orders.cfg:3-6).
const char* kPerms[] = {"ofm_tile,ifm_tile,oj,kj,ki", "ifm_tile,ofm_tile,oj,kj,ki",
                        "oj,ofm_tile,ifm_tile,kj,ki", "kj,ki,oj,ofm_tile,ifm_tile"};

std::vector<std::tuple<int, int, int>> box_candidates(const conv_desc& d) {
  // enumerate boxes, keep the best few by useful-row fraction
  struct B {
    double eff;
    int q, p, n;
  };
  std::vector<B> all;
  const int64_t Q = d.ofw, P = d.ofh, N = d.nImg;
  for (int p = 1; p <= 128 && p <= P && p * d.stride_h <= 256; ++p)
    for (int q = 1; q * p <= 128 && q <= Q && q * d.stride_w <= 256; ++q) {
      const int n = static_cast<int>(std::min<int64_t>({N, 128 / (q * p), 256}));
      const int64_t tiles = ((Q + q - 1) / q) * ((P + p - 1) / p) * ((N + n - 1) / n);
      all.push_back({double(Q * P * N) / double(tiles * 128), q, p, n});
    }
  std::sort(all.begin(), all.end(), [](const B& a, const B& b) {
    if (std::fabs(a.eff - b.eff) > 1e-12) return a.eff > b.eff;
    if (a.q != b.q) return a.q > b.q;
    return a.p > b.p;
  });
  std::vector<std::tuple<int, int, int>> out;
  for (const B& b : all) {
    if (out.size() >= 4 || b.eff < all.front().eff - 0.15) break;
    out.emplace_back(b.q, b.p, b.n);
  }
  return out;
}

}  // namespace

ModelBreakdown model_schedule(const conv_desc& d, const Schedule& s, int mode) {
  const Machine& m = kB200;
  const Geo g = geo(d);
  // MMA work relative to TF32: 3xTF32 three K=8 products; f16x2 three K=16 f16
  // products (one f16 MMA of K=16 ~ one tf32 MMA of K=8)
  const double mult = mode == PSCONV_MODE_3XTF32 ? 3.0 : (mode == PSCONV_MODE_F16X2 ? 1.5 : 1.0);
  const bool x3 = mode == PSCONV_MODE_3XTF32;  // separate B_lo rows (f16x2 packs hi|lo per row)
  const int64_t tq = (g.Q + s.qb - 1) / s.qb, tp = (g.P + s.pb - 1) / s.pb,
                tn = (g.N + s.nb - 1) / s.nb, tk = g.K / s.bn;
  const int64_t mt = tq * tp * tn, tiles = mt * tk;
  const int64_t ksteps = g.Cb * g.R * g.S;
  const double per_sm = std::ceil(double(tiles) / m.sms);  // static round-robin waves

  ModelBreakdown b{};
  b.m_tiles = mt;
  b.tiles = tiles;
  if (s.pp) {
    // few-channel kernel (conv_pp.cuh): nmma tap-pair MMAs per tile (N=64: ~48
    // cycles each, N=128: 64), the planes' 16-B pixels read once (32-B sectors),
    // the filter resident; output written once
    const PpGeom pg = pp_geom(d, s.bn, mode);
    // per tap pair: TF32 one N = BN MMA; 3xTF32 (N-concat) one N = 2 BN + one N = BN
    auto mma_n = [](double n) { return std::max(n / 2.0, 48.0); };
    const double mma_cyc = pg.nmma * (mode == PSCONV_MODE_TF32 ? mma_n(s.bn) : mma_n(2.0 * s.bn) + mma_n(s.bn));
    b.us_mma = per_sm * mma_cyc / (m.clock_ghz * 1e3);
    b.us_tensor = b.us_mma;
    b.hbm_bytes = 32.0 * g.N * g.H * g.W + 4.0 * g.N * g.K * g.P * g.Q;
    b.us_hbm = b.hbm_bytes / (0.8 * m.hbm_gbs * 1e9) * 1e6;
    b.us_rows = per_sm * pg.planes * pg.PR * pg.PC / m.row_requests_per_cycle / (m.clock_ghz * 1e3);
    b.us_epi = 128.0 * s.bn * 4.0 / (64.0 * 1.8e9) * 1e6;
    const double hi = std::max({b.us_tensor, b.us_hbm, b.us_rows});
    const double lo = std::max(std::min(b.us_tensor, b.us_hbm), 1e-9);
    b.us_total = hi * std::pow(1.0 + std::pow(lo / hi, 4.0), 0.25) + m.launch_us + b.us_epi;
    b.flops_issued = 2.0 * tiles * 128.0 * s.bn * 8.0 * pg.nmma * mult;
    return b;
  }
  const double tile_flops = 2.0 * 128 * s.bn * 16.0 * ksteps * mult;
  b.flops_issued = tile_flops * tiles;

  // Per-SM k-step pipeline (cycles), fitted to r01 measurements (cfg5 tf32 /
  // 3xtf32, per-layer sweep): the MMA needs BN cycles per k-step (two
  // M=128,N=BN,K=8 tf32 MMAs at BN/2 cycles each; x3 for 3xTF32); the operand
  // delivery (A box + filter block, multicast or not, every CTA ingests all of
  // it) streams through the ~128 B/cycle L2->SMEM port at ~85%; the two
  // overlap imperfectly.
  // Shared memory (~128 B/cycle/SM, measured r01: the single-CTA loop runs at
  // exactly this rate) carries the tensor-core operand reads (each M=128,K=8
  // MMA reads 4 KB of A and BN*32 B of B; a CTA pair reads only its half of B),
  // the TMA writes and, in 3xTF32, the splitter's A -> A_lo pass.
  const int cs = std::max(1, s.cs);
  const double a_box = double(s.qb) * s.pb * s.nb * 64.0;
  const double b_rows = double(s.bn) / cs;
  // MMA: two K=8 MMAs per k-step (x3 for 3xTF32) of max(BN/2, 46) cycles each --
  // an M=128 tf32 MMA takes >= ~46 cycles whatever N (tools/probe_mma_rate.cu:
  // N=64 48, N=128 64, N=256 128 cycles)
  // 3xTF32 at BN <= 64 outside halo mode (N-concat): per K half one N = 2 BN MMA
  // (A_hi x [B_hi;B_lo]) + one N = BN MMA (A_lo x B_hi) instead of three N = BN
  const bool ncat = x3 && s.bn <= 64 && std::max(1, s.cs) == 1;
  double mma_cyc = ncat ? 2.0 * (std::max(double(s.bn), 46.0) + std::max(s.bn / 2.0, 46.0))
                        : 2.0 * mult * std::max(s.bn / 2.0, 46.0);
  // tap concat (TF32 halo, tc:1): one N = 3 bn MMA per filter row covers three taps
  if (s.tc) mma_cyc = 2.0 * std::max(1.5 * s.bn, 46.0) / 3.0;
  // TMEM-resident A: the splitter's tcgen05.st traffic slows the TS MMAs that read the
  // same tensor memory (tools/probe_kstep.cu: the N-concat k-step 192 -> ~296 cycles)
  if (x3 && s.tmem_a) mma_cyc *= 1.5;
  // Operand delivery is bounded by TMA/L2 row requests, not bytes: ~0.75 rows
  // per cycle per SM with every SM loading, for 64-B and 128-B rows alike
  // (tools/probe_tma_issue.cu). A rows are 64 B (NCHW16c pixels); filter rows
  // are 128 B when a stage pairs channel blocks (b128), halving their count.
  const bool b128 = s.kps % 2 == 0 && g.Cb % std::max(1, s.kps) == 0;
  double rows = double(s.qb) * s.pb * s.nb + b_rows * (x3 ? 2 : 1) * (b128 ? 0.5 : 1.0);
  double a_bytes = a_box;  // TMA writes of A per k-step
  if (s.halo) {
    // halo mode: the (Pb + R - 1) x (Q + S - 1) halo of a channel block is loaded
    // once for its R*S taps; the filter is resident (b_res: loaded once per CTA)
    // or streamed per tap through the B ring
    const double hw = s.tc ? 32.0 : double(g.Q + g.S - 1);
    const double halo_rows = double(s.pb + g.R - 1) * hw / (double(g.R) * g.S);
    rows = halo_rows + (s.b_res ? 0.0 : b_rows * (x3 ? 2 : 1) * (b128 ? 0.5 : 1.0));
    a_bytes = halo_rows * 64.0;
  }
  const double deliver_b = a_bytes + (s.halo && s.b_res ? 0.0 : b_rows * 64.0 * (x3 ? 2 : 1));
  // strided layers: every A row is an isolated 64-B pixel; boxes taking few pixels per
  // image spread the requests over many DRAM pages and the row delivery slows (r02 tuner
  // rows, l3 ds 1x1/s2: box 1x1x128 1.7x slower than 2x2x32)
  const double ppi = double(s.qb) * s.pb;  // pixels per image in the box
  const double a_rows = s.halo ? rows : double(s.qb) * s.pb * s.nb;
  const double a_eff = (d.stride_h > 1 || d.stride_w > 1) ? 0.5 + 0.5 * std::min(1.0, ppi / 4.0) : 1.0;
  const double del_cyc = (rows + a_rows * (1.0 / a_eff - 1.0)) / m.row_requests_per_cycle;
  // operand reads per k-step: 2 K-halves x (A 4 KB + B rows x 32 B) per MMA; with
  // TMEM-resident A (3xTF32) the MMAs read only B and the splitter reads A once
  const double tc_reads = 2.0 * mult * ((s.tmem_a ? 0.0 : 4096.0) + b_rows * 32.0);
  const double split_b = mult > 1 ? (s.tmem_a ? 8192.0 * 0.5 : 4096.0) : 0.0;
  // (the splitter's LSU traffic only partly competes with the async-proxy traffic)
  const double smem_cyc = 0.94 * (tc_reads + deliver_b + split_b) / 128.0;
  const double busy = std::max(mma_cyc, smem_cyc);
  const double other = std::min(mma_cyc, smem_cyc);
  double kstep_cyc = busy * std::pow(1.0 + std::pow(other / busy, 4.0), 0.25);
  // + per-stage issue cost (barrier round trip, TMA issue ~45 cycles each, MMA
  // commit) amortised over the stage's kps k-steps
  const double boxes = s.kps > 1 && g.Cb % s.kps == 0 ? 2.0 : 2.0 * std::max(1, s.kps);
  double stage_cyc = m.kstep_sync_cyc * 4 + 45.0 * boxes;
  if (s.halo) {
    // halo issuers (clock trace, l1 3x3 TF32): the generic one spends ~300 cycles
    // of bookkeeping per tap (kps k-steps); the lean 3x3 one (one chunk per tile)
    // issues a whole channel group (9 taps) per ~300 cycles, + a B-ring wait per
    // tap when the filter is not resident
    const bool fast = g.R == 3 && g.S == 3 && (s.chunk <= 0 || s.chunk >= ksteps);
    stage_cyc = fast ? (s.b_res ? 300.0 / 9.0 : 60.0) : 300.0;
  }
  // the CTA pair synchronises its two CTAs per stage (the leader waits for both CTAs'
  // loads): ~200 cycles a stage, which only the wide-N (MMA-bound) layers hide
  if (cs == 2) stage_cyc += 100.0;
  kstep_cyc = std::max(kstep_cyc, del_cyc) + stage_cyc / std::max(1, s.kps);
  const int chunk = s.chunk > 0 ? s.chunk : static_cast<int>(ksteps);
  const double nchunks = std::ceil(double(ksteps) / chunk);
  // 3xTF32 chunk drain: tcgen05.ld acc + sum, fadd, tcgen05.st, 32 columns per
  // round trip; hidden behind the next chunk unless TMEM holds a single
  // accumulator (bn 256)
  const double drain_cyc = (s.bn / 32.0) * m.drain_round_trip_cyc;
  const bool drain_exposed = mult > 1 && s.bn == 256;
  // Static round-robin over persistent clusters: W full waves of whole tiles,
  // then (tail split-K) the rem tiles of the last partial wave as ks units of
  // ksteps / ks each, with their own drain
  const int ks = std::max(1, s.ksplit);
  const int64_t clusters = m.sms / cs, groups = (mt + cs - 1) / cs * tk;
  // (kt:1 splits every tile: no whole-tile waves)
  const int64_t waves = s.split_all && ks > 1 ? 0 : groups / clusters, rem = groups - waves * clusters;
  const int kt = rem > 0 ? ks : 1;
  // Epilogue throughput (CTA-0 clock traces, r02): ~1000 cycles per 32-channel round
  // (TMEM load, staging, store-warp handoff; ~1300 with the tap-concat's three loads),
  // EG groups in parallel, ~+500 per round for every non-last 3xTF32 chunk (running
  // sum); double-buffered, so a tile costs max(mainloop, epilogue). The CTA pair couples
  // both CTAs' epilogues on one accumulator release (~1.3x when it binds).
  const double rounds = std::max(1.0, s.bn / 32.0);
  // deep output staging (os:8 / 12): the TMA stores' shared-memory reads overlap the next
  // rounds; A/B on the epilogue-bound TF32 1x1 layers (tools/refine_plans.py, r02): a tile's
  // rounds cost ~0.82x (os:8), ~0.78x (os:12+). Its price -- 32+ KB less ring, so fewer
  // k-steps per stage -- is already in s.kps / s.stages.
  const double os_f = s.ostages >= 12 ? 0.78 : (s.ostages >= 8 ? 0.82 : 1.0);
  const double epi_tile = (EPI_FIX + rounds * ((s.tc ? EPI_TC : EPI_ROUND) * os_f + (nchunks - 1.0) * 250.0)) /
                          (s.egroups == 2 ? EPI_EG : 1.0) * (cs == 2 ? EPI_PAIR : 1.0);
  const double main_tile = double(ksteps) * kstep_cyc;
  const double tile_cyc = std::max(main_tile, epi_tile) + (drain_exposed ? nchunks * drain_cyc : drain_cyc);
  // (a split unit also refills the pipeline (~1500 cycles) and writes its
  // 128 x BN fp32 partial to the workspace; the last unit of the tile then reads
  // all kt partials back in split order before its store (~64 B/cycle each way;
  // r01 A/B fit of the refill, conv_kernel.cuh ConvParams::split_ctr)
  const double split_cyc = 3000.0 + (1.0 + ks) * 128.0 * s.bn * 4.0 / 64.0;
  const double unit_cyc = std::max(double(ksteps) / kt * kstep_cyc, epi_tile) +
                          (drain_exposed ? nchunks / kt * drain_cyc : drain_cyc) + (kt > 1 ? split_cyc : 0.0);
  double tail_units = std::ceil(double(rem) * kt / clusters);
  // a partial wave of whole tiles runs faster than a full one (fewer SMs share
  // L2/HBM and the power budget): fitted to the r01 tail-split A/B timings
  // (l3/l4 layers at 1.3-2.7 waves, cfg5 at 21.2)
  if (kt == 1 && rem > 0) tail_units = 0.5 + 0.5 * double(rem) / clusters;
  b.us_tensor = (waves * tile_cyc + tail_units * unit_cyc) / (m.clock_ghz * 1e3);
  const double to_us = (waves + tail_units / kt) * double(ksteps) / (m.clock_ghz * 1e3);
  b.us_mma = mma_cyc * to_us;
  b.us_smem_traffic = smem_cyc * to_us;
  b.us_rows = del_cyc * to_us;
  b.l2_bytes = ksteps * (a_bytes + (s.halo && s.b_res ? 0.0 : s.bn * 64.0 * (x3 ? 2 : 1) / cs)) * tiles;
  b.us_l2 = b.l2_bytes / (m.l2_gbs * 1e9) * 1e6;
  (void)per_sm;

  // HBM: compulsory bytes + input re-reads when the rasterisation sweeps all
  // pixels once per output-channel tile and the input does not stay in L2.
  const double in_b = 4.0 * g.N * g.C * g.H * g.W;
  const double flt_b = 4.0 * g.K * g.C * g.R * g.S * (mult > 1 ? 3 : 1);  // + hi/lo copies
  const double out_b = 4.0 * g.N * g.K * g.P * g.Q;
  const bool ofm_outer = s.raster[0] == 1 || (s.raster[1] == 1 && s.raster[2] != 1 && s.raster[0] == 0 &&
                                              tn == 1);
  double in_reads = 1.0;
  if (ofm_outer && tk > 1 && in_b + flt_b > m.l2_bytes) in_reads = double(tk);
  // (1x1 strided layers touch 1 / (sh * sw) of the input)
  const double touched = (g.R == 1 && g.S == 1) ? 1.0 / (d.stride_h * d.stride_w) : 1.0;
  b.hbm_bytes = in_b * touched * in_reads + flt_b + out_b;
  // split-K: every unit of a split tile writes its partial to the workspace and the
  // last reads them all back (mostly in L2, partly written back to HBM)
  if (kt > 1) b.hbm_bytes += 0.5 * out_b * double(s.split_all ? groups : rem) / groups * kt;
  b.us_hbm = b.hbm_bytes / (0.8 * m.hbm_gbs * 1e9) * 1e6;  // ~80% of copy bandwidth sustained
  b.us_smem = 0;
  b.us_epi = 128.0 * s.bn * 4.0 / (64.0 * 1.8e9) * 1e6;  // one trailing tile's drain
  // SM-side and HBM-side times overlap imperfectly (soft max, p = 4)
  const double hi = std::max({b.us_tensor, b.us_l2, b.us_hbm});
  const double lo = std::max(std::min(b.us_tensor, b.us_hbm), 1e-9);
  b.us_total = hi * std::pow(1.0 + std::pow(lo / hi, 4.0), 0.25) + m.launch_us + m.tile_fill_us + b.us_epi +
               (mult > 1 ? 2.0 + 3.0 * flt_b / 3 / (m.hbm_gbs * 1e9) * 1e6 : 0.0);
  return b;
}

void model_stats(const conv_desc& d, const Schedule& s, int mode, double out[4]) {
  const ModelBreakdown b = model_schedule(d, s, mode);
  out[0] = b.us_mma;
  out[1] = b.us_smem_traffic;
  out[2] = b.us_rows;
  out[3] = b.us_hbm;
}

std::vector<Schedule> candidate_schedules(const conv_desc& d, int mode, int c_logical) {
  std::vector<Schedule> out;
  std::set<std::string> seen;
  std::vector<int> bns;
  for (int c : {256, 128, 64, 32, 16})
    if (d.nOfm % c == 0) bns.push_back(c);
  const auto boxes = box_candidates(d);
  for (const char* perm : kPerms)
    for (int bn : bns)
      for (const auto& [q, p, n] : boxes) {
        Recipe r = Recipe::parse(std::string("perm=") + perm);
        r.has_gpu = true;
        r.bn = bn;
        r.box_q = q;
        r.box_p = p;
        r.box_n = n;
        Schedule s = resolve_schedule(d, r, mode);
        if (seen.insert(s.recipe_id).second) out.push_back(s);
        // the same tile over the kernel's structural options, so that the model -- not a
        // hand-written list in the tuner -- ranks them: deep output staging (os:8, epilogue-
        // bound layers), the single CTA instead of the pair (TF32; HBM-bound K <= 64 layers),
        // TMEM-resident A at bn 128 (3xTF32)
        for (int os : {0, 8})
          for (int alt = 0; alt < 2; ++alt) {
            if (os == 0 && alt == 0) continue;  // the default above
            Recipe v = r;
            v.os = os;
            if (alt == 1) {
              if (mode == PSCONV_MODE_TF32) v.cs = 1;
              else if (split_mode(mode) && bn == 128) v.ta = 1;
              else continue;
            }
            try {
              Schedule sv = resolve_schedule(d, v, mode);
              if (seen.insert(sv.recipe_id).second) out.push_back(sv);
            } catch (const ConfigError&) {
              // (the smaller ring does not hold two stages at this bn)
            }
          }
      }
  // halo mode (stride-1 R x S > 1): its own tile shape (whole padded rows)
  if (halo_eligible(d))
    for (const char* perm : kPerms)
      for (int bn : bns) {
        Recipe r = Recipe::parse(std::string("perm=") + perm);
        r.has_gpu = true;
        r.bn = bn;
        r.halo = 1;
        try {
          Schedule s = resolve_schedule(d, r, mode);
          if (seen.insert(s.recipe_id).second) out.push_back(s);
        } catch (const ConfigError&) {
          // the halo tile does not fit at this bn
        }
      }
  // tap concat (TF32, 3x3 stride 1, nOfm <= 64: one N = 3 nOfm MMA per filter row),
  // single CTA and pair, one or two epilogue groups
  if (mode == PSCONV_MODE_TF32 && d.kh == 3 && d.kw == 3 && d.stride_h == 1 && d.stride_w == 1 &&
      d.nOfm <= 64)
    for (const char* perm : kPerms)
      for (int cs : {1, 2})
        for (int eg : {1, 2}) {
          Recipe r = Recipe::parse(std::string("perm=") + perm);
          r.has_gpu = true;
          r.bn = static_cast<int>(d.nOfm);
          r.tc = 1;
          r.cs = cs;
          r.eg = eg == 2 ? 2 : 0;
          try {
            Schedule s = resolve_schedule(d, r, mode);
            if (seen.insert(s.recipe_id).second) out.push_back(s);
          } catch (const ConfigError&) {
          }
        }
  // few-channel kernel (conv_pp.cuh): only when the caller asserts <= 4 real input channels
  if (c_logical > 0 && c_logical <= 4 && d.nIfm == 16)
    for (int bn : {64, 128}) {
      if (d.nOfm % bn) continue;
      Recipe r = Recipe::parse(std::string("perm=") + kPerms[1]);
      r.has_gpu = true;
      r.bn = bn;
      r.pp = c_logical;
      try {
        Schedule s = resolve_schedule(d, r, mode);
        if (seen.insert(s.recipe_id).second) out.push_back(s);
      } catch (const ConfigError&) {
        // (strides, taps or the resident filter rule it out)
      }
    }
  return out;
}

}  // namespace psconv

using namespace psconv;

extern "C" {

int conv_select_topk(const conv_desc* d_in, int mode, int k, char* buf, size_t len, double* us) {
  return conv_select_topk_ex(d_in, mode, 0, k, buf, len, us);
}

int conv_select_topk_ex(const conv_desc* d_in, int mode, int c_logical, int k, char* buf, size_t len, double* us) {
  int written = 0;
  const int rc = guarded([&] {
    if (!d_in || !buf || k < 1 || c_logical < 0) throw ConfigError("bad argument");
    conv_desc d = *d_in;
    validate_desc(d);
    auto cands = candidate_schedules(d, mode, c_logical);
    if (cands.empty()) throw ConfigError("no GPU schedule for this descriptor");
    std::vector<std::pair<double, std::string>> scored;
    for (const auto& s : cands) scored.emplace_back(model_schedule(d, s, mode).us_total, s.recipe_id);
    std::sort(scored.begin(), scored.end());
    std::string txt;
    for (int i = 0; i < k && i < static_cast<int>(scored.size()); ++i) {
      txt += (i ? "\n" : "") + scored[i].second;
      if (us) us[i] = scored[i].first;
      ++written;
    }
    if (txt.size() + 1 > len) throw ConfigError("buffer too small");
    std::memcpy(buf, txt.c_str(), txt.size() + 1);
  });
  return rc == PSCONV_OK ? written : -rc;
}

int conv_select_set_machine(const char* text) {
  return guarded([&] {
    if (!text) throw ConfigError("null machine text");
    Machine m = kB200;
    std::istringstream in(text);
    std::string line;
    int lineno = 0;
    while (std::getline(in, line)) {
      ++lineno;
      const size_t hash = line.find('#');
      if (hash != std::string::npos) line.resize(hash);
      std::istringstream ls(line);
      std::string key;
      double v = 0;
      if (!(ls >> key)) continue;
      if (!(ls >> v) || !(v > 0)) throw ConfigError("machine line " + std::to_string(lineno) + ": expected '<key> <positive number>'");
      if (key == "hbm_gbs") m.hbm_gbs = v;
      else if (key == "tf32_tflops") m.tf32_tflops = v;
      else if (key == "clock_ghz") m.clock_ghz = v;
      else if (key == "sms") m.sms = v;
      else if (key == "l2_bytes") m.l2_bytes = v;
      else throw ConfigError("machine line " + std::to_string(lineno) + ": unknown key '" + key + "'");
    }
    kB200 = m;
  });
}

double conv_model_us(const conv_desc* d_in, int mode, const char* recipe) {
  double us = -1;
  guarded([&] {
    if (!d_in) throw ConfigError("null descriptor");
    conv_desc d = *d_in;
    validate_desc(d);
    const Schedule s = resolve_schedule(d, Recipe::parse(recipe ? recipe : ""), mode);
    us = model_schedule(d, s, mode).us_total;
  });
  return us;
}

}  // extern "C"
