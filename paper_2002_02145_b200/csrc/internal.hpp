// Internal host-side declarations shared by the C-ABI translation units.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "psconv.h"

namespace psconv {

// Error classes mirror the reference hierarchy (include/nestrank/common.hpp:10-36):
// ConfigError -> exit/status 2 (ConfigRejectedError, InvalidPermutationError,
// TileSizeNonPositiveError, ParseError ...), RuntimeError -> status 1.
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct RuntimeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);
void clear_last_error();

// Runs f, translating exceptions into status codes + conv_last_error().
template <typename F>
int guarded(F&& f) {
  try {
    clear_last_error();
    f();
    return PSCONV_OK;
  } catch (const ConfigError& e) {
    set_last_error(e.what());
    return PSCONV_ERR_CONFIG;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return PSCONV_ERR_RUNTIME;
  }
}

void validate_desc(conv_desc& d);  // throws ConfigError; fills ifh/ifw

// The reference loop names (presets.hpp:75-85) of the tunable outer loops.
enum LoopId { L_IMG = 0, L_OFM_TILE, L_IFM_TILE, L_OJ, L_KJ, L_KI, L_COUNT };
const char* loop_name(int id);
int loop_id(const std::string& name);  // -1 if unknown

// Reference recipe (variants.hpp:16-65) + the GPU clause.
struct Recipe {
  std::vector<std::string> perm;                              // listed loops, new order
  std::vector<std::pair<std::string, int64_t>> tiles;         // loop -> tile size
  int bn = 0;                                                 // 0 = selector decides
  int box_q = 0, box_p = 0, box_n = 0;                        // 0 = selector decides
  int stages = 0;                                             // informational
  int kg = 0;                                                 // k-steps per stage, 0 = auto
  int halo = 0;                                               // 1: halo mode (stride-1 R x S)
  int gm = -1;                                                // grouped raster block, -1 = auto
  int fold = 0;                                               // (c,s) fold: C real channels
  int ta = -1;                                                // TMEM-resident A: -1 auto, 0/1
  int ks = 0;                                                 // split-K units per tile, 0 = auto
  int kt = 0;                                                 // split-K scope: 0 tail wave, 1 all tiles
  int br = -1;                                                // halo: resident filter, -1 auto
  int chunk = 0;                                              // 0 = default (3x: 16 k-steps)
  int eg = 0;                                                 // epilogue warp groups, 0 = auto (1)
  int os = 0;                                                 // output staging blocks (4 or 8), 0 = default (4)
  int pp = 0;                                                 // parity-plane tap pairs: C real channels (<= 4)
  int tc = 0;                                                 // halo: the kw taps of a row concatenated on N
  int cs = 0;                                                 // cluster size, 0 = default
  bool has_gpu = false;
  static Recipe parse(const std::string& text);  // throws ConfigError
  std::string id() const;                        // reference grammar + ";gpu=..."
};

// A fully resolved GPU schedule.
struct Schedule {
  int order[L_COUNT];  // loop ids in execution order (outer -> inner), band excluded
  int bn;              // output channels per tile (64/128/256)
  int qb, pb, nb;      // pixel box (ofw x ofh x img) of one 128-row M tile
  int oj_tile;         // reference tile=oj:T (0 = untiled)
  int chunk;           // k-steps per TMEM accumulation chunk (0 = whole reduction)
  int cs;              // CTAs per cluster sharing (multicasting) the filter block
  int kps;             // k-steps (input-channel blocks) per pipeline stage
  int stages;          // pipeline stages in the shared-memory ring (halo: A ring)
  int halo = 0;        // halo mode: Pb whole output rows, input halo loaded once per block
  int m_block = 0;     // grouped raster block (M groups); 0 = the recipe's loop order
  int hb_stages = 0;   // halo: B-ring stages
  int b_res = 0;       // halo: whole filter slice resident in smem (one N tile), no B ring
  int br = -1;         // recipe request for b_res (-1 auto)
  int tmem_a = 0;      // 3xTF32, bn <= 128, not halo: A_hi/A_lo in TMEM (no A_lo smem region)
  int ta = -1;         // recipe request for tmem_a (-1 auto)
  int ksplit = 1;      // split-K: reduction split into ksplit work units per tile
  int split_all = 0;   // split every tile (zeroed output, all partials reduce-added)
                       // instead of only the last partial wave's (flag-ordered)
  int egroups = 1;     // epilogue warp groups draining alternate 32-channel rounds (1 or 2)
  int ostages = 4;     // output staging blocks of 8 KB (recipe os:8 -- 32 KB less ring, deferred
                       // staging-slot hand-back in the store warp; not halo)
  int pp = 0;          // few-channel kernel (conv_pp.cuh): C <= 4 real channels, tap pairs per MMA
  int tc = 0;          // halo tap concat (TF32, 3x3, bn == nOfm <= 64): one N = 3 bn MMA per filter row
                       // (the three ki taps share the A rows; the epilogue adds D_ki shifted by ki rows)
  int raster[3];       // {0 img, 1 ofm_tile, 2 oj} outer -> inner
  int kord[3];         // {0 ifm_tile, 1 kj, 2 ki} outer -> inner
  std::string recipe_id;
};

// Resolves a recipe (possibly partial) against a descriptor; throws ConfigError
// for illegal recipes (same checks as variants.hpp:186-228 plan_recipe).
Schedule resolve_schedule(const conv_desc& d, const Recipe& r, int mode, bool gpu = true);

// Shared-memory pipeline geometry (conv_kernel.cuh): k-steps per stage and ring depth.
constexpr int kSmemStageBudget = 227 * 1024 - 4 * 128 * 64 - 2048 - 1024;  // == conv_kernel.cuh kStageBudget
constexpr int kSmemMaxStages = 16;
int stage_bytes(const Schedule& s, int mode);  // bytes of one stage of s.kps k-steps
void plan_stages(const conv_desc& d, Schedule& s, int mode, int kg);  // throws ConfigError

// Halo-mode geometry (conv_kernel.cuh ConvParams::halo): padded row pitch hw,
// halo rows hr, byte sizes of one A stage (kps halo tiles + junk-row slack,
// A_lo mirror in 3xTF32) and one B stage (one tap over kps blocks; tap concat: one
// filter row's kw taps, kw * bn rows). Tap concat pitches the halo at 32 pixels so
// that each epilogue warp holds one output row (qb <= 33 - kw valid columns).
struct HaloGeom {
  int hw, hr, a_tile, a_lo_off, a_stage, b_lo_off, b_stage;
};
bool halo_eligible(const conv_desc& d);
void nest_recognise(const std::string& text, nest_info* out);  // nest.cpp, throws ConfigError
HaloGeom halo_geom(const conv_desc& d, const Schedule& s, int mode);

// Parity-plane tap-pair geometry (conv_pp.cuh, recipe pp:C): s*s input parity
// planes of PR x PC 16-B pixels per 8 x 16 output tile; taps sorted by operand
// address and paired per K=8 MMA (tap_b = -1: zero second half).
constexpr int kPpMaxMmaHost = 32;
struct PpGeom {
  int s, PR, PC, planes, plane_bytes, pitch, box_bytes, stage_bytes, lo_off, stages;
  int bn, nmma, tiles_k, b_bytes, smem_bytes;
  int a_off[kPpMaxMmaHost], a_lbo[kPpMaxMmaHost], tap_a[kPpMaxMmaHost], tap_b[kPpMaxMmaHost];
};
PpGeom pp_geom(const conv_desc& d, int bn, int mode);  // throws ConfigError

// Modes that split operands into hi/lo pieces (3xTF32, f16x2): same pipeline
// stage structure (a lo / f16 region beside the fp32 A tile, chunked TMEM sums).
inline bool split_mode(int mode) { return mode == PSCONV_MODE_3XTF32 || mode == PSCONV_MODE_F16X2; }

// Closed-form model (select.cpp).
struct ModelBreakdown {
  double us_total, us_tensor, us_hbm, us_l2, us_smem, us_epi;
  // per-resource times (us) of the SM-side pipeline: MMA issue, shared-memory
  // traffic, operand-row delivery (TMA/L2 requests) -- the pairwise ranker's
  // inputs together with us_hbm (dnnrank.cpp)
  double us_mma, us_smem_traffic, us_rows;
  double hbm_bytes, l2_bytes, flops_issued;
  int64_t m_tiles, tiles;
};
ModelBreakdown model_schedule(const conv_desc& d, const Schedule& s, int mode);
std::vector<Schedule> candidate_schedules(const conv_desc& d, int mode, int c_logical = 0);
// The four per-variant statistics of the pairwise ranker (mirrors VariantStats,
// dnnrank.hpp:17-24, with B200 resources instead of cache levels).
void model_stats(const conv_desc& d, const Schedule& s, int mode, double out[4]);

// emit.cpp
std::string emit_driver(const conv_desc& d, const Schedule& s);

}  // namespace psconv
