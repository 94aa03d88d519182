// Recipe grammar and recipe -> GPU schedule resolution.
//
// The recipe grammar is the reference's (include/nestrank/variants.hpp:16-65):
//   perm=ofm_tile,oj,ifm_tile,kj,ki;tile=oj:2
// extended with one optional clause for the GPU tile axes:
//   ;gpu=bn:128,box:8x8x2        (BN output channels; pixel box ofw x ofh x img)
// Validation follows plan_recipe (variants.hpp:186-228) with the same error
// classes; the conv nest has no order-constraining dependences (all 120
// orders of the five movable loops are legal), so the
// legality check reduces to the structural ones.
//
// GPU meaning of a recipe:
//   * relative order of the parallel loops {img, ofm_tile, oj} = tile
//     rasterisation order of the persistent scheduler (oi innermost);
//   * relative order of the reduction loops {ifm_tile, kj, ki} = k-step order;
//   * tile=oj:T  -> T output rows per 128-pixel tile (box P extent);
//     tile=img:T -> T images per tile; tile=ofm_tile:T -> BN = 16*T channels.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cctype>
#include <map>
#include <set>
#include <sstream>

#include "internal.hpp"

namespace psconv {

namespace {

std::vector<std::string> split_names(const std::string& s) {  // loopnest.hpp:317-329
  std::vector<std::string> out;
  std::string cur;
  for (char c : s) {
    if (c == ',' || std::isspace(static_cast<unsigned char>(c))) {
      if (!cur.empty()) {
        out.push_back(cur);
        cur.clear();
      }
    } else {
      cur += c;
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

int64_t parse_int(const std::string& s, const std::string& what) {
  try {
    size_t pos = 0;
    const long long v = std::stoll(s, &pos);
    (void)pos;
    return v;
  } catch (const std::logic_error&) {
    throw ConfigError("bad " + what + " '" + s + "'");
  }
}

bool is_band(const std::string& v) { return v == "oi" || v == "ofm" || v == "ifm"; }

}  // namespace

Recipe Recipe::parse(const std::string& text) {
  Recipe r;
  size_t pos = 0;
  while (pos < text.size()) {
    size_t end = text.find(';', pos);
    if (end == std::string::npos) end = text.size();
    const std::string part = text.substr(pos, end - pos);
    if (part.rfind("perm=", 0) == 0) {
      r.perm = split_names(part.substr(5));
    } else if (part.rfind("tile=", 0) == 0) {
      for (const std::string& item : split_names(part.substr(5))) {
        const size_t colon = item.find(':');
        if (colon == std::string::npos)
          throw ConfigError("bad tile entry '" + item + "' in recipe");
        const int64_t size = parse_int(item.substr(colon + 1), "tile size in recipe entry");
        r.tiles.emplace_back(item.substr(0, colon), size);
      }
    } else if (part.rfind("gpu=", 0) == 0) {
      r.has_gpu = true;
      for (const std::string& item : split_names(part.substr(4))) {
        const size_t colon = item.find(':');
        if (colon == std::string::npos) throw ConfigError("bad gpu entry '" + item + "' in recipe");
        const std::string key = item.substr(0, colon), val = item.substr(colon + 1);
        if (key == "bn") {
          r.bn = static_cast<int>(parse_int(val, "gpu bn"));
        } else if (key == "box") {
          int q = 0, p = 0, n = 0;
          if (std::sscanf(val.c_str(), "%dx%dx%d", &q, &p, &n) != 3)
            throw ConfigError("bad gpu box '" + val + "' (expected QxPxN)");
          r.box_q = q;
          r.box_p = p;
          r.box_n = n;
        } else if (key == "st") {
          r.stages = static_cast<int>(parse_int(val, "gpu stages"));
        } else if (key == "cl") {
          r.cs = static_cast<int>(parse_int(val, "gpu cluster size"));
          if (r.cs != 1 && r.cs != 2) throw ConfigError("gpu cl must be 1 (single CTA) or 2 (CTA pair)");
        } else if (key == "kg") {
          r.kg = static_cast<int>(parse_int(val, "gpu k-steps per stage"));
          if (r.kg != 1 && r.kg != 2 && r.kg != 4 && r.kg != 8)
            throw ConfigError("gpu kg must be 1, 2, 4 or 8");
        } else if (key == "ks") {
          r.ks = static_cast<int>(parse_int(val, "gpu split-K"));
          if (r.ks < 1 || r.ks > 64) throw ConfigError("gpu ks must be in [1, 64]");
        } else if (key == "br") {
          r.br = static_cast<int>(parse_int(val, "gpu resident filter"));
          if (r.br != 0 && r.br != 1) throw ConfigError("gpu br must be 0 or 1");
        } else if (key == "kt") {
          r.kt = static_cast<int>(parse_int(val, "gpu split-K scope"));
          if (r.kt != 0 && r.kt != 1) throw ConfigError("gpu kt must be 0 (tail wave) or 1 (all tiles)");
        } else if (key == "ta") {
          r.ta = static_cast<int>(parse_int(val, "gpu TMEM-resident A"));
          if (r.ta != 0 && r.ta != 1) throw ConfigError("gpu ta must be 0 or 1");
        } else if (key == "fold") {
          r.fold = static_cast<int>(parse_int(val, "gpu fold channels"));
          if (r.fold < 1 || r.fold > 8) throw ConfigError("gpu fold must be in [1, 8] (real input channels)");
        } else if (key == "gm") {
          r.gm = static_cast<int>(parse_int(val, "gpu raster group"));
          if (r.gm < 0) throw ConfigError("gpu gm must be >= 0");
        } else if (key == "halo") {
          r.halo = static_cast<int>(parse_int(val, "gpu halo"));
          if (r.halo != 0 && r.halo != 1) throw ConfigError("gpu halo must be 0 or 1");
        } else if (key == "tc") {
          r.tc = static_cast<int>(parse_int(val, "gpu tap concat"));
          if (r.tc != 0 && r.tc != 1) throw ConfigError("gpu tc must be 0 or 1");
        } else if (key == "pp") {
          r.pp = static_cast<int>(parse_int(val, "gpu parity-plane channels"));
          if (r.pp < 1 || r.pp > 4) throw ConfigError("gpu pp must be in [1, 4] (real input channels)");
        } else if (key == "eg") {
          r.eg = static_cast<int>(parse_int(val, "gpu epilogue groups"));
          if (r.eg != 1 && r.eg != 2) throw ConfigError("gpu eg must be 1 or 2");
        } else if (key == "os") {
          r.os = static_cast<int>(parse_int(val, "gpu output staging blocks"));
          if (r.os != 4 && r.os != 8 && r.os != 12 && r.os != 16) throw ConfigError("gpu os must be 4, 8, 12 or 16");
        } else if (key == "ch") {
          r.chunk = static_cast<int>(parse_int(val, "gpu chunk"));
          if (r.chunk < 1) throw ConfigError("gpu chunk must be positive");
        } else {
          throw ConfigError("unknown gpu recipe key '" + key + "'");
        }
      }
    } else if (!part.empty()) {
      throw ConfigError("unknown recipe clause '" + part + "'");
    }
    pos = end + 1;
  }
  return r;
}

std::string Recipe::id() const {
  std::string s = "perm=";
  for (size_t i = 0; i < perm.size(); ++i) s += (i ? "," : "") + perm[i];
  if (!tiles.empty()) {
    s += ";tile=";
    for (size_t i = 0; i < tiles.size(); ++i)
      s += (i ? "," : "") + tiles[i].first + ":" + std::to_string(tiles[i].second);
  }
  if (has_gpu) {
    s += ";gpu=bn:" + std::to_string(bn) + ",box:" + std::to_string(box_q) + "x" +
         std::to_string(box_p) + "x" + std::to_string(box_n);
    if (cs) s += ",cl:" + std::to_string(cs);
    if (halo) s += ",halo:1";
    if (tc) s += ",tc:1";
    if (gm >= 0) s += ",gm:" + std::to_string(gm);
    if (fold) s += ",fold:" + std::to_string(fold);
    if (ta >= 0) s += ",ta:" + std::to_string(ta);
    if (ks) s += ",ks:" + std::to_string(ks);
    if (kt) s += ",kt:" + std::to_string(kt);
    if (br >= 0) s += ",br:" + std::to_string(br);
    if (kg) s += ",kg:" + std::to_string(kg);
    if (eg) s += ",eg:" + std::to_string(eg);
    if (os) s += ",os:" + std::to_string(os);
    if (pp) s += ",pp:" + std::to_string(pp);
    if (chunk) s += ",ch:" + std::to_string(chunk);
  }
  return s;
}

// Best 128-row pixel box for a (Q, P, N) output grid: maximal useful-row
// fraction, then longest contiguous input run (qb), then taller boxes.
static void choose_box(int64_t Q, int64_t P, int64_t N, int64_t sh, int64_t sw, int fix_p,
                       int fix_n, int& qb, int& pb, int& nb) {
  double best_eff = -1;
  int bq = 1, bp = 1, bn = 1;
  const int64_t useful = Q * P * N;
  for (int p = 1; p <= 128 && p <= P; ++p) {
    if (fix_p && p != fix_p) continue;
    if (p * sh > 256) break;
    for (int q = 1; q * p <= 128 && q <= Q; ++q) {
      if (q * sw > 256) break;
      const int nmax = static_cast<int>(std::min<int64_t>(N, 128 / (q * p)));
      for (int n = nmax; n >= 1; --n) {
        if (fix_n && n != fix_n) continue;
        if (n > 256) continue;
        const int64_t tiles = ((Q + q - 1) / q) * ((P + p - 1) / p) * ((N + n - 1) / n);
        const double eff = double(useful) / double(tiles * 128);
        const bool better = eff > best_eff + 1e-12 ||
                            (eff > best_eff - 1e-12 && (q > bq || (q == bq && p > bp)));
        if (better) {
          best_eff = eff;
          bq = q;
          bp = p;
          bn = n;
        }
        break;  // largest n for this (q,p) that fits is best for efficiency
      }
    }
  }
  if (best_eff < 0) {  // fixed p/n infeasible: fall back to unconstrained
    if (fix_p || fix_n) return choose_box(Q, P, N, sh, sw, 0, 0, qb, pb, nb);
  }
  qb = bq;
  pb = bp;
  nb = bn;
}

Schedule resolve_schedule(const conv_desc& d, const Recipe& r, int mode, bool gpu) {
  (void)mode;
  if (gpu && d.gemm_block != 16) throw ConfigError("GPU path requires gemm_block == 16 (NCHW16c layout)");
  // --- plan_recipe (variants.hpp:186-228) structural checks
  std::map<std::string, int> pos;
  for (int i = 0; i < L_COUNT; ++i) pos[loop_name(i)] = i;
  std::set<std::string> seen;
  std::vector<int> listed;
  for (const std::string& v : r.perm) {
    auto it = pos.find(v);
    if (it == pos.end()) {
      if (is_band(v)) throw ConfigError("recipe permutes microkernel band loop '" + v + "'");
      throw ConfigError("recipe names unknown loop '" + v + "'");
    }
    if (!seen.insert(v).second) throw ConfigError("recipe lists loop '" + v + "' twice");
    listed.push_back(it->second);
  }
  std::vector<int> order(L_COUNT);
  for (int i = 0; i < L_COUNT; ++i) order[i] = i;
  std::vector<int> slots = listed;
  std::sort(slots.begin(), slots.end());
  for (size_t k = 0; k < slots.size(); ++k) order[slots[k]] = listed[k];

  std::map<std::string, int64_t> tile_of;
  for (const auto& [var, size] : r.tiles) {
    if (size <= 0)
      throw ConfigError("tile size for loop '" + var + "' must be positive");
    auto it = pos.find(var);
    if (it == pos.end()) {
      if (is_band(var)) throw ConfigError("recipe tiles microkernel band loop '" + var + "'");
      throw ConfigError("recipe tiles unknown loop '" + var + "'");
    }
    if (tile_of.count(var)) throw ConfigError("recipe tiles loop '" + var + "' twice");
    tile_of[var] = size;
  }

  Schedule s{};
  for (int i = 0; i < L_COUNT; ++i) s.order[i] = order[i];
  // raster: relative order of {img, ofm_tile, oj}; kord: of {ifm_tile, kj, ki}
  int nr = 0, nk = 0;
  for (int i = 0; i < L_COUNT; ++i) {
    const int l = order[i];
    if (l == L_IMG) s.raster[nr++] = 0;
    if (l == L_OFM_TILE) s.raster[nr++] = 1;
    if (l == L_OJ) s.raster[nr++] = 2;
    if (l == L_IFM_TILE) s.kord[nk++] = 0;
    if (l == L_KJ) s.kord[nk++] = 1;
    if (l == L_KI) s.kord[nk++] = 2;
  }

  s.oj_tile = tile_of.count("oj") ? static_cast<int>(tile_of["oj"]) : 0;
  if (!gpu) {
    Recipe canon;
    for (int i = 0; i < L_COUNT; ++i)
      if (order[i] != L_IMG || i != 0) canon.perm.push_back(loop_name(order[i]));
    for (const auto& t : r.tiles) canon.tiles.push_back(t);
    s.recipe_id = canon.id();
    return s;
  }
  // --- tile axes
  const int64_t K = d.nOfm;
  // f16x2: no halo variant; the few-channel kernel has no fp16 variant either, so an
  // f16x2 pp plan runs its 3xTF32 arithmetic (equally fp32-faithful)
  if (r.halo && mode == PSCONV_MODE_F16X2) throw ConfigError("gpu halo is not implemented for the f16x2 mode");
  if (r.pp) {
    // few-channel kernel (conv_pp.cuh): fixed 8 x 16 pixel tile, bn 64 or 128,
    // the whole reduction in one MMA chain of tap pairs
    if (r.fold) throw ConfigError("gpu pp and fold are exclusive");
    const int pbn = r.bn ? r.bn : (K % 128 == 0 ? 128 : 64);
    const PpGeom g = pp_geom(d, pbn, mode);  // validates
    s.pp = r.pp;
    s.bn = g.bn;
    s.qb = 8;
    s.pb = 16;
    s.nb = 1;
    s.cs = 1;
    s.kps = 1;
    s.stages = g.stages;
    s.chunk = 0;
    s.ksplit = 1;
    s.egroups = 1;
    Recipe canon;
    for (int i = 0; i < L_COUNT; ++i)
      if (order[i] != L_IMG || i != 0) canon.perm.push_back(loop_name(order[i]));
    for (const auto& t : r.tiles) canon.tiles.push_back(t);
    canon.has_gpu = true;
    canon.bn = s.bn;
    canon.box_q = 8;
    canon.box_p = 16;
    canon.box_n = 1;
    canon.pp = r.pp;
    s.recipe_id = canon.id();
    return s;
  }
  int bn = r.bn;
  if (tile_of.count("ofm_tile") && !bn) bn = static_cast<int>(16 * tile_of["ofm_tile"]);
  if (!bn) {
    for (int c : {256, 128, 64, 32, 16})
      if (K % c == 0) {
        bn = c;
        break;
      }
  }
  if (bn != 16 && bn != 32 && bn != 64 && bn != 128 && bn != 256)
    throw ConfigError("GPU tile: bn must be 16, 32, 64, 128 or 256 (got " + std::to_string(bn) + ")");
  if (K % bn != 0)
    throw ConfigError("GPU tile: nOfm=" + std::to_string(K) + " is not a multiple of bn=" +
                      std::to_string(bn));
  s.bn = bn;

  int fix_p = tile_of.count("oj") ? static_cast<int>(std::min<int64_t>(tile_of["oj"], d.ofh)) : 0;
  int fix_n = tile_of.count("img") ? static_cast<int>(std::min<int64_t>(tile_of["img"], d.nImg)) : 0;
  if (r.tc) {
    // tap concat (halo variant): a filter row's kw taps as one N = kw * bn MMA over
    // shared A rows; the halo is pitched at 32 pixels -- one output row per epilogue
    // warp, qb = 33 - kw columns -- so the epilogue's row shift by ki stays in a warp
    if (mode != PSCONV_MODE_TF32) throw ConfigError("gpu tc (tap concat) is a TF32 option");
    if (d.stride_h != 1 || d.stride_w != 1 || d.kh != 3 || d.kw != 3)
      throw ConfigError("gpu tc needs a 3x3 stride-1 layer");
    if (s.bn != K || s.bn > 64) throw ConfigError("gpu tc needs bn == nOfm <= 64 (one N tile, N = 3 bn <= 192)");
    if (r.halo == 0 && r.has_gpu && r.box_q) throw ConfigError("gpu tc implies halo mode (no box)");
    s.qb = static_cast<int>(std::min<int64_t>(33 - d.kw, d.ofw));
    s.pb = static_cast<int>(std::min<int64_t>(4, d.ofh));
    s.nb = 1;
    s.halo = 1;
    s.tc = 1;
  } else if (r.halo) {
    // halo mode: whole output rows of one image at the padded pitch hw
    if (!halo_eligible(d))
      throw ConfigError("GPU tile: halo mode needs stride 1, a filter larger than 1x1 and ofw + kw - 1 <= 128");
    const int hw = static_cast<int>(d.ofw + d.kw - 1);
    s.qb = static_cast<int>(d.ofw);
    s.pb = static_cast<int>(std::min<int64_t>(128 / hw, d.ofh));
    if (fix_p) s.pb = std::min(s.pb, fix_p);
    s.nb = 1;
    s.halo = 1;
  } else if (r.box_q || r.box_p || r.box_n) {
    s.qb = r.box_q;
    s.pb = r.box_p;
    s.nb = r.box_n;
    if (s.qb < 1 || s.pb < 1 || s.nb < 1 || s.qb * s.pb * s.nb > 128)
      throw ConfigError("GPU tile: box QxPxN must be positive with Q*P*N <= 128");
    if (s.qb * d.stride_w > 256 || s.pb * d.stride_h > 256 || s.nb > 256)
      throw ConfigError("GPU tile: box exceeds the TMA box limit (256 per dimension)");
  } else {
    if (fix_p > 128) fix_p = 128;
    choose_box(d.ofw, d.ofh, d.nImg, d.stride_h, d.stride_w, fix_p, fix_n, s.qb, s.pb, s.nb);
  }

  Recipe canon;
  for (int i = 0; i < L_COUNT; ++i)
    if (order[i] != L_IMG || i != 0) canon.perm.push_back(loop_name(order[i]));
  for (const auto& t : r.tiles) canon.tiles.push_back(t);
  canon.has_gpu = true;
  canon.bn = s.bn;
  canon.box_q = s.qb;
  canon.box_p = s.pb;
  canon.box_n = s.nb;
  canon.halo = s.halo;
  canon.tc = s.tc;
  canon.fold = r.fold;
  canon.ta = r.ta;
  s.ta = r.ta;
  s.br = r.br;
  canon.br = r.br;
  if (r.os > 4 && s.halo) throw ConfigError("GPU tile: os (deep output staging) is not available in halo mode");
  if (r.os > 4 && r.pp) throw ConfigError("GPU tile: os is not an option of the few-channel kernel (pp)");
  s.ostages = r.os > 4 ? r.os : 4;
  if (s.ostages == 12 && (r.eg == 2 || s.bn < 32))  // whole rounds per epilogue group
    throw ConfigError("GPU tile: os:12 needs one epilogue group and bn >= 32");
  // cluster size sharing the filter block: largest of {4, 2, 1} keeping >= 8-row pieces
  // cl:2 = CTA pair (tcgen05.mma.cta_group::2, M=256, each SM stages half of B);
  // TF32 only (see conv_kernel.cuh)
  s.cs = r.cs ? r.cs : (mode == PSCONV_MODE_TF32 ? 2 : 1);
  if (s.cs == 2 && split_mode(mode))
    throw ConfigError("GPU tile: the CTA pair (cl:2) is TF32-only; use cl:1 for 3xTF32 / f16x2");
  if (s.bn / s.cs < 8) throw ConfigError("GPU tile: bn / cluster size must be >= 8");
  canon.cs = s.cs;
  // TMEM accumulation chunk (3xTF32 numerics, see conv_kernel.cuh); tf32: whole reduction
  const int ksteps = static_cast<int>(d.nIfm / 16 * d.kh * d.kw);
  // bn 256 has a single TMEM chunk buffer (drain not overlapped): longer chunks
  // (error ~1.2e-7 per k-step of chunk, tools/chunk_sweep.py: ch 32 -> 3.5e-6)
  // 3xTF32 default: equal chunks of at most 16 k-steps, or 40 at bn 256 where
  // each chunk boundary stalls the MMA on the drain (measured cfg5: ch 72 / 36 /
  // 32 / 24 -> 1738 / 1775 / 1789 / 1815 us; 40 k-steps ~ 4.8e-6 relL2)
  // At bn <= 64 (TMEM-resident A, not halo) one chunk of up to 40 k-steps frees the running
  // sum's TMEM columns for two more A slots (conv_fwd.cu a_slot_col).
  int chunk_def = ksteps;
  if (split_mode(mode)) {
    const int cmax = (s.bn == 256 || (s.bn <= 64 && !s.halo)) ? 40 : 16;
    const int nch = (ksteps + cmax - 1) / cmax;
    chunk_def = (ksteps + nch - 1) / nch;
  }
  // (TF32 accumulates the whole reduction in one TMEM buffer: the chunk running
  // sum needs the 3xTF32 TMEM layout, so ch: is a 3xTF32-only key)
  if (r.chunk && !split_mode(mode)) throw ConfigError("gpu ch (accumulation chunk) is a 3xtf32 / f16x2 option");
  s.chunk = r.chunk ? r.chunk : chunk_def;
  if (s.chunk > ksteps) s.chunk = ksteps;
  plan_stages(d, s, mode, r.kg);
  // Tail split-K (wave quantisation): the tiles of the last partial wave are
  // split into ks stage ranges run as separate work units (each writes its
  // partial to the plan's workspace; the last to finish adds them in split order
  // and stores the tile: deterministic, no inter-CTA waits on non-running CTAs,
  // conv_kernel.cuh ConvParams::split_ctr). Auto: the ks in 1..8 (>= 4 stages
  // each) with the lowest modelled time, charging the per-unit refill/drain
  // and the extra output traffic (select.cpp); a split must win by 3%.
  {
    const int ksteps_all = static_cast<int>(d.nIfm / 16 * d.kh * d.kw);
    const int nst = (ksteps_all + s.kps - 1) / s.kps;
    const int64_t tq = (d.ofw + s.qb - 1) / s.qb, tp = (d.ofh + s.pb - 1) / s.pb,
                  tn = (d.nImg + s.nb - 1) / s.nb;
    const int cs = std::max(1, s.cs);
    const int64_t groups = (tq * tp * tn + cs - 1) / cs * (d.nOfm / s.bn);
    const int64_t clusters = 148 / cs;
    int best = 1;
    if (r.ks) {
      best = std::min(r.ks, nst);
    } else if (!s.halo && groups % clusters != 0) {
      double best_us = 1e300;
      for (int k = 1; k <= 8 && nst / k >= 4; ++k) {
        Schedule t = s;
        t.ksplit = k;
        const double us = model_schedule(d, t, mode).us_total;
        if (us < best_us * 0.97) {
          best_us = us;
          best = k;
        }
      }
    }
    s.ksplit = s.halo ? 1 : best;
    s.split_all = s.ksplit > 1 && r.kt == 1;
    canon.ks = (r.ks || s.ksplit > 1) ? s.ksplit : 0;  // shown when it splits
    canon.kt = s.split_all ? 1 : 0;
  }
  // Grouped raster (auto): when both the activation rows and the filter of all
  // tiles exceed the L2 share, a wave of 148 concurrent tiles should cover a
  // ~12 x 12 block of (M group, N tile) so A rows and B columns are reused in
  // L2 instead of being re-read from HBM per N tile (GEMM-like shapes).
  {
    const int64_t tq = (d.ofw + s.qb - 1) / s.qb, tp = (d.ofh + s.pb - 1) / s.pb,
                  tn = (d.nImg + s.nb - 1) / s.nb;
    const int64_t mgroups = (tq * tp * tn + std::max(1, s.cs) - 1) / std::max(1, s.cs);
    const int64_t tiles_k = d.nOfm / s.bn;
    const double a_bytes = 4.0 * d.nImg * d.nIfm * d.ifh * d.ifw;
    const double b_bytes = 4.0 * d.nOfm * d.nIfm * d.kh * d.kw * (mode == PSCONV_MODE_3XTF32 ? 2 : 1);  // f16x2: hi|lo in 4 B
    int gm = 0;
    if (tiles_k >= 4 && mgroups >= 24 && a_bytes > 48e6 && b_bytes > 24e6) gm = 12;
    s.m_block = r.gm >= 0 ? r.gm : gm;
    canon.gm = r.gm >= 0 ? r.gm : -1;
  }
  s.chunk = (s.chunk + s.kps - 1) / s.kps * s.kps;  // chunks hold whole stages
  canon.chunk = split_mode(mode) ? s.chunk : 0;
  canon.kg = r.kg ? s.kps : 0;
  s.egroups = r.eg ? r.eg : 1;
  canon.eg = s.egroups == 2 ? 2 : 0;
  canon.os = s.ostages > 4 ? s.ostages : 0;
  s.recipe_id = canon.id();
  return s;
}

int stage_bytes(const Schedule& s, int mode) {
  // f16x2: fp32 A tile + its fp16 hi|lo tile (64-B rows) + B rows of fp16 hi|lo (64 B)
  if (mode == PSCONV_MODE_F16X2) return s.kps * (128 * 64 * (s.tmem_a ? 1 : 2) + (s.bn / s.cs) * 64);
  const int mult = mode == PSCONV_MODE_3XTF32 ? 2 : 1;
  // TMEM-A stages hold A once (its lo part lives in TMEM) and B hi + lo
  if (s.tmem_a) return s.kps * (128 * 64 + (s.bn / s.cs) * 64 * 2);
  return s.kps * (128 * 64 + (s.bn / s.cs) * 64) * mult;
}

// One pipeline stage carries kps k-steps. When kps divides Cb they are kps
// consecutive input-channel blocks at one (kj, ki), loaded by one TMA box per
// operand (conv_fwd.cu; the A box is split per block when its rows are not
// whole 8-row swizzle atoms); otherwise kps consecutive k-steps of the
// reduction order with one box each (e.g. the stem, Cb = 1). Auto: the largest
// of {4, 2} that keeps >= 3 stages in the ring, preferring divisors of Cb.
bool halo_eligible(const conv_desc& d) {
  return d.stride_h == 1 && d.stride_w == 1 && d.kh * d.kw > 1 && d.ofw + d.kw - 1 <= 128 &&
         d.ofh + d.kh - 1 <= 256;
}

HaloGeom halo_geom(const conv_desc& d, const Schedule& s, int mode) {
  HaloGeom h{};
  const int mult = mode == PSCONV_MODE_3XTF32 ? 2 : 1;
  h.hw = s.tc ? 32 : static_cast<int>(d.ofw + d.kw - 1);
  h.hr = s.pb + static_cast<int>(d.kh) - 1;
  h.a_tile = h.hr * h.hw * 64;
  // the last block's shifted operands read up to (kh-1)*hw + kw-1 + 127 rows in (tap
  // concat: the ki shift moves to the epilogue, the operands start at kj*hw)
  const int rows = (s.kps - 1) * h.hr * h.hw + static_cast<int>(d.kh - 1) * h.hw +
                   (s.tc ? 0 : static_cast<int>(d.kw - 1)) + 128;
  h.a_lo_off = (rows * 64 + 1023) / 1024 * 1024;
  h.a_stage = h.a_lo_off * mult;
  h.b_lo_off = s.kps * (s.bn / s.cs) * (s.tc ? static_cast<int>(d.kw) : 1) * 64;
  h.b_stage = h.b_lo_off * mult;
  return h;
}

void plan_stages(const conv_desc& d, Schedule& s, int mode, int kg) {
  const int Cb = static_cast<int>(d.nIfm / 16);
  // TMEM-resident A (3xTF32, bn <= 128, not halo): default at bn <= 64, where the
  // three MMAs per K-half are smem-read bound (cfg1 69.6 -> 56.8 us, l1 3x3 499 ->
  // 390 us); at bn 128 only 4 slots fit beside the accumulators (l2 3x3 312 ->
  // 339 us), so it is a tuner option there (recipe ta:1)
  {
    const bool ok = split_mode(mode) && s.bn <= 128 && !s.halo;
    const bool want = s.ta == 1 || (s.ta < 0 && s.bn <= 64);
    s.tmem_a = (ok && want && std::getenv("PSCONV_NO_TMEMA") == nullptr) ? 1 : 0;
  }
  if (s.halo && s.br != 0 && d.nOfm == s.bn) {
    // resident filter (one N tile): the CTA's whole filter slice -- R*S*Cb/kps boxes
    // -- loaded once; the rest of the budget is A halo stages (>= 2, <= 8). The B
    // ring's per-tap round trip (<= 8 stages in flight over ~1-2 us of L2
    // latency) bounds the ringed halo mode; auto whenever it fits.
    for (int k : {4, 2, 1}) {
      if (kg && k != kg) continue;
      if (Cb % k) continue;
      Schedule t = s;
      t.kps = k;
      const HaloGeom h = halo_geom(d, t, mode);
      const int64_t bres = int64_t(s.tc ? d.kh : d.kh * d.kw) * (Cb / k) * h.b_stage;
      const int64_t left = kSmemStageBudget - bres;
      const int a = left > 0 ? static_cast<int>(std::min<int64_t>(8, left / h.a_stage)) : 0;
      if (a >= 2) {
        s.kps = k;
        s.stages = a;
        s.hb_stages = 1;
        s.b_res = 1;
        return;
      }
    }
    if (s.br == 1) throw ConfigError("GPU tile: resident filter (br:1) does not fit in shared memory");
  }
  if (s.br == 1 && !(s.halo && d.nOfm == s.bn))
    throw ConfigError("GPU tile: br:1 needs halo mode and a single N tile (bn == nOfm)");
  if (s.halo) {
    // A ring of 2 halo stages, the rest B stages (<= 8 each); largest kps in
    // {4, 2, 1} dividing Cb that leaves >= 3 B stages
    for (int k : {4, 2, 1}) {
      if (kg && k != kg) continue;
      if (Cb % k) continue;
      Schedule t = s;
      t.kps = k;
      const HaloGeom h = halo_geom(d, t, mode);
      const int hb = std::min(8, (kSmemStageBudget - 2 * h.a_stage) / h.b_stage);
      if (hb >= 3 || (k == 1 && hb >= 2) || (kg && hb >= 2)) {
        s.kps = k;
        s.stages = 2;
        s.hb_stages = hb;
        return;
      }
    }
    throw ConfigError("GPU tile: halo tile does not fit in shared memory");
  }
  const int ksteps = static_cast<int>(Cb * d.kh * d.kw);
  auto ring = [&](int k) {
    Schedule t = s;
    t.kps = k;
    return std::min(kSmemMaxStages, (kSmemStageBudget - (s.ostages - 4) * 8192) / stage_bytes(t, mode));
  };
  int kps = 1;
  if (kg) {
    if (kg > ksteps) throw ConfigError("GPU tile: kg=" + std::to_string(kg) + " exceeds the reduction");
    if (ring(kg) < 2) throw ConfigError("GPU tile: kg=" + std::to_string(kg) + " leaves < 2 stages");
    kps = kg;
  } else {
    for (int k : {4, 2})
      if (Cb % k == 0 && ring(k) >= 3) {
        kps = k;
        break;
      }
    if (kps == 1 && ksteps > 1)
      for (int k : {4, 2})
        if (k <= ksteps && ring(k) >= 3) {
          kps = k;
          break;
        }
  }
  s.kps = kps;
  s.stages = ring(kps);
}

}  // namespace psconv

namespace psconv {

PpGeom pp_geom(const conv_desc& d, int bn, int mode) {
  PpGeom g{};
  if (d.nIfm != 16 || d.gemm_block != 16) throw ConfigError("gpu pp needs nIfm = gemm_block = 16");
  if (d.stride_h != d.stride_w || d.stride_h < 1 || d.stride_h > 2)
    throw ConfigError("gpu pp needs equal strides of 1 or 2");
  if (bn != 64 && bn != 128) throw ConfigError("gpu pp needs bn 64 or 128");
  if (d.nOfm % bn) throw ConfigError("gpu pp: nOfm is not a multiple of bn");
  const int R = static_cast<int>(d.kh), S = static_cast<int>(d.kw), s = static_cast<int>(d.stride_h);
  if (R * S > 2 * kPpMaxMmaHost || R * S < 2) throw ConfigError("gpu pp needs 2..64 filter taps");
  g.s = s;
  g.bn = bn;
  g.PR = 16 + (R - 1) / s;
  g.PC = 8 + (S - 1) / s;
  g.planes = s * s;
  g.pitch = g.PC * 16;
  g.box_bytes = g.PR * g.PC * 16;
  g.plane_bytes = (g.box_bytes + 127) / 128 * 128;
  const bool split3 = mode != PSCONV_MODE_TF32;  // f16x2 plans use the 3xTF32 arithmetic here
  g.lo_off = g.planes * g.plane_bytes;
  g.stage_bytes = g.lo_off * (split3 ? 2 : 1);
  // taps sorted by operand address; pairs (t0, t1), (t2, t3), ... -- with an odd
  // count the lowest tap gets a zero-weight partner (the next tap, so every read
  // stays inside the loaded planes) and is paired again below
  std::vector<std::pair<int, int>> taps;  // (offset, tap index r*S + s)
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < S; ++c) {
      const int pl = (r % s) * s + (c % s);
      taps.emplace_back(pl * g.plane_bytes + (r / s) * g.pitch + (c / s) * 16, r * S + c);
    }
  std::sort(taps.begin(), taps.end());
  const int nt = static_cast<int>(taps.size());
  int i = 0, k = 0;
  if (nt % 2 == 1) {
    g.a_off[k] = taps[0].first;
    g.a_lbo[k] = nt > 1 ? taps[1].first - taps[0].first : 16;
    g.tap_a[k] = taps[0].second;
    g.tap_b[k] = -1;
    ++k;
    i = 1;
  }
  for (; i + 1 < nt; i += 2, ++k) {
    g.a_off[k] = taps[i].first;
    g.a_lbo[k] = taps[i + 1].first - taps[i].first;
    g.tap_a[k] = taps[i].second;
    g.tap_b[k] = taps[i + 1].second;
  }
  g.nmma = k;
  g.tiles_k = static_cast<int>(d.nOfm / bn);
  g.b_bytes = g.tiles_k * g.nmma * bn * 32;
  const int bres = (g.b_bytes * (split3 ? 2 : 1) + 1023) / 1024 * 1024;
  // (four 8 KB output staging blocks: eight, with three TMA stores in flight, measured no
  // faster on the stem -- TF32 299 -> 302 us, 3xTF32 352 -> 390 us with the plane ring cut to 2)
  const int fixed = bres + 4 * 128 * 64 + 1024 + 1024;
  const int avail = 227 * 1024 - fixed;
  g.stages = std::min(16, avail / g.stage_bytes);
  if (g.stages < 2)
    throw ConfigError("gpu pp: the resident filter leaves fewer than two plane stages in shared memory");
  g.smem_bytes = (g.stages * g.stage_bytes + 1023) / 1024 * 1024 + fixed;
  return g;
}

}  // namespace psconv
