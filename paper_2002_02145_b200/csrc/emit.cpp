// Driver emission: renders a plan's outer loop nest as C text in the format of
// the reference emitter (include/nestrank/emit.hpp:60-134), so a plan can be
// diffed against the reference's golden driver (tests/golden/conv_identity.c)
// and against the reference's own `emit --recipe` output.
//
// Loop structure after a recipe follows apply_recipe (variants.hpp:230-284):
// permuted loops, tiled loops replaced in place by their tile loop, intra-tile
// loops hoisted just above the band in permuted order; a tile size that does
// not divide the trip count yields a full-tile loop plus a remainder block.
#include <cstring>
#include <map>
#include <set>
#include <sstream>

#include "internal.hpp"

namespace psconv {
namespace {

struct Affine {  // c0 + sum coef*var, printed like NamedExpr::str (loopnest.hpp:69-88)
  std::map<std::string, int64_t> terms;
  int64_t cst = 0;
  std::string str() const {
    std::string out;
    for (const auto& [v, c] : terms) {
      if (c == 0) continue;
      if (out.empty()) {
        if (c == -1) out += "-";
        else if (c != 1) out += std::to_string(c) + " * ";
      } else {
        out += c > 0 ? " + " : " - ";
        const int64_t a = c > 0 ? c : -c;
        if (a != 1) out += std::to_string(a) + " * ";
      }
      out += v;
    }
    if (out.empty()) return std::to_string(cst);
    if (cst > 0) out += " + " + std::to_string(cst);
    if (cst < 0) out += " - " + std::to_string(-cst);
    return out;
  }
};

struct ELoop {
  std::string var;
  Affine lower;
  std::vector<Affine> uppers;  // 2 uppers = remainder intra loop
};

std::string indent(int d) { return std::string(static_cast<size_t>(d) * 2, ' '); }

}  // namespace

std::string emit_driver(const conv_desc& d, const Schedule& s) {
  const int64_t trips[L_COUNT] = {d.nImg, d.nOfm / d.gemm_block, d.nIfm / d.gemm_block,
                                  d.ofh,  d.kh,                  d.kw};
  std::map<std::string, int64_t> tile_of;
  // Tiles are carried on the canonical recipe id; recover them from it.
  {
    const Recipe r = Recipe::parse(s.recipe_id);
    for (const auto& t : r.tiles) tile_of[t.first] = t.second;
  }
  std::set<std::string> taken = {"img", "ofm_tile", "ifm_tile", "oj", "kj", "ki", "oi", "ofm", "ifm"};
  std::vector<ELoop> loops, intra;
  for (int i = 0; i < L_COUNT; ++i) {
    const int l = s.order[i];
    const std::string var = loop_name(l);
    auto t = tile_of.find(var);
    if (t == tile_of.end()) {
      ELoop e;
      e.var = var;
      e.uppers.push_back(Affine{{}, trips[l]});
      loops.push_back(e);
      continue;
    }
    const int64_t tile = t->second;
    std::string tvar = var + "_t";
    while (taken.count(tvar)) tvar += "_";
    ELoop tl;
    tl.var = tvar;
    tl.uppers.push_back(Affine{{}, (trips[l] + tile - 1) / tile});
    loops.push_back(tl);
    ELoop il;
    il.var = var;
    il.lower.terms[tvar] = tile;
    Affine end = il.lower;
    end.cst += tile;
    il.uppers.push_back(end);
    if (trips[l] % tile != 0) il.uppers.push_back(Affine{{}, trips[l]});
    intra.push_back(il);
  }
  for (auto& l : intra) loops.push_back(l);

  const std::string sh = d.stride_h != 1 ? "oj * " + std::to_string(d.stride_h) + " + kj" : "oj + kj";
  const std::string call = "gemm_microkernel(&output[img][ofm_tile][oj][0][0], "
                           "&filter[ofm_tile][ifm_tile][kj][ki][0][0], &input[img][ifm_tile][" +
                           sh + "][ki][0]);";

  std::ostringstream os;
  os << "#pragma omp parallel for private(ofm_tile, ifm_tile, oj, kj, ki)\n";  // presets.hpp:125
  std::map<std::string, bool> rem_mode;
  auto is_rem = [](const ELoop& l) { return l.uppers.size() == 2; };
  auto tile_var_of = [](const ELoop& l) { return l.lower.terms.begin()->first; };
  auto rec = [&](auto&& self, size_t dpt, int depth) -> void {
    if (dpt == loops.size()) {
      os << indent(depth) << call << "\n";
      return;
    }
    const ELoop& l = loops[dpt];
    const std::string step = "++" + l.var;
    const ELoop* rem = nullptr;
    for (size_t j = dpt + 1; j < loops.size(); ++j)
      if (is_rem(loops[j]) && tile_var_of(loops[j]) == l.var) {
        rem = &loops[j];
        break;
      }
    if (rem) {
      const int64_t tile = rem->lower.terms.at(l.var);
      const int64_t full = (rem->uppers[1].cst - rem->lower.cst) / tile;
      os << indent(depth) << "for (int " << l.var << " = 0; " << l.var << " < " << full << "; "
         << step << ") {\n";
      rem_mode[l.var] = false;
      self(self, dpt + 1, depth + 1);
      os << indent(depth) << "}\n";
      os << indent(depth) << "{\n";
      os << indent(depth + 1) << "const int " << l.var << " = " << full << ";\n";
      rem_mode[l.var] = true;
      self(self, dpt + 1, depth + 1);
      rem_mode.erase(l.var);
      os << indent(depth) << "}\n";
      return;
    }
    std::string upper;
    if (is_rem(l)) {
      const bool r = rem_mode.count(tile_var_of(l)) && rem_mode.at(tile_var_of(l));
      upper = l.uppers[r ? 1 : 0].str();
    } else {
      upper = l.uppers[0].str();
    }
    os << indent(depth) << "for (int " << l.var << " = " << l.lower.str() << "; " << l.var << " < "
       << upper << "; " << step << ") {\n";
    self(self, dpt + 1, depth + 1);
    os << indent(depth) << "}\n";
  };
  rec(rec, 0, 0);
  return os.str();
}

}  // namespace psconv

using namespace psconv;

extern "C" int64_t conv_emit_driver(const conv_desc* d_in, const char* recipe, char* buf,
                                       size_t len) {
  int64_t need = -1;
  const int rc = guarded([&] {
    if (!d_in) throw ConfigError("null descriptor");
    conv_desc d = *d_in;
    validate_desc(d);
    const Schedule s = resolve_schedule(d, Recipe::parse(recipe ? recipe : ""), PSCONV_MODE_3XTF32, false);
    const std::string txt = emit_driver(d, s);
    need = static_cast<int64_t>(txt.size());
    if (buf && len) {
      const size_t n = txt.size() < len - 1 ? txt.size() : len - 1;
      std::memcpy(buf, txt.data(), n);
      buf[n] = 0;
    }
  });
  return rc == PSCONV_OK ? need : -rc;
}
