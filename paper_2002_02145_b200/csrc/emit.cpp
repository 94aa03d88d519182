// Driver emission: the plan's outer loop nest as C text, in the text format the
// reference's emitter produces (emit.hpp:60-134; golden tests/golden/conv_identity.c),
// so a B200 plan can be diffed against the reference's own `emit --recipe` output.
//
// Built directly from the resolved Schedule (Schedule::order = the recipe's loop
// order; tiles from the canonical recipe id), in three steps:
//   1. levels(): one Level per emitted loop -- untiled loops and the tile loops of
//      tiled ones in the schedule's order, then the intra-tile loops in the same
//      order, just above the band (the placement apply_recipe gives, variants.hpp:
//      243-274);
//   2. a tile loop whose tile does not divide the trip count is "versioned": its
//      full tiles run in a for loop, the last partial tile in a block that pins the
//      tile index, and everything nested inside is written once per version with the
//      intra loop's bound switched to the trip count in the partial version;
//   3. an explicit work stack walks the levels (no recursion) and a Writer turns the
//      open/close events into indented lines.
#include <cstring>
#include <set>
#include <sstream>

#include "internal.hpp"

namespace psconv {
namespace {

// `k * v + c` in the reference's affine text form (coefficient first, `1 *` and
// `+ 0` omitted); only the shapes the conv driver needs (k >= 0, c >= 0).
std::string affine(int64_t k, const std::string& v, int64_t c) {
  if (k == 0 || v.empty()) return std::to_string(c);
  std::string s = (k == 1 ? std::string() : std::to_string(k) + " * ") + v;
  if (c > 0) s += " + " + std::to_string(c);
  return s;
}

struct Level {
  std::string var;
  int64_t trip = 0;     // untiled / tile loop: iterations
  // intra-tile loop of tile loop `outer`: var in [tile * outer, tile * outer + tile),
  // clipped to `trip` (the original extent) in the partial-tile version
  std::string outer;
  int64_t tile = 0;
  bool versioned = false;  // tile loop whose last tile is partial
  int64_t full = 0;        // its full tiles
};

class Writer {
 public:
  void line(const std::string& s) { out_ << std::string(2 * depth_, ' ') << s << '\n'; }
  void open(const std::string& s) {  // "<header> {"; a bare block for an empty header
    line(s.empty() ? "{" : s + " {");
    ++depth_;
  }
  void close() {
    --depth_;
    line("}");
  }
  std::string str() const { return out_.str(); }

 private:
  std::ostringstream out_;
  int depth_ = 0;
};

std::vector<Level> levels(const conv_desc& d, const Schedule& s) {
  const int64_t trips[L_COUNT] = {d.nImg, d.nOfm / d.gemm_block, d.nIfm / d.gemm_block, d.ofh, d.kh, d.kw};
  const Recipe r = Recipe::parse(s.recipe_id);  // tiles ride on the canonical id
  std::set<std::string> names = {"img", "ofm_tile", "ifm_tile", "oj", "kj", "ki", "oi", "ofm", "ifm"};
  std::vector<Level> outer, inner;
  for (int i = 0; i < L_COUNT; ++i) {
    const int id = s.order[i];
    Level l;
    l.var = loop_name(id);
    l.trip = trips[id];
    int64_t tile = 0;
    for (const auto& t : r.tiles)
      if (t.first == l.var) tile = t.second;
    if (tile == 0) {
      outer.push_back(l);
      continue;
    }
    Level t;  // the tile loop takes the loop's place
    t.var = l.var + "_t";
    while (names.count(t.var)) t.var += "_";
    names.insert(t.var);
    t.trip = (l.trip + tile - 1) / tile;
    t.versioned = l.trip % tile != 0;
    t.full = l.trip / tile;
    outer.push_back(t);
    l.outer = t.var;
    l.tile = tile;
    inner.push_back(l);
  }
  outer.insert(outer.end(), inner.begin(), inner.end());
  return outer;
}

}  // namespace

std::string emit_driver(const conv_desc& d, const Schedule& s) {
  const std::vector<Level> lv = levels(d, s);
  const std::string row = d.stride_h == 1 ? "oj + kj" : "oj * " + std::to_string(d.stride_h) + " + kj";
  const std::string call =
      "gemm_microkernel(&output[img][ofm_tile][oj][0][0], &filter[ofm_tile][ifm_tile][kj][ki][0][0], "
      "&input[img][ifm_tile][" + row + "][ki][0]);";
  Writer w;
  w.line("#pragma omp parallel for private(ofm_tile, ifm_tile, oj, kj, ki)");  // presets.hpp:125
  // Work items: enter a level (in the current version), or close a scope. The
  // partial-tile set records which versioned tile loops are in their last tile.
  struct Item {
    enum Kind { kEnter, kClose, kPartial, kUnpartial } kind;
    size_t level;
  };
  std::set<std::string> partial;
  std::vector<Item> work = {{Item::kEnter, 0}};
  while (!work.empty()) {
    const Item it = work.back();
    work.pop_back();
    if (it.kind == Item::kClose) {
      w.close();
      continue;
    }
    if (it.kind == Item::kPartial || it.kind == Item::kUnpartial) {
      const Level& t = lv[it.level];
      if (it.kind == Item::kUnpartial) {
        partial.erase(t.var);
        w.close();
        continue;
      }
      // the last, partial tile: a block pinning the tile index, the nest inside it again
      w.open("");
      w.line("const int " + t.var + " = " + std::to_string(t.full) + ";");
      partial.insert(t.var);
      work.push_back({Item::kUnpartial, it.level});
      work.push_back({Item::kEnter, it.level + 1});
      continue;
    }
    if (it.level == lv.size()) {
      w.line(call);
      continue;
    }
    const Level& l = lv[it.level];
    std::string lo = "0", hi = std::to_string(l.trip);
    if (!l.outer.empty()) {
      lo = affine(l.tile, l.outer, 0);
      hi = partial.count(l.outer) ? std::to_string(l.trip) : affine(l.tile, l.outer, l.tile);
    } else if (l.versioned) {
      hi = std::to_string(l.full);
    }
    w.open("for (int " + l.var + " = " + lo + "; " + l.var + " < " + hi + "; ++" + l.var + ")");
    // LIFO: the partial-tile version (if any) follows the for loop's closing brace
    if (l.versioned) work.push_back({Item::kPartial, it.level});
    work.push_back({Item::kClose, it.level});
    work.push_back({Item::kEnter, it.level + 1});
  }
  return w.str();
}

}  // namespace psconv

using namespace psconv;

extern "C" int64_t conv_emit_driver(const conv_desc* d_in, const char* recipe, char* buf, size_t len) {
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
