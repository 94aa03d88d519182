// REFERENCE INTERPRETER — TEST INFRASTRUCTURE ONLY (oracle pinning).
//
// Compiled from the reference's own headers where they lie
// (/root/reference/proj/include, header-only C++20) into oracle/_ref/ by
// oracle/build_ref.sh; never copied. It executes the reference IR numerically:
//   ConvPreset::parse(csv).build()            include/nestrank/presets.hpp:26-127
//   [apply_recipe(nest, VariantRecipe)]       include/nestrank/variants.hpp:230-284
//   oracle_detail::for_each_iteration         include/nestrank/oracle.hpp:22-43
// and at every iteration point evaluates the statement's ArrayRef subscripts
// (detail::SparseExpr, loopnest.hpp:732-749) to perform the body
//   output[...] += filter[...] * input[...]   presets.hpp:110-114
// in fp32 on caller arrays laid out exactly as the subscripts say
// (input pre-padded to the implied extent (ofh-1)*stride+kh, presets.hpp:88-91).
#include <cstdint>
#include <cstring>
#include <string>

#include "nestrank/emit.hpp"
#include "nestrank/oracle.hpp"
#include "nestrank/presets.hpp"
#include "nestrank/variants.hpp"

using namespace nestrank;

namespace {
thread_local std::string g_err;

struct Resolved {
  std::vector<detail::SparseExpr> idx;
  std::vector<std::int64_t> extent;
};

std::int64_t flat(const Resolved& r, const Point& x) {
  std::int64_t off = 0;
  for (std::size_t j = 0; j < r.idx.size(); ++j) off = off * r.extent[j] + r.idx[j].eval(x);
  return off;
}
}  // namespace

extern "C" {

const char* ref_interp_error() { return g_err.c_str(); }

// Returns the number of iteration points executed, or -1 on error.
std::int64_t ref_interp_conv(const char* csv10, const char* recipe, const float* in_padded,
                             const float* flt, float* out) {
  try {
    const ConvPreset p = ConvPreset::parse(csv10);
    LoopNest n = p.build();
    if (recipe && *recipe) n = apply_recipe(n, VariantRecipe::parse(recipe));
    const auto dim_index = detail::dim_index_of(n.loop_vars());
    const std::int64_t Hp = (p.ofh - 1) * p.stride_h + p.kh, Wp = (p.ofw - 1) * p.stride_w + p.kw;
    const std::int64_t B = p.gemm_block;
    auto resolve = [&](const ArrayRef& ref, std::vector<std::int64_t> ext) {
      Resolved r;
      for (const NamedExpr& e : ref.index_exprs) r.idx.push_back(detail::SparseExpr::from(e, dim_index));
      r.extent = std::move(ext);
      return r;
    };
    // stmt.reads = {output, filter, input} (presets.hpp:105)
    const Resolved ro = resolve(n.stmt.reads[0], {p.nImg, p.nOfm / B, p.ofh, p.ofw, B});
    const Resolved rf = resolve(n.stmt.reads[1], {p.nOfm / B, p.nIfm / B, p.kh, p.kw, B, B});
    const Resolved ri = resolve(n.stmt.reads[2], {p.nImg, p.nIfm / B, Hp, Wp, B});
    std::int64_t count = 0;
    oracle_detail::for_each_iteration(n, [&](const Point& x) {
      float& o = out[flat(ro, x)];
      o += flt[flat(rf, x)] * in_padded[flat(ri, x)];
      ++count;
    });
    return count;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// The reference emitter's text for a preset + recipe (emit.hpp:60-134).
std::int64_t ref_emit(const char* csv10, const char* recipe, char* buf, std::size_t len) {
  try {
    const ConvPreset p = ConvPreset::parse(csv10);
    LoopNest n = p.build();
    if (recipe && *recipe) n = apply_recipe(n, VariantRecipe::parse(recipe));
    const std::string s = emit_source(n);
    if (buf && len) {
      const std::size_t k = s.size() < len - 1 ? s.size() : len - 1;
      std::memcpy(buf, s.data(), k);
      buf[k] = 0;
    }
    return static_cast<std::int64_t>(s.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
