// nestrank_b200/psconv_binding.hpp -- the reference-side binding (header-only C++20) a
// nestrank maintainer adds to call the B200 path through include/psconv.h.
//
// Reference interfaces bound (paths under /root/reference/proj/include/nestrank):
//   ConvPreset (presets.hpp:13-58)            -> conv_desc / conv_desc_validate
//   gemm_microkernel(out, flt, in) call of the emitted driver (presets.hpp:116-123,
//     emit.hpp:75-81; LIBXSMM in the paper)   -> gemm_microkernel_dispatch
//   a VariantRecipe id (variants.hpp:16-65)   -> conv_plan_create's recipe
//   exit-status classes (cli.hpp:290-321)     -> ConfigRejectedError (2) / Error (1)
// Compiled against the reference headers and exercised by tests/test_adapter.py.
#pragma once
#include <cstdint>
#include <memory>
#include <string>

#include "nestrank/common.hpp"
#include "nestrank/presets.hpp"
#include "psconv.h"

namespace nestrank::b200 {

inline void check(int rc) {
  if (rc == PSCONV_ERR_CONFIG) throw ConfigRejectedError(conv_last_error());
  if (rc != PSCONV_OK) throw Error(conv_last_error());
}

// The preset as the C-ABI descriptor; pad / input extent default to the reference's
// implied extent (no padding, presets.hpp:88-91).
inline conv_desc to_desc(const ConvPreset& p, std::int64_t pad_h = 0, std::int64_t pad_w = 0,
                         std::int64_t ifh = 0, std::int64_t ifw = 0) {
  conv_desc d{p.nImg,     p.nOfm,     p.nIfm,       p.ofh, p.ofw, p.kh,  p.kw,
              p.stride_h, p.stride_w, p.gemm_block, pad_h, pad_w, ifh, ifw};
  check(conv_desc_validate(&d));
  return d;
}

// CPU: the microkernel an emitted driver calls, bound to the preset's shape (LIBXSMM-style
// dispatch: the returned function takes only the three pointers).
inline gemm_microkernel_fn microkernel(const ConvPreset& p) {
  conv_desc d = to_desc(p);
  gemm_microkernel_fn fn = nullptr;
  check(gemm_microkernel_dispatch(&d, &fn));
  return fn;
}

// GPU: one layer on one device; `recipe` is a VariantRecipe id (e.g. the top of
// rank_variants) or "" (the B200 selector decides).
class Layer {
 public:
  Layer(const ConvPreset& p, const std::string& recipe, int device = 0, int mode = PSCONV_MODE_3XTF32)
      : Layer(to_desc(p), recipe, device, mode) {}
  Layer(conv_desc d, const std::string& recipe, int device = 0, int mode = PSCONV_MODE_3XTF32) {
    conv_plan* raw = nullptr;
    check(conv_plan_create(&d, mode, device, recipe.empty() ? nullptr : recipe.c_str(), &raw));
    plan_.reset(raw);
  }
  std::string recipe() const { return conv_plan_recipe(plan_.get()); }
  // device pointers in NCHW16c / KCRS16c16k / NKPQ16k (the ArrayRef layouts, presets.hpp:93-97)
  void forward(const float* in, const float* flt, float* out, std::int64_t img_begin, std::int64_t img_count,
               void* stream = nullptr) const {
    check(conv_fwd(plan_.get(), in, flt, out, img_begin, img_count, stream, 0));
  }
  // host pointers (pinned for overlap), e.g. the arrays an emitted driver is handed
  void forward_host(const float* in, const float* flt, float* out, std::int64_t img_begin,
                    std::int64_t img_count, void* stream = nullptr) const {
    check(conv_fwd_host(plan_.get(), in, flt, out, img_begin, img_count, stream, 0));
  }

 private:
  std::unique_ptr<conv_plan, void (*)(conv_plan*)> plan_{nullptr, conv_plan_destroy};
};

}  // namespace nestrank::b200
