// CPU microkernel with the reference's 3-pointer call convention
// (ConvPreset::build call args, include/nestrank/presets.hpp:116-123;
// MicrokernelSpec, loopnest.hpp:139-148). In the paper this is LIBXSMM's
// JIT'ed small GEMM: the shape is bound at dispatch time and
// the kernel is called with pointers only. Without a JIT, dispatch binds the
// shape to one of a fixed pool of trampolines, each reading its own slot.
//
// Band semantics (presets.hpp:82-84,112-114) for one call:
//   for oi < ofw, ofm < 16, ifm < 16:
//     out[oi*16 + ofm] += flt[ifm*16 + ofm] * in[oi*stride_w*16 + ifm]
// Per output element the accumulation runs over ifm in order, as in the band.
#include <array>
#include <mutex>
#include <utility>

#include "internal.hpp"

namespace psconv {
namespace {

struct MkShape {
  int ofw = 0, sw = 0;
};

constexpr int kSlots = 64;
MkShape g_shape[kSlots];
int g_nslots = 0;
std::mutex g_mu;

__attribute__((target_clones("avx512f", "avx2", "default"))) void mk_run(int ofw, int sw,
                                                                          float* __restrict out,
                                                                          const float* __restrict flt,
                                                                          const float* __restrict in) {
  int oi = 0;
  for (; oi + 4 <= ofw; oi += 4) {
    float acc[4][16];
    for (int j = 0; j < 4; ++j)
      for (int k = 0; k < 16; ++k) acc[j][k] = out[(oi + j) * 16 + k];
    for (int c = 0; c < 16; ++c) {
      const float* f = flt + c * 16;
      for (int j = 0; j < 4; ++j) {
        const float x = in[(oi + j) * sw * 16 + c];
        for (int k = 0; k < 16; ++k) acc[j][k] += f[k] * x;
      }
    }
    for (int j = 0; j < 4; ++j)
      for (int k = 0; k < 16; ++k) out[(oi + j) * 16 + k] = acc[j][k];
  }
  for (; oi < ofw; ++oi) {
    float acc[16];
    for (int k = 0; k < 16; ++k) acc[k] = out[oi * 16 + k];
    for (int c = 0; c < 16; ++c) {
      const float x = in[oi * sw * 16 + c];
      for (int k = 0; k < 16; ++k) acc[k] += flt[c * 16 + k] * x;
    }
    for (int k = 0; k < 16; ++k) out[oi * 16 + k] = acc[k];
  }
}

template <int SLOT>
void mk_slot(float* out, const float* flt, const float* in) {
  mk_run(g_shape[SLOT].ofw, g_shape[SLOT].sw, out, flt, in);
}

template <size_t... I>
constexpr auto make_table(std::index_sequence<I...>) {
  return std::array<gemm_microkernel_fn, sizeof...(I)>{&mk_slot<static_cast<int>(I)>...};
}
const auto g_table = make_table(std::make_index_sequence<kSlots>{});

gemm_microkernel_fn dispatch(int ofw, int sw) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (int i = 0; i < g_nslots; ++i)
    if (g_shape[i].ofw == ofw && g_shape[i].sw == sw) return g_table[i];
  if (g_nslots == kSlots) throw RuntimeError("gemm_microkernel_dispatch: shape pool exhausted");
  g_shape[g_nslots] = MkShape{ofw, sw};
  return g_table[g_nslots++];
}

}  // namespace
}  // namespace psconv

using namespace psconv;

extern "C" {

int gemm_microkernel_dispatch(const conv_desc* d_in, gemm_microkernel_fn* fn) {
  return guarded([&] {
    if (!d_in || !fn) throw ConfigError("null argument");
    conv_desc d = *d_in;
    validate_desc(d);
    if (d.gemm_block != 16) throw ConfigError("gemm_microkernel: only gemm_block == 16 is built");
    if (d.ofw * d.stride_w > 4096) throw ConfigError("gemm_microkernel: ofw*stride_w > 4096");
    *fn = dispatch(static_cast<int>(d.ofw), static_cast<int>(d.stride_w));
  });
}

int brgemm_f32(const conv_desc* d_in, float* out, const float* const* flt_blocks,
               const float* const* in_rows, int64_t count) {
  return guarded([&] {
    if (!d_in || !out || (count > 0 && (!flt_blocks || !in_rows))) throw ConfigError("null argument");
    conv_desc d = *d_in;
    validate_desc(d);
    if (d.gemm_block != 16) throw ConfigError("brgemm_f32: only gemm_block == 16 is built");
    const int ofw = static_cast<int>(d.ofw), sw = static_cast<int>(d.stride_w);
    for (int64_t i = 0; i < count; ++i) mk_run(ofw, sw, out, flt_blocks[i], in_rows[i]);
  });
}

}  // extern "C"
