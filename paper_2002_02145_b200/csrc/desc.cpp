// Conv-layer descriptor: parse / validate / format, error plumbing, loop names.
// Mirrors nestrank::ConvPreset (include/nestrank/presets.hpp:13-58) and the
// `conv:` loader (include/nestrank/cli.hpp:54-66).
#include <cctype>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "internal.hpp"

namespace psconv {

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }
void clear_last_error() { g_last_error.clear(); }

static const char* kLoopNames[L_COUNT] = {"img", "ofm_tile", "ifm_tile", "oj", "kj", "ki"};

const char* loop_name(int id) { return (id >= 0 && id < L_COUNT) ? kLoopNames[id] : "?"; }

int loop_id(const std::string& name) {
  for (int i = 0; i < L_COUNT; ++i)
    if (name == kLoopNames[i]) return i;
  return -1;
}

void validate_desc(conv_desc& d) {
  // presets.hpp:52-58
  const int64_t ref[] = {d.nImg, d.nOfm, d.nIfm, d.ofh, d.ofw, d.kh, d.kw, d.stride_h, d.stride_w,
                         d.gemm_block};
  for (int64_t v : ref)
    if (v < 1) throw ConfigError("conv preset values must be positive");
  if (d.nOfm % d.gemm_block != 0 || d.nIfm % d.gemm_block != 0)
    throw ConfigError("conv preset: channel widths must be divisible by gemm_block");
  // extension fields
  if (d.pad_h < 0 || d.pad_w < 0) throw ConfigError("conv preset: padding must be non-negative");
  if (d.pad_h >= d.kh || d.pad_w >= d.kw)
    throw ConfigError("conv preset: padding must be smaller than the filter extent");
  const int64_t need_h = (d.ofh - 1) * d.stride_h + d.kh;  // reference-implied padded extent
  const int64_t need_w = (d.ofw - 1) * d.stride_w + d.kw;
  if (d.ifh == 0) d.ifh = need_h - 2 * d.pad_h;
  if (d.ifw == 0) d.ifw = need_w - 2 * d.pad_w;
  if (d.ifh < 1 || d.ifw < 1) throw ConfigError("conv preset: input extent must be positive");
  if (d.ifh + 2 * d.pad_h < need_h || d.ifw + 2 * d.pad_w < need_w)
    throw ConfigError("conv preset: input extent too small for ofh/ofw, stride, filter and pad");
  // every output window must touch at least one real input row/column
  if ((d.ofh - 1) * d.stride_h - d.pad_h > d.ifh - 1 || (d.ofw - 1) * d.stride_w - d.pad_w > d.ifw - 1)
    throw ConfigError("conv preset: last output window lies entirely in padding");
  const int64_t lim = int64_t(1) << 31;
  if (d.nImg >= lim || d.nOfm >= lim || d.nIfm >= lim || d.ifh >= lim || d.ifw >= lim ||
      d.ofh >= lim || d.ofw >= lim)
    throw ConfigError("conv preset: extent too large");
}

}  // namespace psconv

using namespace psconv;

extern "C" {

const char* conv_last_error(void) { return g_last_error.c_str(); }

const char* psconv_version(void) { return "psconv-b200 0.1 (sm_100a)"; }

int conv_desc_validate(conv_desc* d) {
  return guarded([&] {
    if (!d) throw ConfigError("null descriptor");
    validate_desc(*d);
  });
}

int conv_desc_parse(const char* text, conv_desc* out) {
  return guarded([&] {
    if (!text || !out) throw ConfigError("null argument");
    std::string s(text);
    // cli.hpp:58-60: the preset form is "conv:<ints>"; a bare list is the
    // ConvPreset::parse form. Any other "name:" prefix is an unknown preset.
    if (s.rfind("conv:", 0) == 0) {
      s = s.substr(5);
    } else {
      const auto colon = s.find(':');
      if (colon != std::string::npos)
        throw ConfigError("unknown preset '" + s + "' (expected conv:<10 ints>)");
    }
    // presets.hpp:26-43: split on ',', drop whitespace, skip empty fields.
    std::vector<int64_t> v;
    std::string cur;
    for (char c : s + ",") {
      if (c == ',') {
        if (!cur.empty()) {
          try {
            v.push_back(std::stoll(cur));
          } catch (const std::logic_error&) {
            throw ConfigError("bad conv preset value '" + cur + "'");
          }
          cur.clear();
        }
      } else if (!std::isspace(static_cast<unsigned char>(c))) {
        cur += c;
      }
    }
    if (v.size() != 10 && v.size() != 12 && v.size() != 14)
      throw ConfigError("conv preset needs 10 integers, got " + std::to_string(v.size()));
    conv_desc d{};
    d.nImg = v[0];
    d.nOfm = v[1];
    d.nIfm = v[2];
    d.ofh = v[3];
    d.ofw = v[4];
    d.kh = v[5];
    d.kw = v[6];
    d.stride_h = v[7];
    d.stride_w = v[8];
    d.gemm_block = v[9];
    if (v.size() >= 12) {
      d.pad_h = v[10];
      d.pad_w = v[11];
    }
    if (v.size() == 14) {
      d.ifh = v[12];
      d.ifw = v[13];
    }
    validate_desc(d);
    *out = d;
  });
}

int conv_desc_format(const conv_desc* d, char* buf, size_t len) {
  return guarded([&] {
    if (!d || !buf) throw ConfigError("null argument");
    conv_desc v = *d;
    validate_desc(v);
    const bool ext = v.pad_h || v.pad_w || v.ifh != (v.ofh - 1) * v.stride_h + v.kh ||
                     v.ifw != (v.ofw - 1) * v.stride_w + v.kw;
    char tmp[512];
    int n;
    if (!ext)
      n = std::snprintf(tmp, sizeof tmp, "conv:%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld",
                        (long long)v.nImg, (long long)v.nOfm, (long long)v.nIfm, (long long)v.ofh,
                        (long long)v.ofw, (long long)v.kh, (long long)v.kw,
                        (long long)v.stride_h, (long long)v.stride_w, (long long)v.gemm_block);
    else
      n = std::snprintf(
          tmp, sizeof tmp,
          "conv:%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld",
          (long long)v.nImg, (long long)v.nOfm, (long long)v.nIfm, (long long)v.ofh,
          (long long)v.ofw, (long long)v.kh, (long long)v.kw, (long long)v.stride_h,
          (long long)v.stride_w, (long long)v.gemm_block, (long long)v.pad_h, (long long)v.pad_w,
          (long long)v.ifh, (long long)v.ifw);
    if (n < 0 || static_cast<size_t>(n) + 1 > len) throw ConfigError("buffer too small");
    std::memcpy(buf, tmp, static_cast<size_t>(n) + 1);
  });
}

}  // extern "C"
