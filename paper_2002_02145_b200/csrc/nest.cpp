// Nest-document front end: reads the reference's
// textual loop-nest format (grammar of parse_nest, loopnest.hpp:340-523 — param,
// loop ... lower/upper/step, stmt, read/write with affine subscripts, body,
// microkernel/band/arg, annotation; '#' comments) and recognises the two
// computations the GPU path executes:
//   * the blocked direct convolution of presets.hpp:60-127 / samples/conv2d.nest
//     (any variable names, any order of the six outer loops) -> conv_desc + the
//     outer-loop order as a reference recipe id (variants.hpp:16-65);
//   * the matrix multiplication C[i][j] += A[i][k] * B[k][j] (samples/matmul.nest)
//     -> GEMM (M, N, K), executed as a 1x1 convolution (nest_info docs in psconv.h).
// Errors map to the reference's classes: ParseError / NotSupported -> status 2.
#include <cctype>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "internal.hpp"

namespace psconv {
namespace {

// affine expression: sum coeff[var] * var + cst
struct Affine {
  std::map<std::string, int64_t> coeff;
  int64_t cst = 0;
  bool is_const() const {
    for (const auto& kv : coeff)
      if (kv.second) return false;
    return true;
  }
  int64_t of(const std::string& v) const {
    auto it = coeff.find(v);
    return it == coeff.end() ? 0 : it->second;
  }
  int nvars() const {
    int n = 0;
    for (const auto& kv : coeff) n += kv.second != 0;
    return n;
  }
};

Affine add(Affine a, const Affine& b, int64_t sign) {
  for (const auto& kv : b.coeff) a.coeff[kv.first] += sign * kv.second;
  a.cst += sign * b.cst;
  return a;
}
Affine scale(Affine a, int64_t f) {
  for (auto& kv : a.coeff) kv.second *= f;
  a.cst *= f;
  return a;
}

class ExprParser {
 public:
  ExprParser(const std::string& t, const std::map<std::string, int64_t>& params,
             const std::set<std::string>& vars, int line)
      : t_(t), params_(params), vars_(vars), line_(line) {}
  Affine parse() {
    Affine e = expr();
    ws();
    if (p_ != t_.size()) fail("trailing characters in expression '" + t_ + "'");
    return e;
  }

 private:
  [[noreturn]] void fail(const std::string& m) const {
    throw ConfigError("nest line " + std::to_string(line_) + ": " + m);
  }
  void ws() {
    while (p_ < t_.size() && std::isspace(static_cast<unsigned char>(t_[p_]))) ++p_;
  }
  char peek() {
    ws();
    return p_ < t_.size() ? t_[p_] : '\0';
  }
  Affine expr() {
    Affine a = term();
    for (;;) {
      const char c = peek();
      if (c == '+') {
        ++p_;
        a = add(a, term(), 1);
      } else if (c == '-') {
        ++p_;
        a = add(a, term(), -1);
      } else {
        return a;
      }
    }
  }
  Affine term() {
    Affine a = factor();
    for (;;) {
      const char c = peek();
      if (c == '*') {
        ++p_;
        Affine b = factor();
        if (a.is_const()) a = scale(b, a.cst);
        else if (b.is_const()) a = scale(a, b.cst);
        else fail("product of two variables in '" + t_ + "' (non-affine)");
      } else if (c == '/') {
        ++p_;
        Affine b = factor();
        if (!a.is_const() || !b.is_const()) fail("division must be between constants in '" + t_ + "'");
        if (b.cst == 0) fail("division by zero");
        if (a.cst % b.cst) fail("non-exact constant division in '" + t_ + "'");
        a.cst /= b.cst;
      } else {
        return a;
      }
    }
  }
  Affine factor() {
    const char c = peek();
    Affine a;
    if (c == '(') {
      ++p_;
      a = expr();
      if (peek() != ')') fail("expected ')' in '" + t_ + "'");
      ++p_;
      return a;
    }
    if (c == '-') {
      ++p_;
      return scale(factor(), -1);
    }
    if (std::isdigit(static_cast<unsigned char>(c))) {
      int64_t v = 0;
      while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) v = v * 10 + (t_[p_++] - '0');
      a.cst = v;
      return a;
    }
    if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
      std::string name;
      while (p_ < t_.size() && (std::isalnum(static_cast<unsigned char>(t_[p_])) || t_[p_] == '_'))
        name += t_[p_++];
      auto it = params_.find(name);
      if (it != params_.end()) {
        a.cst = it->second;
        return a;
      }
      if (vars_.count(name)) {
        a.coeff[name] = 1;
        return a;
      }
      fail("unbound parameter '" + name + "'");
    }
    fail(std::string("unexpected character '") + c + "' in expression '" + t_ + "'");
  }

  const std::string& t_;
  const std::map<std::string, int64_t>& params_;
  const std::set<std::string>& vars_;
  int line_;
  size_t p_ = 0;
};

std::string trim(const std::string& s) {
  const size_t b = s.find_first_not_of(" \t\r\n");
  if (b == std::string::npos) return "";
  return s.substr(b, s.find_last_not_of(" \t\r\n") - b + 1);
}
std::vector<std::string> words(const std::string& s) {
  std::vector<std::string> out;
  std::istringstream is(s);
  std::string w;
  while (is >> w) out.push_back(w);
  return out;
}

struct NLoop {
  std::string var;
  Affine lower, upper;
  int64_t step = 1;
};
struct NRef {
  std::string array;
  bool write = false;
  std::vector<Affine> idx;
};
struct Nest {
  std::map<std::string, int64_t> params;
  std::vector<NLoop> loops;
  std::vector<NRef> refs;
  std::vector<std::string> band;
  bool has_stmt = false;
};

Nest parse(const std::string& text) {
  Nest n;
  std::set<std::string> vars;
  bool in_mk = false;
  std::istringstream is(text);
  std::string raw;
  int line = 0;
  auto fail = [&](const std::string& m) { throw ConfigError("nest line " + std::to_string(line) + ": " + m); };
  while (std::getline(is, raw)) {
    ++line;
    const std::string l = trim(raw);
    if (l.empty() || l[0] == '#') continue;
    const std::string kw = words(l)[0];
    const std::string rest = trim(l.substr(kw.size()));
    if (kw == "param") {
      auto t = words(rest);
      if (t.size() == 3 && t[1] == "=") t.erase(t.begin() + 1);
      if (t.size() != 2) fail("expected 'param NAME = INT'");
      try {
        n.params[t[0]] = std::stoll(t[1]);
      } catch (const std::logic_error&) {
        fail("bad parameter value '" + t[1] + "'");
      }
    } else if (kw == "loop") {
      if (n.has_stmt) fail("loops must precede the statement");
      auto t = words(rest);
      if (t.empty()) fail("expected loop variable name");
      NLoop lp;
      lp.var = t[0];
      if (vars.count(lp.var)) fail("duplicate loop variable '" + lp.var + "'");
      std::map<std::string, std::string> seg;
      std::string cur;
      for (size_t i = 1; i < t.size(); ++i) {
        if (t[i] == "lower" || t[i] == "upper" || t[i] == "step") {
          cur = t[i];
          if (seg.count(cur)) fail("duplicate '" + cur + "'");
          seg[cur] = "";
        } else if (cur.empty()) {
          fail("unexpected token '" + t[i] + "'");
        } else {
          seg[cur] += (seg[cur].empty() ? "" : " ") + t[i];
        }
      }
      if (!seg.count("lower") || !seg.count("upper")) fail("loop needs 'lower' and 'upper' bounds");
      lp.lower = ExprParser(seg["lower"], n.params, vars, line).parse();
      lp.upper = ExprParser(seg["upper"], n.params, vars, line).parse();
      if (seg.count("step")) {
        const Affine st = ExprParser(seg["step"], n.params, vars, line).parse();
        if (!st.is_const() || st.cst < 1) fail("loop step must be a positive integer constant");
        lp.step = st.cst;
      }
      vars.insert(lp.var);
      n.loops.push_back(lp);
    } else if (kw == "stmt") {
      if (n.has_stmt) fail("multi-statement nests are not supported");
      if (words(rest).size() != 1) fail("expected 'stmt NAME'");
      n.has_stmt = true;
    } else if (kw == "read" || kw == "write") {
      if (!n.has_stmt) fail("reference before 'stmt'");
      NRef r;
      r.write = kw == "write";
      const size_t br = rest.find('[');
      r.array = trim(br == std::string::npos ? rest : rest.substr(0, br));
      if (r.array.empty()) fail("expected array name");
      size_t pos = br;
      while (pos != std::string::npos && pos < rest.size()) {
        if (rest[pos] != '[') fail("expected '[' in reference");
        int depth = 1;
        size_t e = pos + 1;
        while (e < rest.size() && depth) {
          depth += rest[e] == '[' ? 1 : (rest[e] == ']' ? -1 : 0);
          ++e;
        }
        if (depth) fail("unbalanced ']' in reference");
        r.idx.push_back(ExprParser(rest.substr(pos + 1, e - pos - 2), n.params, vars, line).parse());
        pos = e;
        while (pos < rest.size() && std::isspace(static_cast<unsigned char>(rest[pos]))) ++pos;
      }
      if (r.idx.empty()) fail("reference has no subscripts");
      n.refs.push_back(r);
    } else if (kw == "body") {
      if (!n.has_stmt) fail("'body' before 'stmt'");
    } else if (kw == "microkernel") {
      if (words(rest).size() != 1) fail("expected 'microkernel CALLEE'");
      in_mk = true;
    } else if (kw == "band") {
      if (!in_mk) fail("'band' outside microkernel block");
      std::string s = rest;
      for (char& c : s)
        if (c == ',') c = ' ';
      n.band = words(s);
      if (n.band.empty()) fail("empty band");
    } else if (kw == "arg") {
      if (!in_mk) fail("'arg' outside microkernel block");
    } else if (kw == "annotation") {
    } else {
      fail("unknown directive '" + kw + "'");
    }
  }
  if (n.loops.empty()) throw ConfigError("nest has no loops");
  if (!n.has_stmt) throw ConfigError("nest has no statement");
  if (n.refs.empty()) throw ConfigError("statement has no references");
  if (!n.band.empty()) {
    if (n.band.size() > n.loops.size()) throw ConfigError("microkernel band has more loops than the nest");
    for (size_t i = 0; i < n.band.size(); ++i)
      if (n.loops[n.loops.size() - n.band.size() + i].var != n.band[i])
        throw ConfigError("microkernel band loops must be the contiguous innermost loops in band order");
  }
  return n;
}

// a subscript that is exactly one loop variable (coefficient 1, no constant)
std::string single_var(const Affine& a) {
  if (a.cst != 0 || a.nvars() != 1) return "";
  for (const auto& kv : a.coeff)
    if (kv.second == 1) return kv.first;
  return "";
}

[[noreturn]] void unsupported(const std::string& m) {
  throw ConfigError("nest is not a supported computation: " + m);
}

const NRef* find_ref(const Nest& n, const std::string& array, bool write) {
  for (const auto& r : n.refs)
    if (r.array == array && r.write == write) return &r;
  return nullptr;
}

// extent of a loop with constant bounds, lower 0, step 1
int64_t extent(const Nest& n, const std::string& var) {
  for (const auto& l : n.loops)
    if (l.var == var) {
      if (!l.lower.is_const() || !l.upper.is_const()) unsupported("loop '" + var + "' has non-constant bounds");
      if (l.lower.cst != 0 || l.step != 1) unsupported("loop '" + var + "' must run from 0 with step 1");
      return l.upper.cst;
    }
  unsupported("no loop '" + var + "'");
}

}  // namespace

void nest_recognise(const std::string& text, nest_info* out) {
  const Nest n = parse(text);
  std::memset(out, 0, sizeof(*out));
  // the written array (exactly one) and the two read factors
  const NRef* w = nullptr;
  for (const auto& r : n.refs)
    if (r.write) {
      if (w && w->array != r.array) unsupported("more than one written array");
      w = &r;
    }
  if (!w) unsupported("no written array");
  std::vector<const NRef*> rd;
  for (const auto& r : n.refs)
    if (!r.write && r.array != w->array) rd.push_back(&r);
  if (rd.size() != 2) unsupported("expected two read operands besides the accumulator");
  for (const auto& l : n.loops)
    if (!l.lower.is_const() || !l.upper.is_const()) unsupported("non-rectangular (tiled) loop bounds");

  if (w->idx.size() == 2) {
    // ---- GEMM: C[i][j] += A[i][k] * B[k][j]
    const std::string i = single_var(w->idx[0]), j = single_var(w->idx[1]);
    if (i.empty() || j.empty()) unsupported("GEMM output subscripts must be loop variables");
    const NRef* a = nullptr;
    const NRef* b = nullptr;
    for (const NRef* r : rd) {
      if (r->idx.size() != 2) unsupported("GEMM operands must be 2-D");
      if (single_var(r->idx[0]) == i) a = r;
      else if (single_var(r->idx[1]) == j) b = r;
    }
    if (!a || !b) unsupported("expected A[i][k] and B[k][j]");
    const std::string k = single_var(a->idx[1]);
    if (k.empty() || single_var(b->idx[0]) != k || k == i || k == j) unsupported("reduction index mismatch");
    out->kind = NEST_KIND_GEMM;
    out->M = extent(n, i);
    out->N = extent(n, j);
    out->K = extent(n, k);
    // the GEMM as a 1x1 convolution over M "pixels": A = NCHW16c, C = NKPQ16k
    conv_desc& d = out->desc;
    d.nImg = out->M;
    d.nOfm = out->N;
    d.nIfm = out->K;
    d.ofh = d.ofw = d.kh = d.kw = d.stride_h = d.stride_w = 1;
    d.gemm_block = 16;
    std::snprintf(out->recipe, sizeof(out->recipe), "%s", "");
    return;
  }
  if (w->idx.size() != 5) unsupported("output must be 2-D (GEMM) or 5-D NKPQ16k (conv)");

  // ---- blocked conv (presets.hpp:60-127): out[img][ofm_tile][oj][oi][ofm]
  std::string v_img = single_var(w->idx[0]), v_ot = single_var(w->idx[1]), v_oj = single_var(w->idx[2]),
              v_oi = single_var(w->idx[3]), v_ofm = single_var(w->idx[4]);
  if (v_img.empty() || v_ot.empty() || v_oj.empty() || v_oi.empty() || v_ofm.empty())
    unsupported("output subscripts must be loop variables");
  const NRef* flt = nullptr;
  const NRef* in = nullptr;
  for (const NRef* r : rd) {
    if (r->idx.size() == 6) flt = r;
    else if (r->idx.size() == 5) in = r;
  }
  if (!flt || !in) unsupported("expected a 6-D filter and a 5-D input");
  // filter[ofm_tile][ifm_tile][kj][ki][ifm][ofm]
  if (single_var(flt->idx[0]) != v_ot || single_var(flt->idx[5]) != v_ofm)
    unsupported("filter must be indexed [ofm_tile][ifm_tile][kj][ki][ifm][ofm]");
  const std::string v_it = single_var(flt->idx[1]), v_kj = single_var(flt->idx[2]),
                    v_ki = single_var(flt->idx[3]), v_ifm = single_var(flt->idx[4]);
  if (v_it.empty() || v_kj.empty() || v_ki.empty() || v_ifm.empty()) unsupported("filter subscripts");
  // input[img][ifm_tile][oj*SH + kj][oi*SW + ki][ifm]
  if (single_var(in->idx[0]) != v_img || single_var(in->idx[1]) != v_it || single_var(in->idx[4]) != v_ifm)
    unsupported("input must be indexed [img][ifm_tile][..][..][ifm]");
  const Affine& ih = in->idx[2];
  const Affine& iw = in->idx[3];
  if (ih.nvars() != 2 || ih.of(v_kj) != 1 || ih.of(v_oj) < 1 || ih.cst != 0)
    unsupported("input row subscript must be oj*stride_h + kj");
  if (iw.nvars() != 2 || iw.of(v_ki) != 1 || iw.of(v_oi) < 1 || iw.cst != 0)
    unsupported("input column subscript must be oi*stride_w + ki");
  const int64_t gb = extent(n, v_ofm);
  if (extent(n, v_ifm) != gb) unsupported("ofm and ifm block loops must have the same extent");
  conv_desc& d = out->desc;
  d.nImg = extent(n, v_img);
  d.nOfm = extent(n, v_ot) * gb;
  d.nIfm = extent(n, v_it) * gb;
  d.ofh = extent(n, v_oj);
  d.ofw = extent(n, v_oi);
  d.kh = extent(n, v_kj);
  d.kw = extent(n, v_ki);
  d.stride_h = ih.of(v_oj);
  d.stride_w = iw.of(v_oi);
  d.gemm_block = gb;
  out->kind = NEST_KIND_CONV;
  // outer-loop order -> reference recipe id over the canonical loop names
  const std::map<std::string, std::string> canon = {{v_img, "img"}, {v_ot, "ofm_tile"}, {v_it, "ifm_tile"},
                                                    {v_oj, "oj"},   {v_kj, "kj"},       {v_ki, "ki"},
                                                    {v_oi, "oi"},   {v_ofm, "ofm"},     {v_ifm, "ifm"}};
  if (n.loops.size() != 9) unsupported("expected the 9-loop conv nest");
  std::vector<std::string> order;
  for (const auto& l : n.loops) order.push_back(canon.at(l.var));
  const std::vector<std::string> band = {"oi", "ofm", "ifm"};
  if (std::vector<std::string>(order.end() - 3, order.end()) != band)
    unsupported("the band (oi, ofm, ifm) must be innermost");
  if (order[0] != "img") unsupported("img must stay the outermost loop (variants.hpp:426-433)");
  std::string perm = "perm=";
  for (int i = 1; i < 6; ++i) perm += (i > 1 ? "," : "") + order[i];
  std::snprintf(out->recipe, sizeof(out->recipe), "%s", perm.c_str());
}

}  // namespace psconv

using namespace psconv;

extern "C" int nest_parse(const char* text, nest_info* out) {
  return guarded([&] {
    if (!text || !out) throw ConfigError("null argument");
    nest_recognise(text, out);
    // the GEMM's 1x1-conv descriptor is runnable only when N, K are multiples of 16
    if (out->kind == NEST_KIND_GEMM && (out->N % 16 || out->K % 16)) return;
    conv_desc d = out->desc;
    validate_desc(d);  // same rules as ConvPreset::validate (presets.hpp:52-58)
    out->desc = d;
  });
}
