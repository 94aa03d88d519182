// Pairwise DNN ranker (PolyScientist-DNN; reference
// dnnrank.hpp:87-438, pipeline.hpp:98-173, paper PAPER.md:452-502).
//
// Same contract as the reference: a feed-forward net 8-64-32-16-8-2 (relu,
// relu, softsign, relu, softmax) reads the statistics of two variants, jointly
// normalised by their sum, and calls A or B the faster one when its softmax
// output exceeds theta (else a draw); trained by mini-batch gradient descent
// on the cross-entropy, deterministic under the seed; weights in the plain-text
// "pairnet 1" format; variants ranked by a round-robin tournament (wins desc,
// then modelled cost, then id) with a symmetry diagnostic.
// B200 re-expression: the four per-variant statistics are the closed-form
// model's resource times (MMA issue, shared-memory traffic, operand-row
// delivery, HBM; select.cpp model_stats) instead of cache-level working sets,
// and the training pairs come from measured B200 timings
// (tools/collect_ranker_data.py -> tools/train_ranker.py).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "internal.hpp"

namespace psconv {
namespace {

constexpr int kDims[6] = {8, 64, 32, 16, 8, 2};
const char* const kActs[5] = {"relu", "relu", "softsign", "relu", "softmax"};

// splitmix64 stream: deterministic init / shuffles independent of the C++ library
struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform(double lo, double hi) { return lo + (hi - lo) * (double(next() >> 11) * 0x1.0p-53); }
  size_t below(size_t n) { return size_t(next() % n); }
};

struct Pair {
  double a[4], b[4];
  int winner;  // 0: A faster, 1: B faster
};

struct Net {
  struct Layer {
    int in, out;
    std::vector<double> w, b;  // w row-major out x in
  };
  std::vector<Layer> layers;
  double theta = 0.6;

  static Net init(uint64_t seed) {
    Net n;
    Rng rng(seed);
    for (int l = 0; l < 5; ++l) {
      Layer L{kDims[l], kDims[l + 1], {}, {}};
      L.w.resize(size_t(L.in) * L.out);
      L.b.assign(size_t(L.out), 0.0);
      const double lim = std::sqrt(6.0 / L.in);
      for (double& v : L.w) v = rng.uniform(-lim, lim);
      n.layers.push_back(L);
    }
    return n;
  }

  static void normalise(const double* a, const double* b, double* x) {
    double sum = 0;
    for (int i = 0; i < 4; ++i) {
      if (a[i] < 0 || b[i] < 0 || !std::isfinite(a[i]) || !std::isfinite(b[i]))
        throw ConfigError("ranker: statistics must be finite and non-negative");
      sum += a[i] + b[i];
    }
    if (sum <= 0) throw ConfigError("ranker: both variants have all-zero statistics");
    for (int i = 0; i < 4; ++i) {
      x[i] = a[i] / sum;
      x[4 + i] = b[i] / sum;
    }
  }

  // forward pass keeping pre-activations (z) and layer inputs (act)
  void run(const double* x, std::vector<std::vector<double>>& act, std::vector<std::vector<double>>& z) const {
    act.assign(1, std::vector<double>(x, x + 8));
    z.clear();
    for (size_t l = 0; l < layers.size(); ++l) {
      const Layer& L = layers[l];
      std::vector<double> o(size_t(L.out));
      for (int j = 0; j < L.out; ++j) {
        double v = L.b[size_t(j)];
        for (int i = 0; i < L.in; ++i) v += L.w[size_t(j) * L.in + i] * act.back()[size_t(i)];
        o[size_t(j)] = v;
      }
      z.push_back(o);
      if (l + 1 == layers.size()) break;
      for (double& v : o) v = l == 2 ? v / (1.0 + std::fabs(v)) : (v > 0 ? v : 0.0);
      act.push_back(o);
    }
  }
  static void softmax2(const std::vector<double>& z, double* p) {
    const double m = std::max(z[0], z[1]);
    const double e0 = std::exp(z[0] - m), e1 = std::exp(z[1] - m);
    p[0] = e0 / (e0 + e1);
    p[1] = e1 / (e0 + e1);
  }
  void prob(const double* a, const double* b, double* p) const {
    double x[8];
    normalise(a, b, x);
    std::vector<std::vector<double>> act, z;
    run(x, act, z);
    softmax2(z.back(), p);
  }
  int compare(const double* a, const double* b) const {  // 0 A, 1 B, 2 draw
    double p[2];
    prob(a, b, p);
    return p[0] > theta ? 0 : (p[1] > theta ? 1 : 2);
  }

  void sgd_step(const std::vector<const Pair*>& batch, double lr) {
    std::vector<std::vector<double>> gw(layers.size()), gb(layers.size());
    for (size_t l = 0; l < layers.size(); ++l) {
      gw[l].assign(layers[l].w.size(), 0.0);
      gb[l].assign(layers[l].b.size(), 0.0);
    }
    for (const Pair* pr : batch) {
      double x[8], p[2];
      normalise(pr->a, pr->b, x);
      std::vector<std::vector<double>> act, z;
      run(x, act, z);
      softmax2(z.back(), p);
      std::vector<double> dz = {p[0], p[1]};
      dz[size_t(pr->winner)] -= 1.0;  // d(cross-entropy)/d(logits)
      for (size_t l = layers.size(); l-- > 0;) {
        const Layer& L = layers[l];
        for (int j = 0; j < L.out; ++j) {
          gb[l][size_t(j)] += dz[size_t(j)];
          for (int i = 0; i < L.in; ++i) gw[l][size_t(j) * L.in + i] += dz[size_t(j)] * act[l][size_t(i)];
        }
        if (l == 0) break;
        std::vector<double> din(size_t(L.in), 0.0);
        for (int i = 0; i < L.in; ++i)
          for (int j = 0; j < L.out; ++j) din[size_t(i)] += L.w[size_t(j) * L.in + i] * dz[size_t(j)];
        const std::vector<double>& zp = z[l - 1];
        for (int i = 0; i < L.in; ++i) {
          const double zi = zp[size_t(i)];
          const double g = (l - 1 == 2) ? 1.0 / ((1.0 + std::fabs(zi)) * (1.0 + std::fabs(zi))) : (zi > 0 ? 1.0 : 0.0);
          din[size_t(i)] *= g;
        }
        dz.swap(din);
      }
    }
    const double sc = lr / double(batch.size());
    for (size_t l = 0; l < layers.size(); ++l) {
      for (size_t i = 0; i < layers[l].w.size(); ++i) layers[l].w[i] -= sc * gw[l][i];
      for (size_t i = 0; i < layers[l].b.size(); ++i) layers[l].b[i] -= sc * gb[l][i];
    }
  }

  static Net train(const std::vector<Pair>& data, int epochs, double lr, uint64_t seed, int batch) {
    if (data.empty()) throw ConfigError("ranker: training dataset is empty");
    Net n = init(seed);
    Rng rng(seed ^ 0x5EEDF00Dull);
    std::vector<size_t> order(data.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    for (int e = 0; e < epochs; ++e) {
      for (size_t i = order.size(); i > 1; --i) std::swap(order[i - 1], order[rng.below(i)]);
      for (size_t s = 0; s < order.size(); s += size_t(batch)) {
        std::vector<const Pair*> b;
        for (size_t i = s; i < std::min(order.size(), s + size_t(batch)); ++i) b.push_back(&data[order[i]]);
        n.sgd_step(b, lr);
      }
    }
    return n;
  }

  double accuracy(const std::vector<Pair>& data) const {
    if (data.empty()) return 0.0;
    size_t good = 0;
    for (const Pair& p : data) {
      double pr[2];
      prob(p.a, p.b, pr);
      good += (pr[0] >= pr[1] ? 0 : 1) == p.winner;
    }
    return double(good) / double(data.size());
  }

  std::string save() const {
    std::ostringstream os;
    os.precision(17);
    os << "pairnet 1\ndims";
    for (int d : kDims) os << ' ' << d;
    os << "\nactivations";
    for (const char* a : kActs) os << ' ' << a;
    os << "\ntheta " << theta << "\n";
    for (size_t l = 0; l < layers.size(); ++l) {
      const Layer& L = layers[l];
      os << "layer " << l << ' ' << L.out << ' ' << L.in << "\n";
      for (int j = 0; j < L.out; ++j) {
        for (int i = 0; i < L.in; ++i) os << (i ? " " : "") << L.w[size_t(j) * L.in + i];
        os << "\n";
      }
      os << "bias";
      for (int j = 0; j < L.out; ++j) os << ' ' << L.b[size_t(j)];
      os << "\n";
    }
    return os.str();
  }

  static Net load(const std::string& text) {
    std::istringstream is(text);
    std::string tok;
    auto bad = [](const std::string& m) { throw ConfigError("ranker weights: " + m); };
    int ver = 0;
    if (!(is >> tok) || tok != "pairnet" || !(is >> ver) || ver != 1) bad("bad magic/version");
    if (!(is >> tok) || tok != "dims") bad("missing dims");
    for (int d : kDims) {
      int g;
      if (!(is >> g) || g != d) bad("unexpected layer dimensions");
    }
    if (!(is >> tok) || tok != "activations") bad("missing activations");
    for (const char* a : kActs) {
      if (!(is >> tok) || tok != a) bad("unexpected activations");
    }
    Net n = init(0);
    if (!(is >> tok) || tok != "theta" || !(is >> n.theta)) bad("missing theta");
    for (size_t l = 0; l < n.layers.size(); ++l) {
      size_t idx;
      int o, i;
      if (!(is >> tok >> idx >> o >> i) || tok != "layer" || idx != l || o != n.layers[l].out ||
          i != n.layers[l].in)
        bad("malformed layer header");
      for (double& w : n.layers[l].w)
        if (!(is >> w)) bad("truncated weights");
      if (!(is >> tok) || tok != "bias") bad("missing bias");
      for (double& b : n.layers[l].b)
        if (!(is >> b)) bad("truncated bias");
    }
    return n;
  }
};

// Dataset rows (pipeline.hpp:98-133 shape): 8 numbers (A's four statistics, then
// B's) and a label A|B|0|1; '#' comments.
std::vector<Pair> parse_pairs(const std::string& text) {
  std::vector<Pair> rows;
  std::istringstream is(text);
  std::string line;
  int ln = 0;
  while (std::getline(is, line)) {
    ++ln;
    const size_t b = line.find_first_not_of(" \t\r\n");
    if (b == std::string::npos || line[b] == '#') continue;
    std::istringstream ls(line);
    Pair p{};
    for (int i = 0; i < 8; ++i) {
      double v;
      if (!(ls >> v)) throw ConfigError("dataset line " + std::to_string(ln) + ": expected 8 statistics and a label");
      (i < 4 ? p.a[i] : p.b[i - 4]) = v;
    }
    std::string lab, extra;
    if (!(ls >> lab)) throw ConfigError("dataset line " + std::to_string(ln) + ": missing label");
    if (lab == "A" || lab == "0") p.winner = 0;
    else if (lab == "B" || lab == "1") p.winner = 1;
    else throw ConfigError("dataset line " + std::to_string(ln) + ": bad label '" + lab + "'");
    if (ls >> extra) throw ConfigError("dataset line " + std::to_string(ln) + ": trailing tokens");
    rows.push_back(p);
  }
  if (rows.empty()) throw ConfigError("dataset has no rows");
  return rows;
}

void copy_out(const std::string& txt, char* buf, size_t len) {
  if (!buf || txt.size() + 1 > len) throw ConfigError("buffer too small (" + std::to_string(txt.size() + 1) + " bytes needed)");
  std::memcpy(buf, txt.c_str(), txt.size() + 1);
}

}  // namespace
}  // namespace psconv

using namespace psconv;

extern "C" {

int conv_model_stats(const conv_desc* d_in, int mode, const char* recipe, double* stats) {
  return guarded([&] {
    if (!d_in || !stats) throw ConfigError("null argument");
    conv_desc d = *d_in;
    validate_desc(d);
    const Schedule s = resolve_schedule(d, Recipe::parse(recipe ? recipe : ""), mode);
    model_stats(d, s, mode, stats);
  });
}

int ranker_train(const char* dataset, int epochs, double learning_rate, uint64_t seed, double split,
                 char* weights, size_t len, double* acc) {
  return guarded([&] {
    if (!dataset) throw ConfigError("null dataset");
    if (epochs < 0 || learning_rate <= 0) throw ConfigError("bad training hyper-parameters");
    if (split <= 0.0 || split > 1.0) throw ConfigError("split must be in (0, 1]");
    std::vector<Pair> all = parse_pairs(dataset);
    // seeded shuffle, hold out floor((1 - split) * n) rows (pipeline.hpp:151-174 protocol)
    Rng rng(seed ^ 0x9E3779B97F4A7C15ull);
    for (size_t i = all.size(); i > 1; --i) std::swap(all[i - 1], all[rng.below(i)]);
    const size_t hold = size_t(std::floor(double(all.size()) * (1.0 - split)));
    if (hold >= all.size()) throw ConfigError("split leaves no training rows");
    std::vector<Pair> tr(all.begin(), all.end() - long(hold)), ho(all.end() - long(hold), all.end());
    const Net n = Net::train(tr, epochs, learning_rate, seed, 32);
    copy_out(n.save(), weights, len);
    if (acc) {
      acc[0] = n.accuracy(tr);
      acc[1] = ho.empty() ? -1.0 : n.accuracy(ho);
    }
  });
}

int ranker_compare(const char* weights, const double* a, const double* b, double* prob) {
  int out = -1;
  const int rc = guarded([&] {
    if (!weights || !a || !b) throw ConfigError("null argument");
    const Net n = Net::load(weights);
    if (prob) n.prob(a, b, prob);
    out = n.compare(a, b);
  });
  return rc == PSCONV_OK ? out : -rc;
}

int conv_select_topk_dnn(const conv_desc* d_in, int mode, int k, const char* weights, char* buf, size_t len,
                         double* symmetry) {
  int written = 0;
  const int rc = guarded([&] {
    if (!d_in || !weights || k < 1) throw ConfigError("bad argument");
    conv_desc d = *d_in;
    validate_desc(d);
    const Net net = Net::load(weights);
    auto cands = candidate_schedules(d, mode);
    if (cands.empty()) throw ConfigError("no GPU schedule for this descriptor");
    struct E {
      std::string id;
      double cost, st[4];
      int wins = 0;
    };
    std::vector<E> es;
    for (const auto& s : cands) {
      E e;
      e.id = s.recipe_id;
      e.cost = model_schedule(d, s, mode).us_total;
      model_stats(d, s, mode, e.st);
      es.push_back(e);
    }
    std::sort(es.begin(), es.end(), [](const E& a, const E& b) { return a.id < b.id; });
    // tournament (dnnrank.hpp:394-429): every unordered pair plays once
    int64_t consistent = 0, games = 0;
    for (size_t i = 0; i < es.size(); ++i)
      for (size_t j = i + 1; j < es.size(); ++j) {
        const int o = net.compare(es[i].st, es[j].st);
        if (o == 0) ++es[i].wins;
        if (o == 1) ++es[j].wins;
        const int r = net.compare(es[j].st, es[i].st);
        consistent += (o == 2 && r == 2) || (o == 0 && r == 1) || (o == 1 && r == 0);
        ++games;
      }
    std::stable_sort(es.begin(), es.end(), [](const E& a, const E& b) {
      if (a.wins != b.wins) return a.wins > b.wins;
      if (a.cost != b.cost) return a.cost < b.cost;
      return a.id < b.id;
    });
    if (symmetry) *symmetry = games ? double(consistent) / double(games) : 1.0;
    std::string txt;
    for (int i = 0; i < k && i < int(es.size()); ++i) {
      txt += (i ? "\n" : "") + es[size_t(i)].id;
      ++written;
    }
    copy_out(txt, buf, len);
  });
  return rc == PSCONV_OK ? written : -rc;
}

}  // extern "C"
