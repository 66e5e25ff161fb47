#include "hk_host.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "hk_device.cuh"
#include "hk_fgt.cuh"

namespace hk {

void validate_catalog(const double* t, const double* x, const double* y, const double* d,
                      std::size_t n, bool coarse_only) {
  if (n == 0) throw std::invalid_argument("Catalog: need at least one event");
  if (n >= (std::size_t{1} << 31) - 1024)
    throw std::invalid_argument("Catalog: more than 2^31 events is not supported");
  for (std::size_t i = 0; i < n; ++i) {
    if (!(t[i] >= 0.0) || !std::isfinite(t[i]))
      throw std::invalid_argument("Catalog: event " + std::to_string(i) + " has invalid time");
    if (!(d[i] > 0.0))
      throw std::invalid_argument("Catalog: event " + std::to_string(i) +
                                  " has nonpositive density");
    if (!coarse_only && (!std::isfinite(x[i]) || !std::isfinite(y[i])))
      throw std::invalid_argument("Catalog: event " + std::to_string(i) +
                                  " has non-finite location");
    if (i > 0 && t[i - 1] > t[i])
      throw std::invalid_argument("Catalog: times not sorted at index " + std::to_string(i));
  }
}

void validate_params(const ParamsIn& p) {
  auto pos = [](double v, const char* name) {
    if (!(v > 0.0) || !std::isfinite(v))
      throw std::invalid_argument(std::string("HawkesParams: ") + name +
                                  " must be positive and finite");
  };
  pos(p.mu0, "mu0");
  pos(p.tau_t, "tau_t");
  pos(p.xi0, "xi0");
  pos(p.sigma_x, "sigma_x");
  pos(p.sigma_t, "sigma_t");
  pos(p.area, "area");
  if (p.variant != 0 && p.variant != 1) throw std::invalid_argument("unknown variant");
}

namespace {

// mt19937_64 (the standard's parameters).
class Mt64 {
 public:
  explicit Mt64(std::uint64_t seed) {
    s_[0] = seed;
    for (int i = 1; i < kN; ++i)
      s_[i] = 6364136223846793005ULL * (s_[i - 1] ^ (s_[i - 1] >> 62)) + static_cast<std::uint64_t>(i);
    idx_ = kN;
  }
  std::uint64_t operator()() {
    if (idx_ >= kN) twist();
    std::uint64_t z = s_[idx_++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
  }

 private:
  static constexpr int kN = 312, kM = 156;
  void twist() {
    constexpr std::uint64_t kUpper = ~std::uint64_t{0} << 31, kLower = ~kUpper;
    for (int i = 0; i < kN; ++i) {
      const std::uint64_t v = (s_[i] & kUpper) | (s_[(i + 1) % kN] & kLower);
      s_[i] = s_[(i + kM) % kN] ^ (v >> 1) ^ ((v & 1) ? 0xB5026F5AA96619E9ULL : 0);
    }
    idx_ = 0;
  }
  std::uint64_t s_[kN];
  int idx_;
};

// libstdc++ generate_canonical<double, 53> over a 64-bit engine (one draw),
// then uniform_real_distribution's affine map u*(b-a)+a, which the
// reference's build (-O3 -march=native, GCC's default -ffp-contract=fast)
// contracts into one fused multiply-add.
double uniform(Mt64& g, double a, double b) {
  double u = static_cast<double>(g()) / 18446744073709551616.0;
  if (u >= 1.0) u = std::nextafter(1.0, 0.0);
  return std::fma(u, b - a, a);
}

}  // namespace

void benchmark_catalog(std::size_t n, std::uint64_t seed, double* t, double* x, double* y,
                       double* d) {
  Mt64 g(seed);
  std::vector<double> tt(n), xx(n), yy(n), dd(n);
  for (std::size_t i = 0; i < n; ++i) {  // braced-init order: t, lon, lat, density
    tt[i] = uniform(g, 0.0, 100.0);
    xx[i] = uniform(g, -5.0, 5.0);
    yy[i] = uniform(g, -5.0, 5.0);
    dd[i] = uniform(g, 10.0, 5000.0);
  }
  std::vector<std::size_t> order(n);
  std::iota(order.begin(), order.end(), std::size_t{0});
  std::stable_sort(order.begin(), order.end(),
                   [&](std::size_t a, std::size_t b) { return tt[a] < tt[b]; });
  for (std::size_t i = 0; i < n; ++i) {
    t[i] = tt[order[i]];
    x[i] = xx[order[i]];
    y[i] = yy[order[i]];
    d[i] = dd[order[i]];
  }
}

void make_exp2_table(double* out, int n) {
  int b = 0;
  while ((1 << b) < n) ++b;
  for (int j = 0; j < n; ++j) {
    // long double exp2 (64-bit significand), rounded once to double
    const double v = static_cast<double>(std::exp2l(static_cast<long double>(j) / n));
    std::uint64_t u;
    std::memcpy(&u, &v, sizeof u);
    u -= static_cast<std::uint64_t>(j) << (32 + 20 - b);  // high word minus (j << (20 - b))
    std::memcpy(&out[j], &u, sizeof u);
  }
}

std::vector<std::size_t> partition_make(std::size_t n, std::size_t g) {
  if (g == 0) throw std::invalid_argument("Partition: worker count must be positive");
  if (g > n) throw std::invalid_argument("Partition: more workers than terms");
  std::vector<std::size_t> b(g + 1, 0);
  const std::size_t base = n / g, rem = n % g;
  for (std::size_t w = 0; w < g; ++w) b[w + 1] = b[w] + base + (w < rem ? 1 : 0);
  return b;
}

void tie_bounds(const std::vector<double>& t, std::vector<int>& lb, std::vector<int>& ub) {
  const std::size_t n = t.size();
  lb.assign(n, 0);
  ub.assign(n, 0);
  std::size_t i = 0;
  while (i < n) {
    std::size_t k = i;
    while (k < n && t[k] == t[i]) ++k;
    for (std::size_t m = i; m < k; ++m) {
      lb[m] = static_cast<int>(i);
      ub[m] = static_cast<int>(k);
    }
    i = k;
  }
}

std::vector<std::size_t> plan_shards(const std::vector<int>& lb, std::size_t g, double beta) {
  const std::size_t n = lb.size();
  if (g == 0) throw std::invalid_argument("plan_shards: shard count must be positive");
  if (g > n) throw std::invalid_argument("plan_shards: more shards than rows");
  std::vector<double> cum(n + 1, 0.0);
  const double row_bg = background_cost(n) * static_cast<double>(n - 1);
  for (std::size_t i = 0; i < n; ++i) cum[i + 1] = cum[i] + row_bg + beta * lb[i];
  std::vector<std::size_t> b(g + 1, 0);
  b[g] = n;
  for (std::size_t s = 1; s < g; ++s) {
    const double target = cum[n] * static_cast<double>(s) / static_cast<double>(g);
    std::size_t r = static_cast<std::size_t>(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
    r = std::max(r, b[s - 1] + 1);            // every shard non-empty
    r = std::min(r, n - (g - s));
    b[s] = r;
  }
  return b;
}

int plan_items(const std::vector<int>& lb, const std::vector<int>& ub, int n, int rb, int re,
               int kBI, std::vector<Item>& items, int window, int cell_tiles) {
  items.clear();
  const int npad = (n + kBJ - 1) / kBJ * kBJ;
  const int ntiles = cell_tiles > 0 ? cell_tiles : npad / kBJ;
  const int nblocks = (re - rb + kBI - 1) / kBI;
  const int G = std::max(1, window);
  // Column chunks per row block ("slots"): about kItemTarget work items
  // (heaviest first, so the tail stays short), at most kMaxSlots, and chunks
  // of at most kMaxItemTiles tiles (the kernel classifies an item's tiles in
  // shared memory).  The partial-sum buffer [slots][5][rows] (40 B per row
  // and slot) is therefore O(N) with a bounded constant: 17 slots at
  // N = 1e6 (0.68 GB), 20 at N = 1e7 (8 GB).  HK_ITEM_TARGET overrides the
  // item target (tuning).
  int target = G > 1 ? kItemTargetVarying : kItemTarget;
  if (const char* e = std::getenv("HK_ITEM_TARGET")) target = std::max(1, std::atoi(e));
  int slots = std::min(kMaxSlots, (target + nblocks - 1) / nblocks);
  slots = std::max(slots, (ntiles + kMaxItemTiles - 1) / kMaxItemTiles);
  slots = std::max(1, std::min(slots, ntiles));
  const int per = (ntiles + slots - 1) / slots;
  slots = (ntiles + per - 1) / per;
  struct Cand {
    Item it;
    double cost;
  };
  std::vector<Cand> cands;
  cands.reserve(static_cast<std::size_t>(nblocks) * slots);
  for (int b = 0; b < nblocks; ++b) {
    // the block's own rows [r0, r1) and the rows [w0, w1) it is classified
    // against (its window)
    const int r0 = rb + b * kBI, r1 = std::min(re, r0 + kBI);
    // near-equal windows of <= G blocks; rperm holds G*kBI slots per window
    const int nw = window_count(nblocks, G);
    const int w = window_of_block(b, nblocks, nw);
    const int b0 = window_first_block(w, nblocks, nw);
    const int w0 = G > 1 ? rb + b0 * kBI : r0;
    const int w1 = G > 1 ? std::min(re, rb + window_first_block(w + 1, nblocks, nw) * kBI) : r1;
    const int pos = G > 1 ? w * G * kBI + (b - b0) * kBI : -1;
    const int lbmin = lb[w0], ubmax = ub[w1 - 1];
    // Hermite-expansion checkpoint of this block (homogeneous plan): the
    // prefix of whole tiles before the checkpoint's first row (hk_fgt.cu)
    const int xt = G > 1 ? 0 : lb[rb + (b / kFgtBlocks) * kFgtBlocks * kBI] / kBJ;
    for (int c = 0; c < slots; ++c) {
      const int tb = c * per, te = std::min(ntiles, (c + 1) * per);
      double cost = 0.0;
      // cell tiles hold columns of every time: the work of a row block grows
      // with the columns before it (its rank in time)
      if (cell_tiles > 0) cost = static_cast<double>(te - tb) * (r0 + kBI);
      for (int J = tb; cell_tiles <= 0 && J < te; ++J) {
        const int j0 = J * kBJ, j1 = j0 + kBJ;
        const double alpha = background_cost(static_cast<std::size_t>(n));
        if (j1 <= lbmin) cost += alpha + kCostBeta;
        else if (j0 >= ubmax && j1 <= n) cost += alpha;
        else cost += kCostAlphaDirect + kCostBeta + 8.0;
      }
      cands.push_back({Item{w0, w1, tb, te, c, pos, xt}, cost * (r1 - r0)});
    }
  }
  std::stable_sort(cands.begin(), cands.end(),
                   [](const Cand& a, const Cand& b) { return a.cost > b.cost; });
  items.reserve(cands.size());
  for (const auto& c : cands) items.push_back(c.it);
  return slots;
}

int plan_items_fgt(const std::vector<int>& lb, const std::vector<int>& ub, int n, int rb, int re,
                   int kBI, std::vector<Item>& items) {
  items.clear();
  const int ntiles = (n + kBJ - 1) / kBJ;
  const int nblocks = (re - rb + kBI - 1) / kBI;
  struct Span {
    int r0, r1, tb, te;
  };
  std::vector<Span> spans(nblocks);
  int max_tiles = 1;
  for (int b = 0; b < nblocks; ++b) {
    const int r0 = rb + b * kBI, r1 = std::min(re, r0 + kBI);
    const int xt = lb[rb + (b / kFgtBlocks) * kFgtBlocks * kBI] / kBJ;  // as plan_items' Item::xt
    const int te = std::min(ntiles, (ub[r1 - 1] + kBJ - 1) / kBJ);     // beyond: background only
    spans[b] = {r0, r1, xt, std::max(te, xt + 1)};
    max_tiles = std::max(max_tiles, spans[b].te - spans[b].tb);
  }
  const int slots = (max_tiles + kMaxItemTiles - 1) / kMaxItemTiles;
  struct Cand {
    Item it;
    double cost;
  };
  std::vector<Cand> cands;
  for (const Span& sp : spans) {
    const int per = (sp.te - sp.tb + slots - 1) / slots;
    for (int c = 0; c < slots; ++c) {
      const int tb = std::min(sp.te, sp.tb + c * per), te = std::min(sp.te, tb + per);
      cands.push_back({Item{sp.r0, sp.r1, tb, std::max(te, tb), c, -1, sp.tb},
                       static_cast<double>(te - tb) * (sp.r1 - sp.r0)});
    }
  }
  std::stable_sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) { return a.cost > b.cost; });
  for (const auto& c : cands) items.push_back(c.it);
  return slots;
}

EvalCoef make_coef(const ParamsIn& p, double t_min, double t_max, double d2_max, double q_max) {
  EvalCoef c{};
  c.mu0 = p.mu0;
  c.tau_t = p.tau_t;
  c.xi0 = p.xi0;
  c.sigma_x = p.sigma_x;
  c.sigma_t = p.sigma_t;
  c.tau_prec = 1.0 / p.tau_t;
  c.sx_prec = 1.0 / p.sigma_x;
  c.omega = 1.0 / p.sigma_t;
  const double inv_area = 1.0 / p.area;
  c.a = p.mu0 * inv_area * c.tau_prec * kInvSqrt2Pi;         // model.hpp:203-205
  c.c = p.xi0 * c.omega * c.sx_prec * c.sx_prec * kInv2Pi;   // model.hpp:207-210
  c.half_s2 = 0.5 * c.sx_prec * c.sx_prec;                   // model.hpp:151
  c.Kb = -0.5 * c.tau_prec * c.tau_prec * kLog2eT;
  c.Kq0 = -c.half_s2 * kLog2eT;
  c.Kw = -c.omega * kLog2eT;
  c.t_end = t_max;
  c.u_scale = c.tau_prec * 0.7071067811865476;
  c.two_tau2 = 2.0 * p.tau_t * p.tau_t;
  c.bg_expansion = 1;
  c.varying = p.variant;
  const double span = t_max - t_min;
  const double qm = p.variant ? q_max : 1.0;
  const double bound = std::max({span * span * (-c.Kb), d2_max * (-c.Kq0) * qm + span * (-c.Kw),
                                 span * (-c.Kw)});
  // NaN/inf bounds fall through to the checked path.
  c.mode = bound < kExactArg ? kExact : (bound < kCheckArg ? kFlush : kChecked);
  return c;
}

}  // namespace hk
