// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the UNMODIFIED reference headers under
// /root/reference/proj/include (compiled in place by oracle/Makefile into
// oracle/_ref/libhawkes_ref.so).  It exposes the reference's own CPU path to
// the parity tests, the golden-vector generator (tests/golden/make_golden.py)
// and bench.py's cpu_baseline / `--impl reference` legs.  No reference
// source is copied here: every function below only marshals plain arrays
// into the reference's types and calls the reference's functions.
//
// Reference entry points wrapped (file:line under proj/include/hawkes/):
//   benchmark_catalog          engine.hpp:251-259
//   log_likelihood             engine.hpp:101-110  (Partition::make :27-40)
//   slice_log_likelihood       engine.hpp:65-83
//   event_contribution         model.hpp:225-230
//   naive_log_likelihood       simulate.hpp:121-136
//   pair_rate / integral_term  model.hpp:234-250 / :175-180
//   gaussian_pdf / gaussian_cdf model.hpp:27-34
//   LikelihoodWorkspace<double> engine.hpp:117-229
#include <cmath>
#include <cstdint>
#include <random>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "hawkes/engine.hpp"
#include "hawkes/model.hpp"
#include "hawkes/simulate.hpp"
#include "hawkes/types.hpp"

using namespace hawkes;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::out_of_range& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

std::vector<Event> to_events(const double* t, const double* x, const double* y, const double* d,
                             std::size_t n) {
  std::vector<Event> ev(n);
  for (std::size_t i = 0; i < n; ++i) ev[i] = Event{t[i], x[i], y[i], "", d[i]};
  return ev;
}

// params layout: mu0, tau_t, xi0, sigma_x, sigma_t, area
HawkesParams to_params(const double* p, int variant) {
  HawkesParams hp;
  hp.mu0 = p[0];
  hp.tau_t = p[1];
  hp.xi0 = p[2];
  hp.sigma_x = p[3];
  hp.sigma_t = p[4];
  hp.area = p[5];
  hp.variant = variant ? Variant::varying : Variant::constant;
  return hp;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_benchmark_catalog(std::size_t n, std::uint64_t seed, double* t, double* x, double* y,
                          double* d) {
  return guarded([&] {
    const Catalog c = benchmark_catalog(n, seed);
    for (std::size_t i = 0; i < n; ++i) {
      t[i] = c[i].t;
      x[i] = c[i].lon;
      y[i] = c[i].lat;
      d[i] = c[i].density;
    }
  });
}

int ref_log_likelihood(const double* t, const double* x, const double* y, const double* d,
                       std::size_t n, const double* params, int variant, std::size_t workers,
                       int single, double* out) {
  return guarded([&] {
    const Catalog c(to_events(t, x, y, d, n));
    *out = log_likelihood(c, to_params(params, variant), make_partition(n, workers),
                          single ? Precision::single : Precision::dbl);
  });
}

int ref_naive_log_likelihood(const double* t, const double* x, const double* y, const double* d,
                             std::size_t n, const double* params, int variant, double* out) {
  return guarded([&] {
    const Catalog c(to_events(t, x, y, d, n));
    *out = naive_log_likelihood(c, to_params(params, variant));
  });
}

int ref_event_contribution(const double* t, const double* x, const double* y, const double* d,
                           std::size_t n, const double* params, int variant, std::size_t row,
                           double* out) {
  return guarded([&] {
    const Catalog c(to_events(t, x, y, d, n));
    *out = event_contribution(to_params(params, variant), c, row);
  });
}

// Per-row contributions ell_i = slice_log_likelihood(d, p, i, i+1) for an
// arbitrary row list, spread over `threads` std::threads (row r goes to
// thread r % threads).  This is the reference's own row kernel; it is what
// the sampled-row parity tests and the CPU baseline time.
int ref_rows(const double* t, const double* x, const double* y, const double* d, std::size_t n,
             const double* params, int variant, const std::uint64_t* rows, std::size_t nrows,
             std::size_t threads, double* out) {
  return guarded([&] {
    const Catalog c(to_events(t, x, y, d, n));
    const HawkesParams p = to_params(params, variant);
    p.validate();
    const auto data = EvalData<double>::from(c, p.variant);
    for (std::size_t r = 0; r < nrows; ++r)
      if (rows[r] >= n) throw std::out_of_range("ref_rows: row index out of range");
    const std::size_t g = threads == 0 ? 1 : threads;
    auto work = [&](std::size_t w) {
      for (std::size_t r = w; r < nrows; r += g)
        out[r] = slice_log_likelihood(data, p, rows[r], rows[r] + 1);
    };
    std::vector<std::thread> pool;
    for (std::size_t w = 1; w < g; ++w) pool.emplace_back(work, w);
    work(0);
    for (auto& th : pool) th.join();
  });
}

int ref_pair_rate(const double* params, int variant, const double* source5, const double* target5,
                  double* out) {
  return guarded([&] {
    const Event s{source5[0], source5[1], source5[2], "", source5[3]};
    const Event tg{target5[0], target5[1], target5[2], "", target5[3]};
    *out = pair_rate(to_params(params, variant), s, tg);
  });
}

int ref_integral_term(const double* params, double t_n, double t_end, double* out) {
  return guarded([&] { *out = integral_term(to_params(params, 0), t_n, t_end); });
}

double ref_gaussian_pdf(double z) { return gaussian_pdf(z); }
double ref_gaussian_cdf(double z) { return gaussian_cdf(z); }

// BASELINE config 5's county densities: grid x grid square
// counties, densities log-uniform on [1, 7.4e4] drawn in row-major county
// order from std::mt19937_64(seed) through std::uniform_real_distribution
// (the same draws as tools/cpp/cut_posterior_bench.cpp).
int ref_county_densities(int grid, std::uint64_t seed, double* out) {
  return guarded([&] {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> ulog(0.0, std::log(7.4e4));
    for (int k = 0; k < grid * grid; ++k) out[k] = std::exp(ulog(rng));
  });
}

// Partition::make, flattened to n_workers+1 boundaries.
int ref_partition(std::size_t n, std::size_t g, std::size_t* bounds) {
  return guarded([&] {
    const Partition p = make_partition(n, g);
    bounds[0] = 0;
    for (std::size_t w = 0; w < p.workers(); ++w) bounds[w + 1] = p.ranges[w].second;
  });
}

// Drives the reference LikelihoodWorkspace<double> through a scripted
// sequence: op 0 = evaluate_full, 1 = evaluate_proposal, 2 = commit_proposal.
// params_seq holds 6 doubles per step (ignored for commit).
int ref_workspace_script(const double* t, const double* x, const double* y, const double* d,
                         std::size_t n, int variant, std::size_t workers, const int* ops,
                         const double* params_seq, std::size_t steps, double* out) {
  return guarded([&] {
    const Catalog c(to_events(t, x, y, d, n));
    LikelihoodWorkspace<double> ws(c, variant ? Variant::varying : Variant::constant, workers);
    for (std::size_t s = 0; s < steps; ++s) {
      const HawkesParams p = to_params(params_seq + 6 * s, variant);
      out[s] = 0.0;
      if (ops[s] == 0) out[s] = ws.evaluate_full(p);
      else if (ops[s] == 1) out[s] = ws.evaluate_proposal(p);
      else ws.commit_proposal();
    }
  });
}

}  // extern "C"
