// hawkes_b200/hmc.hpp — cut-posterior Hamiltonian Monte Carlo on the B200
// engine's log-likelihood gradient.
//
// The reference samples Theta = (mu0, tau_t, xi0, sigma_x, sigma_t) with a
// fixed-order univariate random-walk Metropolis sweep (mcmc.hpp:157-181) and
// has no gradient.  This driver keeps everything else of the reference's cut
// posterior unchanged and replaces only the Theta update:
//
//   * target in z = log Theta: the same posterior the reference's sampler
//     targets, ell(e^z) + PriorSpec::log_density(e^z) + sum z (the log-scale
//     proposal's Jacobian, mcmc.hpp:165-171);
//   * one HMC transition per iteration: `leapfrog_steps` leapfrog steps with
//     a diagonal metric (`scales`), every step one full log-likelihood +
//     gradient evaluation on the GPU (hk_eval), then a Metropolis test on the
//     Hamiltonian; non-finite energies reject (mcmc.hpp:168);
//   * step size adapted by dual averaging during burn-in (Hoffman & Gelman
//     2014, section 3.2), frozen afterwards so the post-burn-in kernel is fixed
//     (mcmc.hpp:99-111 convention);
//   * the X refresh is by default the reference's own resample_locations
//     (mcmc.hpp:80-97) on its own RNG stream (location_rng_, seeded like
//     mcmc.hpp:126), so the sequence of location draws is the reference's.
//     Because X does not depend on Theta (cut posterior), the next draw is
//     computed on a host thread while the GPU runs the current iteration's
//     leapfrog steps (overlap the resample).
//     HmcConfig::gpu_resample = true draws X on the GPU instead
//     (hawkes_b200/regions.hpp: the same algorithm, one thread per event,
//     Philox-keyed by (seed, refresh index)) straight into the engine's
//     device locations: no host resample, no location upload.
//
// Output is the reference's ChainOutput (mcmc.hpp:63-76), so its chain CSV /
// sidecar writers and diagnostics apply unchanged.  The per-iteration time
// split (resample wait / location upload / evaluations) is reported in
// HmcTiming.
#ifndef HAWKES_B200_HMC_HPP
#define HAWKES_B200_HMC_HPP

#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <future>
#include <memory>
#include <random>
#include <stdexcept>
#include <utility>
#include <vector>

#include "hawkes/geo.hpp"
#include "hawkes/mcmc.hpp"
#include "hawkes_b200/engine.hpp"
#include "hawkes_b200/regions.hpp"

namespace hawkes::b200 {

struct HmcConfig {
  ChainConfig chain;              // iterations, burn_in, seed, initial, prior, refresh_period
  int leapfrog_steps = 8;
  double step_size = 0.02;        // initial leapfrog step in log-parameter space
  double target_accept = 0.75;    // dual-averaging target
  bool adapt = true;
  std::array<double, kParamCount> scales{1, 1, 1, 1, 1};  // diagonal metric (inverse mass sqrt)
  int n_gpus = 1;
  bool gpu_resample = false;      // X refresh on the GPU (Philox stream) instead of the reference's
};

struct HmcTiming {
  double resample_wait = 0.0;   // seconds the chain waited for the prefetched X draw
  double set_locations = 0.0;   // seconds uploading X
  double evaluate = 0.0;        // seconds in log-likelihood + gradient evaluations
  std::size_t evaluations = 0;
};

class HmcSampler {
 public:
  HmcSampler(const HmcConfig& config, const Catalog& catalog, const RegionTable* regions)
      : cfg_(config),
        catalog_(&catalog),
        regions_(regions),
        engine_(catalog, config.n_gpus, config.chain.initial.variant),
        location_rng_(config.chain.seed),
        param_rng_(config.chain.seed ^ 0x9e3779b97f4a7c15ull) {
    cfg_.chain.validate();
    if (cfg_.leapfrog_steps < 1) throw std::invalid_argument("HmcConfig: leapfrog_steps must be >= 1");
    if (!(cfg_.step_size > 0.0)) throw std::invalid_argument("HmcConfig: step_size must be positive");
    if (catalog.coarse_only() && regions == nullptr)
      throw std::invalid_argument("Sampler: coarse-only catalog requires a region table");
    const HawkesParams& p0 = cfg_.chain.initial;
    z_ = {std::log(p0.mu0), std::log(p0.tau_t), std::log(p0.xi0), std::log(p0.sigma_x),
          std::log(p0.sigma_t)};
    eps_ = cfg_.step_size;
    log_eps_bar_ = 0.0;
    mu_ = std::log(10.0 * eps_);
    if (regions_ != nullptr && cfg_.gpu_resample) {
      gpu_regions_ = std::make_unique<GpuRegions>(catalog, *regions_);
      engine_.resample_locations(gpu_regions_->get(), cfg_.chain.seed, refresh_count_++);
    } else if (regions_ != nullptr) {
      auto [lon, lat] = hawkes::resample_locations(*catalog_, *regions_, location_rng_);
      engine_.set_locations(lon, lat);
    }
    value_ = log_density(z_, grad_);
    loglik_ = last_ll_;
  }

  ChainOutput run() {
    const auto start = std::chrono::steady_clock::now();
    ChainOutput out;
    std::future<std::pair<std::vector<double>, std::vector<double>>> next;
    const bool host_resample = regions_ != nullptr && !cfg_.gpu_resample;
    auto prefetch = [&] {
      if (host_resample)
        next = std::async(std::launch::async,
                          [this] { return hawkes::resample_locations(*catalog_, *regions_, location_rng_); });
    };
    prefetch();
    for (std::size_t iter = 0; iter < cfg_.chain.iterations; ++iter) {
      if (regions_ != nullptr && iter % cfg_.chain.refresh_period == 0) {
        if (host_resample) {
          auto t0 = clock::now();
          auto [lon, lat] = next.get();  // X draw for this iteration (reference stream order)
          auto t1 = clock::now();
          prefetch();                    // the next draw overlaps this iteration's GPU work
          engine_.set_locations(lon, lat);
          auto t2 = clock::now();
          timing_.resample_wait += seconds(t0, t1);
          timing_.set_locations += seconds(t1, t2);
        } else {
          auto t0 = clock::now();
          engine_.resample_locations(gpu_regions_->get(), cfg_.chain.seed, refresh_count_++);
          timing_.resample_wait += seconds(t0, clock::now());
        }
        value_ = log_density(z_, grad_);  // the target changed with X
        loglik_ = last_ll_;  // a rejected transition keeps these locations' LL
      }
      const bool in_burn_in = iter < cfg_.chain.burn_in;
      const double accept_prob = transition();
      for (std::size_t k = 0; k < kParamCount; ++k) ++out.proposals[k];
      if (last_accepted_)
        for (std::size_t k = 0; k < kParamCount; ++k) ++out.accepts[k];
      if (cfg_.adapt && in_burn_in) adapt(iter + 1, accept_prob);
      if (cfg_.adapt && iter + 1 == cfg_.chain.burn_in) eps_ = std::exp(log_eps_bar_);
      if (!in_burn_in) {
        out.draws.push_back(theta());
        out.loglik_trace.push_back(loglik_);
      }
    }
    if (next.valid()) next.wait();
    for (std::size_t k = 0; k < kParamCount; ++k) out.final_steps[k] = eps_ * cfg_.scales[k];
    out.seed = cfg_.chain.seed;
    out.seconds = seconds(start, clock::now());
    return out;
  }

  const HmcTiming& timing() const { return timing_; }
  double step_size() const { return eps_; }

 private:
  using clock = std::chrono::steady_clock;
  using Vec = std::array<double, kParamCount>;

  static double seconds(clock::time_point a, clock::time_point b) {
    return std::chrono::duration<double>(b - a).count();
  }

  std::array<double, kParamCount> theta() const {
    std::array<double, kParamCount> t{};
    for (std::size_t k = 0; k < kParamCount; ++k) t[k] = std::exp(z_[k]);
    return t;
  }

  HawkesParams params_of(const Vec& z) const {
    HawkesParams p = cfg_.chain.initial;
    p.mu0 = std::exp(z[0]);
    p.tau_t = std::exp(z[1]);
    p.xi0 = std::exp(z[2]);
    p.sigma_x = std::exp(z[3]);
    p.sigma_t = std::exp(z[4]);
    return p;
  }

  // log target in z = log Theta and its gradient.
  double log_density(const Vec& z, Vec& g) {
    const HawkesParams p = params_of(z);
    for (double v : {p.mu0, p.tau_t, p.xi0, p.sigma_x, p.sigma_t})
      if (!(v > 0.0) || !std::isfinite(v)) {  // a divergent trajectory: rejected
        last_ll_ = -INFINITY;
        return -INFINITY;
      }
    std::array<double, 5> gl{};
    const auto t0 = clock::now();
    const double ll = engine_.log_likelihood_and_gradient(p, p.variant, gl);
    timing_.evaluate += seconds(t0, clock::now());
    ++timing_.evaluations;
    last_ll_ = ll;
    const Vec th = {p.mu0, p.tau_t, p.xi0, p.sigma_x, p.sigma_t};
    double lp = ll;
    for (std::size_t k = 0; k < kParamCount; ++k) {
      const double m = cfg_.chain.prior.log_mean[k], sd = cfg_.chain.prior.log_sd[k];
      const double u = (z[k] - m) / sd;
      lp += -std::log(sd) - 0.5 * u * u;  // prior density of log Theta (Jacobian included)
      g[k] = th[k] * gl[k] - u / sd;
    }
    return lp;
  }

  // One HMC transition; returns the acceptance probability.
  double transition() {
    std::normal_distribution<double> normal(0.0, 1.0);
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    Vec p{}, z = z_, g = grad_;
    for (std::size_t k = 0; k < kParamCount; ++k) p[k] = normal(param_rng_);
    const double u = unit(param_rng_);
    auto kinetic = [&](const Vec& m) {
      double s = 0.0;
      for (std::size_t k = 0; k < kParamCount; ++k) s += 0.5 * m[k] * m[k];
      return s;
    };
    const double h0 = -value_ + kinetic(p);
    double val = value_;
    double ll = loglik_;
    bool finite = true;
    for (std::size_t k = 0; k < kParamCount; ++k) p[k] += 0.5 * eps_ * cfg_.scales[k] * g[k];
    for (int s = 0; s < cfg_.leapfrog_steps && finite; ++s) {
      for (std::size_t k = 0; k < kParamCount; ++k) z[k] += eps_ * cfg_.scales[k] * p[k];
      val = log_density(z, g);
      ll = last_ll_;
      finite = std::isfinite(val);
      const double w = (s + 1 == cfg_.leapfrog_steps) ? 0.5 : 1.0;
      for (std::size_t k = 0; k < kParamCount && finite; ++k) p[k] += w * eps_ * cfg_.scales[k] * g[k];
    }
    const double h1 = finite ? -val + kinetic(p) : INFINITY;
    const double a = std::isfinite(h1) ? std::min(1.0, std::exp(h0 - h1)) : 0.0;
    last_accepted_ = std::log(u) < h0 - h1;
    if (last_accepted_) {
      z_ = z;
      grad_ = g;
      value_ = val;
      loglik_ = ll;
    }
    return a;
  }

  // Dual averaging of log eps (Hoffman & Gelman 2014, eqs. 5-6).
  void adapt(std::size_t m, double accept_prob) {
    const double gamma = 0.05, t0 = 10.0, kappa = 0.75;
    const double w = 1.0 / (static_cast<double>(m) + t0);
    h_bar_ = (1.0 - w) * h_bar_ + w * (cfg_.target_accept - accept_prob);
    const double log_eps = mu_ - std::sqrt(static_cast<double>(m)) / gamma * h_bar_;
    const double mk = std::pow(static_cast<double>(m), -kappa);
    log_eps_bar_ = mk * log_eps + (1.0 - mk) * log_eps_bar_;
    eps_ = std::exp(log_eps);
  }

  HmcConfig cfg_;
  const Catalog* catalog_;
  const RegionTable* regions_;
  Engine engine_;
  std::mt19937_64 location_rng_;
  std::mt19937_64 param_rng_;
  std::unique_ptr<GpuRegions> gpu_regions_;  // gpu_resample only
  std::uint64_t refresh_count_ = 0;
  Vec z_{}, grad_{};
  double value_ = 0.0, loglik_ = 0.0, last_ll_ = 0.0;
  double eps_ = 0.02, mu_ = 0.0, h_bar_ = 0.0, log_eps_bar_ = 0.0;
  bool last_accepted_ = false;
  HmcTiming timing_;

 public:
  double loglik() const { return loglik_; }
};

/// Cut-posterior HMC chain (regions: county polygons; X refreshed every
/// refresh_period iterations by the reference's resample_locations).
inline ChainOutput run_cut_posterior_hmc(const HmcConfig& config, const Catalog& catalog,
                                         const RegionTable& regions, HmcTiming* timing = nullptr) {
  HmcSampler s(config, catalog, &regions);
  ChainOutput out = s.run();
  if (timing) *timing = s.timing();
  return out;
}

/// HMC with the event locations held fixed (the ordinary posterior).
inline ChainOutput run_fixed_posterior_hmc(const HmcConfig& config, const Catalog& catalog,
                                           HmcTiming* timing = nullptr) {
  HmcSampler s(config, catalog, nullptr);
  ChainOutput out = s.run();
  if (timing) *timing = s.timing();
  return out;
}

}  // namespace hawkes::b200

#endif  // HAWKES_B200_HMC_HPP
