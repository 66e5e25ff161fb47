// HMC cut-posterior gate (include/hawkes_b200/hmc.hpp), against the
// reference's own MH sampler and diagnostics (mcmc.hpp, diagnostics.hpp):
//   1. degenerate point regions: the cut-posterior HMC chain equals the
//      fixed-location chain exactly (test_mcmc.cpp:212-231 analogue);
//   2. posterior agreement: HMC on the GPU and the reference's univariate MH
//      (CPU) give posterior means within 4 Monte Carlo standard errors on a
//      simulated catalog (acceptance.cpp:244-296 convention);
//   3. the HMC chain persists through the reference's chain CSV and sidecar
//      writers (io.hpp:129-156) and reads back exactly (read_chain_csv);
//   4. with real (square) regions every loglik_trace entry is the
//      log-likelihood of that draw at that iteration's locations (the
//      reference's location stream, replayed here), including after rejected
//      transitions that follow an X refresh.
// PASS/FAIL lines; exit status = number of failures.
#include <algorithm>
#include <cmath>
#include <random>
#include <cstdio>
#include <string>
#include <vector>

#include "hawkes/diagnostics.hpp"
#include "hawkes/io.hpp"
#include "hawkes/mcmc.hpp"
#include "hawkes/simulate.hpp"
#include "hawkes_b200/hmc.hpp"

using namespace hawkes;

namespace {

int failures = 0;

void report(const std::string& what, bool pass, const std::string& detail) {
  std::printf("%s: %s (%s)\n", pass ? "PASS" : "FAIL", what.c_str(), detail.c_str());
  std::fflush(stdout);
  if (!pass) ++failures;
}

struct PointSetup {  // acceptance.cpp:158-174
  Catalog tagged;
  RegionTable regions;
};

PointSetup point_regions(const Catalog& catalog) {
  RegionTable regions;
  std::vector<Event> tagged = catalog.events();
  for (std::size_t i = 0; i < tagged.size(); ++i) {
    const std::string id = "e" + std::to_string(i);
    regions.add(Region{id, true, {tagged[i].lon, tagged[i].lat}, {}, 1.0, tagged[i].lat});
    tagged[i].region_id = id;
  }
  return {Catalog(std::move(tagged)), std::move(regions)};
}

Catalog simulated() {
  SimConfig sim;
  sim.immigrant_rate = 2.0;
  sim.horizon = 100.0;
  sim.seed = 606;
  return simulate_catalog(sim);
}

ChainConfig base_config(const Catalog& catalog) {
  ChainConfig config;
  config.iterations = 3000;
  config.burn_in = 600;
  config.seed = 42;
  config.initial.mu0 = 0.5;
  config.initial.tau_t = 5.0;
  config.initial.xi0 = 0.5;
  config.initial.sigma_x = 0.1;
  config.initial.sigma_t = 2.0;
  config.initial.area = domain_area(catalog);
  // mu0 and tau_t are weakly identified by the trigger-generated data
  // (README "Simulator vs. model background"); an informative log-normal
  // prior on both (shared by both samplers) keeps the posterior proper and
  // the comparison sharp.
  config.prior.log_mean[0] = std::log(0.5);
  config.prior.log_sd[0] = 0.5;
  config.prior.log_mean[1] = std::log(5.0);
  config.prior.log_sd[1] = 0.5;
  return config;
}

void point_regions_collapse() {
  const Catalog catalog = simulated();
  const PointSetup setup = point_regions(catalog);
  b200::HmcConfig cfg;
  cfg.chain = base_config(catalog);
  cfg.chain.iterations = 300;
  cfg.chain.burn_in = 100;
  const ChainOutput cut = b200::run_cut_posterior_hmc(cfg, setup.tagged, setup.regions);
  const ChainOutput fixed = b200::run_fixed_posterior_hmc(cfg, catalog);
  bool same = cut.draws.size() == fixed.draws.size() && cut.accepts == fixed.accepts;
  for (std::size_t i = 0; same && i < cut.draws.size(); ++i) same = cut.draws[i] == fixed.draws[i];
  report("point regions: cut-posterior HMC == fixed-location HMC", same,
         std::to_string(cut.draws.size()) + " draws, accepts " + std::to_string(cut.accepts[0]));

  // the reference's chain persistence on the HMC output
  const std::string csv = "/tmp/hk_test_hmc_chain.csv", side = "/tmp/hk_test_hmc_chain.json";
  write_chain_csv(csv, cut, cfg.chain.burn_in);
  write_chain_sidecar(side, cut, 12345);
  const auto cols = read_chain_csv(csv);
  bool ok = cols.size() == kParamCount + 1 && cut.loglik_trace.size() == cut.draws.size();
  for (std::size_t k = 0; ok && k < kParamCount; ++k) {
    ok = cols[k].size() == cut.draws.size();
    for (std::size_t i = 0; ok && i < cut.draws.size(); ++i) ok = cols[k][i] == cut.draws[i][k];
  }
  for (std::size_t i = 0; ok && i < cut.draws.size(); ++i) ok = cols[kParamCount][i] == cut.loglik_trace[i];
  report("HMC chain through write_chain_csv / read_chain_csv (io.hpp:129-170)", ok,
         std::to_string(cut.draws.size()) + " rows");
}

void posterior_agreement() {
  const Catalog catalog = simulated();
  ChainConfig mh = base_config(catalog);
  mh.iterations = 8000;
  mh.burn_in = 1000;
  const ChainOutput ref = run_fixed_posterior(mh, catalog);  // reference MH on the CPU
  b200::HmcConfig cfg;
  cfg.chain = base_config(catalog);
  cfg.chain.iterations = 2500;
  cfg.chain.burn_in = 500;
  cfg.leapfrog_steps = 10;
  cfg.step_size = 0.05;
  b200::HmcTiming timing;
  const ChainOutput hmc = b200::run_fixed_posterior_hmc(cfg, catalog, &timing);
  double worst = 0.0;
  std::string detail;
  for (std::size_t k = 0; k < kParamCount; ++k) {
    auto column = [&](const ChainOutput& c) {
      std::vector<double> v;
      for (const auto& d : c.draws) v.push_back(d[k]);
      return v;
    };
    auto mcse = [&](const std::vector<double>& v) {
      double mean = 0.0;
      for (double x : v) mean += x;
      mean /= static_cast<double>(v.size());
      double var = 0.0;
      for (double x : v) var += (x - mean) * (x - mean);
      var /= static_cast<double>(v.size() - 1);
      const double n_eff = std::max(1.0, ess(DrawMatrix{v}, EssKind::bulk).value);
      return std::pair{mean, std::sqrt(var / n_eff)};
    };
    const auto [m1, se1] = mcse(column(ref));
    const auto [m2, se2] = mcse(column(hmc));
    const double z = std::abs(m1 - m2) / std::max(1e-300, std::hypot(se1, se2));
    worst = std::max(worst, z);
    char b[96];
    std::snprintf(b, sizeof b, "%s %.4g vs %.4g; ", kParamNames[k], m1, m2);
    detail += b;
  }
  char b[160];
  std::snprintf(b, sizeof b, "N=%zu, worst |dmean| = %.2f MCSE (tol 4), HMC accept %.2f, eps %.3g, %zu GPU evals",
                catalog.size(), worst, hmc.acceptance_rate(0), hmc.final_steps[0], timing.evaluations);
  report("HMC (GPU gradient) and reference MH agree on the posterior", worst <= 4.0, detail + b);
}

// Square counties over the simulation window; each event tagged with its
// containing square (clamped to the grid) and that county's density.
PointSetup square_regions(const Catalog& catalog, int grid) {
  RegionTable regions;
  std::mt19937_64 drng(3);
  std::uniform_real_distribution<double> ulog(0.0, std::log(50.0));
  const double lo = -1.0, cell = 2.0 / grid;
  for (int gy = 0; gy < grid; ++gy)
    for (int gx = 0; gx < grid; ++gx) {
      const double x0 = lo + gx * cell, y0 = lo + gy * cell;
      Region r;
      r.id = "s" + std::to_string(gy * grid + gx);
      r.polygons.push_back(
          PolygonShape{{{x0, y0}, {x0 + cell, y0}, {x0 + cell, y0 + cell}, {x0, y0 + cell}}, {}});
      r.density = std::exp(ulog(drng));
      r.representative_latitude = y0 + 0.5 * cell;
      regions.add(std::move(r));
    }
  std::vector<Event> tagged = catalog.events();
  for (Event& e : tagged) {
    const int gx = std::clamp(static_cast<int>(std::floor((e.lon - lo) / cell)), 0, grid - 1);
    const int gy = std::clamp(static_cast<int>(std::floor((e.lat - lo) / cell)), 0, grid - 1);
    e.region_id = "s" + std::to_string(gy * grid + gx);
    e.density = regions.at(e.region_id).density;
  }
  return {Catalog(std::move(tagged)), std::move(regions)};
}

void loglik_trace_matches_locations() {
  const PointSetup setup = square_regions(simulated(), 4);
  b200::HmcConfig cfg;
  cfg.chain = base_config(setup.tagged);
  cfg.chain.initial.variant = Variant::varying;
  cfg.chain.iterations = 60;
  cfg.chain.burn_in = 10;
  cfg.chain.refresh_period = 1;
  cfg.leapfrog_steps = 4;
  cfg.step_size = 0.3;  // large: many rejections right after an X refresh
  cfg.adapt = false;
  const ChainOutput out = b200::run_cut_posterior_hmc(cfg, setup.tagged, setup.regions);
  // replay the location stream: the constructor's draw, then one per refresh
  std::mt19937_64 rng(cfg.chain.seed);
  resample_locations(setup.tagged, setup.regions, rng);
  b200::Engine check(setup.tagged);
  double worst = 0.0;
  std::size_t rejected = 0, compared = 0;
  bool ok = out.loglik_trace.size() == out.draws.size();
  for (std::size_t iter = 0; ok && iter < cfg.chain.iterations; ++iter) {
    if (iter % cfg.chain.refresh_period == 0) {
      auto [lon, lat] = resample_locations(setup.tagged, setup.regions, rng);
      check.set_locations(lon, lat);
    }
    if (iter < cfg.chain.burn_in) continue;
    const std::size_t i = iter - cfg.chain.burn_in;
    HawkesParams p = cfg.chain.initial;
    p.mu0 = out.draws[i][0];
    p.tau_t = out.draws[i][1];
    p.xi0 = out.draws[i][2];
    p.sigma_x = out.draws[i][3];
    p.sigma_t = out.draws[i][4];
    std::array<double, 5> g{};
    const double want = check.log_likelihood_and_gradient(p, p.variant, g);
    worst = std::max(worst, std::abs(out.loglik_trace[i] - want) / std::max(1.0, std::abs(want)));
    if (i > 0 && out.draws[i] == out.draws[i - 1]) ++rejected;
    ++compared;
  }
  ok = ok && worst <= 1e-12 && rejected > 0;
  report("cut-posterior HMC: loglik_trace[i] == LL(draw i, X of iteration i)", ok,
         std::to_string(compared) + " draws, " + std::to_string(rejected) +
             " rejected after a refresh, worst rel diff " + std::to_string(worst));
}

// HmcConfig::gpu_resample: X drawn on the GPU (Philox keyed by (seed,
// refresh index)) straight into the engine.  Replaying the same draws
// through b200::GpuRegions::sample must reproduce every loglik_trace entry,
// and every draw must lie in its event's square.
void gpu_resample_chain() {
  const PointSetup setup = square_regions(simulated(), 4);
  b200::HmcConfig cfg;
  cfg.chain = base_config(setup.tagged);
  cfg.chain.initial.variant = Variant::varying;
  cfg.chain.iterations = 40;
  cfg.chain.burn_in = 10;
  cfg.chain.refresh_period = 1;
  cfg.leapfrog_steps = 4;
  cfg.step_size = 0.3;
  cfg.adapt = false;
  cfg.gpu_resample = true;
  b200::HmcTiming timing;
  const ChainOutput out = b200::run_cut_posterior_hmc(cfg, setup.tagged, setup.regions, &timing);
  const b200::GpuRegions gpu(setup.tagged, setup.regions);
  b200::Engine check(setup.tagged);
  double worst = 0.0;
  bool inside = true;
  std::uint64_t refresh = 1;  // the constructor used refresh index 0
  bool ok = out.loglik_trace.size() == out.draws.size();
  for (std::size_t iter = 0; ok && iter < cfg.chain.iterations; ++iter) {
    if (iter % cfg.chain.refresh_period == 0) {
      auto [lon, lat] = gpu.sample(cfg.chain.seed, refresh++);
      for (std::size_t e = 0; e < lon.size(); ++e)
        inside = inside && setup.regions.at(setup.tagged[e].region_id).contains({lon[e], lat[e]});
      check.set_locations(lon, lat);
    }
    if (iter < cfg.chain.burn_in) continue;
    const std::size_t i = iter - cfg.chain.burn_in;
    HawkesParams p = cfg.chain.initial;
    p.mu0 = out.draws[i][0];
    p.tau_t = out.draws[i][1];
    p.xi0 = out.draws[i][2];
    p.sigma_x = out.draws[i][3];
    p.sigma_t = out.draws[i][4];
    std::array<double, 5> g{};
    const double want = check.log_likelihood_and_gradient(p, p.variant, g);
    worst = std::max(worst, std::abs(out.loglik_trace[i] - want) / std::max(1.0, std::abs(want)));
  }
  ok = ok && inside && worst <= 1e-12;
  char d[160];
  std::snprintf(d, sizeof d, "%zu draws, all X in their squares: %d, worst rel diff %.3g, resample %.3f ms/refresh",
                out.draws.size(), inside, worst, 1e3 * timing.resample_wait / cfg.chain.iterations);
  report("cut-posterior HMC with GPU resample: trace == LL(draw i, replayed GPU X)", ok, d);
}

}  // namespace

int main() {
  gpu_resample_chain();
  loglik_trace_matches_locations();
  point_regions_collapse();
  posterior_agreement();
  std::printf("%d failure(s)\n", failures);
  return failures;
}
