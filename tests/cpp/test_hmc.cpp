// HMC cut-posterior gate (include/hawkes_b200/hmc.hpp), against the
// reference's own MH sampler and diagnostics (mcmc.hpp, diagnostics.hpp):
//   1. degenerate point regions: the cut-posterior HMC chain equals the
//      fixed-location chain exactly (test_mcmc.cpp:212-231 analogue);
//   2. posterior agreement: HMC on the GPU and the reference's univariate MH
//      (CPU) give posterior means within 4 Monte Carlo standard errors on a
//      simulated catalog (acceptance.cpp:244-296 convention);
//   3. the HMC chain persists through the reference's chain CSV and sidecar
//      writers (io.hpp:129-156) and reads back exactly (read_chain_csv).
// PASS/FAIL lines; exit status = number of failures.
#include <cmath>
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

}  // namespace

int main() {
  point_regions_collapse();
  posterior_agreement();
  std::printf("%d failure(s)\n", failures);
  return failures;
}
