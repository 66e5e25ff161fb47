// BASELINE config 5: one cut-posterior HMC chain at N events on the B200
// engine: per iteration the reference's county-uniform location resample
// (resample_locations, mcmc.hpp:80-97; overlapped on a host thread), the
// location upload, and (leapfrog_steps + 1) density-scaled log-likelihood +
// gradient evaluations.  Fixture: a 60x60 grid of
// square counties over [-5, 5]^2 with densities log-uniform on [1, 7.4e4]
// drawn from mt19937_64(1); events = benchmark_catalog(N, 42) tagged by
// their containing square.
//
//   cut_posterior_bench [N=1000000] [iterations=4] [leapfrog=8] [gpus=1]
// Prints one JSON line.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "hawkes/engine.hpp"
#include "hawkes/geo.hpp"
#include "hawkes/mcmc.hpp"
#include "hawkes_b200/hmc.hpp"

using namespace hawkes;

int main(int argc, char** argv) {
  const std::size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1000000;
  const std::size_t iters = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 4;
  const int leapfrog = argc > 3 ? std::atoi(argv[3]) : 8;
  const int gpus = argc > 4 ? std::atoi(argv[4]) : 1;
  const bool gpu_resample = argc > 5 && std::atoi(argv[5]) != 0;  // HmcConfig::gpu_resample
  constexpr int kGrid = 60;
  const double cell = 10.0 / kGrid;
  RegionTable regions;
  std::mt19937_64 drng(1);
  std::uniform_real_distribution<double> ulog(0.0, std::log(7.4e4));
  for (int gy = 0; gy < kGrid; ++gy)
    for (int gx = 0; gx < kGrid; ++gx) {
      const double x0 = -5.0 + gx * cell, y0 = -5.0 + gy * cell;
      Region r;
      r.id = "c" + std::to_string(gy * kGrid + gx);
      r.polygons.push_back(PolygonShape{{{x0, y0}, {x0 + cell, y0}, {x0 + cell, y0 + cell}, {x0, y0 + cell}}, {}});
      r.density = std::exp(ulog(drng));
      r.representative_latitude = y0 + 0.5 * cell;
      regions.add(std::move(r));
    }
  std::vector<Event> events = benchmark_catalog(n, 42).events();
  for (Event& e : events) {
    const int gx = std::min(kGrid - 1, static_cast<int>((e.lon + 5.0) / cell));
    const int gy = std::min(kGrid - 1, static_cast<int>((e.lat + 5.0) / cell));
    e.region_id = "c" + std::to_string(gy * kGrid + gx);
    e.density = regions.at(e.region_id).density;
  }
  const Catalog catalog(std::move(events));

  // the reference's resample alone (what the overlap hides)
  std::mt19937_64 probe(7);
  const auto r0 = std::chrono::steady_clock::now();
  resample_locations(catalog, regions, probe);
  const double resample_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - r0).count();

  b200::HmcConfig cfg;
  cfg.chain.iterations = iters + 1;
  cfg.chain.burn_in = 1;  // the first iteration is the warm-up
  cfg.chain.seed = 5;
  cfg.chain.initial = HawkesParams{1.0, 5.0, 0.5, 0.5, 2.0, 100.0, Variant::varying};
  cfg.leapfrog_steps = leapfrog;
  cfg.step_size = 1e-4;
  cfg.adapt = false;
  cfg.n_gpus = gpus;
  cfg.gpu_resample = gpu_resample;
  b200::HmcSampler sampler(cfg, catalog, &regions);
  const ChainOutput out = sampler.run();
  const b200::HmcTiming& t = sampler.timing();
  const double per_iter = out.seconds / static_cast<double>(iters + 1);
  std::printf(
      "{\"config\": \"BASELINE config 5: cut-posterior HMC, county-uniform resample + density-scaled LL+grad\", "
      "\"n_events\": %zu, \"counties\": %d, \"gpus\": %d, \"gpu_resample\": %d, \"iterations\": %zu, "
      "\"leapfrog_steps\": %d, "
      "\"seconds_per_iteration\": %.4f, \"evaluations\": %zu, \"seconds_per_evaluation\": %.4f, "
      "\"resample_wait_s_per_iter\": %.4f, \"set_locations_s_per_iter\": %.4f, "
      "\"reference_resample_s\": %.4f, \"accept_rate\": %.3f, \"final_loglik\": %.10g}\n",
      n, kGrid * kGrid, gpus, gpu_resample ? 1 : 0, iters + 1, leapfrog, per_iter, t.evaluations, t.evaluate / t.evaluations,
      t.resample_wait / (iters + 1), t.set_locations / (iters + 1), resample_s, out.acceptance_rate(0),
      sampler.loglik());
  return 0;
}
