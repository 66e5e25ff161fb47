// hawkes_b200/regions.hpp — the cut posterior's location refresh on the GPU
// (hk_regions_*, include/hawkes_b200.h), over the reference's own Catalog
// and RegionTable types.
//
//   hawkes::resample_locations(catalog, regions, rng)     mcmc.hpp:80-97
//     -> b200::resample_locations(catalog, regions, rng)  same signature; one
//        64-bit draw from `rng` keys the GPU's Philox stream, so successive
//        calls give fresh, reproducible draws
//   hawkes::sample_point_in_region                        geo.hpp:138-161
//     -> one GPU thread per event, same algorithm (area-weighted part,
//        bounding-box rejection, even-odd test, 10000 attempts), same errors
//
// The draws are NOT the reference's mt19937_64 stream (they match it in
// distribution: tests/test_gpu_regions.py); callers that need the
// reference's exact location sequence keep hawkes::resample_locations, which
// stays the default of the HMC driver (HmcConfig::gpu_resample).
#ifndef HAWKES_B200_REGIONS_HPP
#define HAWKES_B200_REGIONS_HPP

#include <cstdint>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "hawkes/geo.hpp"
#include "hawkes/types.hpp"
#include "hawkes_b200/engine.hpp"

namespace hawkes::b200 {

/// A RegionTable and the catalog's event -> region map, resident on `device`.
class GpuRegions {
 public:
  GpuRegions(const Catalog& catalog, const RegionTable& regions, int device = 0)
      : h_(nullptr, &hk_regions_destroy), n_(catalog.size()) {
    const std::vector<Region>& rs = regions.regions();
    std::vector<int> is_point;
    std::vector<double> point_xy, verts;
    std::vector<std::size_t> region_parts{0}, part_rings{0}, ring_verts{0};
    std::vector<const char*> ids;
    std::unordered_map<std::string, int> index;
    for (std::size_t r = 0; r < rs.size(); ++r) {
      const Region& g = rs[r];
      index.emplace(g.id, static_cast<int>(r));
      ids.push_back(g.id.c_str());
      is_point.push_back(g.is_point ? 1 : 0);
      point_xy.push_back(g.point[0]);
      point_xy.push_back(g.point[1]);
      if (!g.is_point)
        for (const PolygonShape& poly : g.polygons) {
          auto ring = [&](const Ring& v) {
            for (const Point& p : v) {
              verts.push_back(p[0]);
              verts.push_back(p[1]);
            }
            ring_verts.push_back(ring_verts.back() + v.size());
          };
          ring(poly.outer);
          for (const Ring& h : poly.holes) ring(h);
          part_rings.push_back(part_rings.back() + 1 + poly.holes.size());
        }
      region_parts.push_back(part_rings.size() - 1);
    }
    std::vector<int> event_region(n_);
    for (std::size_t i = 0; i < n_; ++i) {  // mcmc.hpp:84-88
      auto it = index.find(catalog[i].region_id);
      if (it == index.end())
        throw std::runtime_error("resample_locations: event " + std::to_string(i) +
                                 " has unresolvable region id '" + catalog[i].region_id + "'");
      event_region[i] = it->second;
    }
    hk_regions* raw = nullptr;
    detail::check(hk_regions_create(rs.size(), is_point.data(), point_xy.data(), region_parts.data(),
                                    part_rings.data(), ring_verts.data(), verts.data(), ids.data(), n_,
                                    event_region.data(), device, &raw));
    h_.reset(raw);
  }

  hk_regions* get() const { return h_.get(); }

  /// One draw per event (host arrays), Philox-keyed by (seed, counter).
  std::pair<std::vector<double>, std::vector<double>> sample(std::uint64_t seed,
                                                             std::uint64_t counter) const {
    std::vector<double> lon(n_), lat(n_);
    detail::check(hk_regions_sample(h_.get(), seed, counter, lon.data(), lat.data()));
    return {std::move(lon), std::move(lat)};
  }

 private:
  std::unique_ptr<hk_regions, void (*)(hk_regions*)> h_;
  std::size_t n_;
};

/// mcmc.hpp:80-97's signature on the GPU: one 64-bit draw from `rng` keys
/// the Philox stream of this call.  Builds the region table per call; a
/// chain should keep a GpuRegions and use Engine::resample_locations.
inline std::pair<std::vector<double>, std::vector<double>> resample_locations(
    const Catalog& catalog, const RegionTable& regions, std::mt19937_64& rng) {
  const std::uint64_t seed = rng();
  return GpuRegions(catalog, regions).sample(seed, 0);
}

}  // namespace hawkes::b200

#endif  // HAWKES_B200_REGIONS_HPP
