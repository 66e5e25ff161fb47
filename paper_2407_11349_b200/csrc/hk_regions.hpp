// Region tables for the GPU location sampler (hk_regions.cu).  Plain
// structs: the host build (validation, areas, boxes, region-order
// permutation) and the device view the sampling kernel reads.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <vector>

namespace hk {

enum RegionKind { kRegionPolygons = 0, kRegionPoint = 1, kRegionZeroArea = 2 };
// failure word: (event << 2) | code; all ones = no failure
enum FailCode { kFailZeroArea = 1, kFailBudget = 2 };

struct RegionsHost {
  std::vector<int> kind;            // [R]
  std::vector<double> point;        // [2R]
  std::vector<int> region_parts;    // [R+1] part offsets
  std::vector<double> region_area;  // [R] sum of part areas
  std::vector<double> part_area;    // [P] polygon_area
  std::vector<double> part_box;     // [4P] outer-ring bbox (xmin, ymin, xmax, ymax)
  std::vector<int> part_rings;      // [P+1] ring offsets (first ring of a part: outer)
  std::vector<int> ring_verts;      // [Rings+1] vertex offsets
  std::vector<double2> verts;       // [V]
  std::vector<int> event_region;    // [N]
  std::vector<int> perm;            // [N] events in region order
};

struct RegionsDevice {
  int n_events = 0, attempt_budget = 0;
  const int* kind = nullptr;
  const double* point = nullptr;
  const int* region_parts = nullptr;
  const double* region_area = nullptr;
  const double* part_area = nullptr;
  const double* part_box = nullptr;
  const int* part_rings = nullptr;
  const int* ring_verts = nullptr;
  const double2* verts = nullptr;
  const int* event_region = nullptr;
  const int* perm = nullptr;
  unsigned long long* fail = nullptr;
};

RegionsHost build_regions(std::size_t n_regions, const int* is_point, const double* point_xy,
                          const std::size_t* region_parts, const std::size_t* part_rings,
                          const std::size_t* ring_verts, const double* verts, std::size_t n_events,
                          const int* event_region);
RegionsDevice upload_regions(const RegionsHost& h, cudaStream_t s);
void free_regions(RegionsDevice& d);
// Samples every event's location into x[e], y[e] (device arrays) and resets
// then sets d.fail to the smallest failing (event << 2 | code).
void launch_sample(const RegionsDevice& d, unsigned long long seed, unsigned long long counter,
                   double* x, double* y, cudaStream_t s);

}  // namespace hk
