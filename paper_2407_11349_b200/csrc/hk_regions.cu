// GPU county-uniform location sampler: the cut posterior's X refresh
// (resample_locations, mcmc.hpp:80-97 -> sample_point_in_region,
// geo.hpp:138-161) as one thread per event.
//
// Same algorithm as the reference, per event: a point region returns its
// point; otherwise a polygon part is picked with probability proportional to
// its area (polygon_area: outer shoelace area minus the holes'), then points
// are drawn uniformly in the part's outer bounding box until one passes the
// even-odd point-in-polygon test (outer ring, not in any hole), at most
// `attempt_budget` = 10000 attempts.  A zero-area region or an exhausted
// budget fails the call with the reference's message and the event index.
//
// The random stream is different by design: Philox4x32-10 keyed by the seed,
// counter = (event index, call counter, draw index), so every event's draw is
// independent of every other's and of the thread schedule (bitwise
// reproducible for a fixed (seed, counter)).  The reference's mt19937_64
// stream stays the default everywhere (hmc.hpp: HmcConfig::gpu_resample
// opts in); parity is distributional (tests/test_gpu_regions.py mirrors
// test_geo.cpp:47-120).
//
// Events are processed in region order (a permutation computed once at
// upload), so the threads of a warp mostly share a region: its vertices are
// broadcast loads and the rejection loops stay convergent.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "hk_device.cuh"
#include "hk_regions.hpp"

namespace hk {

namespace {

constexpr int kSampleThreads = 256;

struct Philox {
  // Philox4x32-10 (Salmon et al., SC'11): counter c, key k.
  __device__ static uint4 round(uint4 c, uint2 k) {
    const unsigned long long p0 = 0xD2511F53ull * c.x, p1 = 0xCD9E8D57ull * c.z;
    return make_uint4(static_cast<unsigned>(p1 >> 32) ^ c.y ^ k.x, static_cast<unsigned>(p1),
                      static_cast<unsigned>(p0 >> 32) ^ c.w ^ k.y, static_cast<unsigned>(p0));
  }
  __device__ static uint4 gen(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      c = round(c, k);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
};

// Two doubles uniform on [0, 1) (53 random bits each) per Philox block.
struct Uniforms {
  uint2 key;
  unsigned event, ctr_lo, ctr_hi, draw = 0;
  double u0 = 0.0, u1 = 0.0;
  int left = 0;
  __device__ double next() {
    if (left == 0) {
      const uint4 r = Philox::gen(make_uint4(event, ctr_lo, ctr_hi, draw++), key);
      const unsigned long long a = (static_cast<unsigned long long>(r.x) << 32 | r.y) >> 11;
      const unsigned long long b = (static_cast<unsigned long long>(r.z) << 32 | r.w) >> 11;
      u0 = static_cast<double>(a) * 0x1.0p-53;
      u1 = static_cast<double>(b) * 0x1.0p-53;
      left = 2;
    }
    return left-- == 2 ? u0 : u1;
  }
};

// point_in_ring (geo.hpp:47-58), the same IEEE operations in the same
// order (no contraction), so a point's classification matches the host's.
__device__ bool in_ring(double px, double py, const double2* __restrict__ v, int nv) {
  bool inside = false;
  for (int i = 0, j = nv - 1; i < nv; j = i++) {
    const double2 a = v[i], b = v[j];
    if ((a.y > py) != (b.y > py)) {
      const double xc = __dadd_rn(__ddiv_rn(__dmul_rn(__dsub_rn(b.x, a.x), __dsub_rn(py, a.y)),
                                            __dsub_rn(b.y, a.y)),
                                  a.x);
      if (px < xc) inside = !inside;
    }
  }
  return inside;
}

__global__ void __launch_bounds__(kSampleThreads)
    sample_kernel(const RegionsDevice R, unsigned long long seed, unsigned long long counter,
                  double* __restrict__ x, double* __restrict__ y, unsigned long long* fail) {
  const int k = blockIdx.x * kSampleThreads + threadIdx.x;
  if (k >= R.n_events) return;
  const int e = R.perm[k];
  HK_ASSERT(e >= 0 && e < R.n_events);
  const int r = R.event_region[e];
  const int kind = R.kind[r];
  if (kind == kRegionPoint) {
    x[e] = R.point[2 * r];
    y[e] = R.point[2 * r + 1];
    return;
  }
  if (kind == kRegionZeroArea) {
    atomicMin(fail, static_cast<unsigned long long>(e) << 2 | kFailZeroArea);
    return;
  }
  Uniforms u;
  u.key = make_uint2(static_cast<unsigned>(seed), static_cast<unsigned>(seed >> 32));
  u.event = static_cast<unsigned>(e);
  u.ctr_lo = static_cast<unsigned>(counter);
  u.ctr_hi = static_cast<unsigned>(counter >> 32);
  // area-weighted part (geo.hpp:148-151)
  const int p0 = R.region_parts[r], p1 = R.region_parts[r + 1];
  double pick = u.next() * R.region_area[r];
  int part = p0;
  while (part + 1 < p1 && pick >= R.part_area[part]) pick -= R.part_area[part++];
  const double bx0 = R.part_box[4 * part], by0 = R.part_box[4 * part + 1];
  const double bx1 = R.part_box[4 * part + 2], by1 = R.part_box[4 * part + 3];
  const int rg0 = R.part_rings[part], rg1 = R.part_rings[part + 1];
  for (int attempt = 0; attempt < R.attempt_budget; ++attempt) {
    const double px = bx0 + u.next() * (bx1 - bx0);
    const double py = by0 + u.next() * (by1 - by0);
    // point_in_polygon (geo.hpp:60-65): in the outer ring and in no hole
    bool ok = in_ring(px, py, R.verts + R.ring_verts[rg0], R.ring_verts[rg0 + 1] - R.ring_verts[rg0]);
    for (int h = rg0 + 1; ok && h < rg1; ++h)
      ok = !in_ring(px, py, R.verts + R.ring_verts[h], R.ring_verts[h + 1] - R.ring_verts[h]);
    if (ok) {
      x[e] = px;
      y[e] = py;
      return;
    }
  }
  atomicMin(fail, static_cast<unsigned long long>(e) << 2 | kFailBudget);
}

template <typename T>
T* upload(const std::vector<T>& v, cudaStream_t s) {
  void* p = nullptr;
  if (cudaMalloc(&p, std::max<std::size_t>(v.size(), 1) * sizeof(T)) != cudaSuccess)
    throw std::runtime_error("hk_regions: cudaMalloc failed");
  if (!v.empty() &&
      cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s) != cudaSuccess)
    throw std::runtime_error("hk_regions: upload failed");
  return static_cast<T*>(p);
}

// ring_signed_area / ring_area (geo.hpp:34-45)
double ring_area(const double* v, std::size_t nv) {
  double a = 0.0;
  for (std::size_t i = 0; i < nv; ++i) {
    const std::size_t j = (i + 1) % nv;
    a += v[2 * i] * v[2 * j + 1] - v[2 * j] * v[2 * i + 1];
  }
  return std::abs(0.5 * a);
}

}  // namespace

RegionsHost build_regions(std::size_t n_regions, const int* is_point, const double* point_xy,
                          const std::size_t* region_parts, const std::size_t* part_rings,
                          const std::size_t* ring_verts, const double* verts, std::size_t n_events,
                          const int* event_region) {
  RegionsHost h;
  const std::size_t n_parts = region_parts[n_regions];
  const std::size_t n_rings = n_parts ? part_rings[n_parts] : 0;
  h.kind.resize(n_regions);
  h.point.assign(point_xy, point_xy + 2 * n_regions);
  h.region_parts.resize(n_regions + 1);
  h.region_area.resize(n_regions);
  h.part_area.resize(n_parts);
  h.part_box.resize(4 * n_parts);
  h.part_rings.resize(n_parts + 1);
  h.ring_verts.resize(n_rings + 1);
  for (std::size_t r = 0; r <= n_regions; ++r) h.region_parts[r] = static_cast<int>(region_parts[r]);
  for (std::size_t p = 0; p <= n_parts; ++p) h.part_rings[p] = static_cast<int>(part_rings[p]);
  for (std::size_t g = 0; g <= n_rings; ++g) h.ring_verts[g] = static_cast<int>(ring_verts[g]);
  const std::size_t n_verts = n_rings ? ring_verts[n_rings] : 0;
  if (n_verts >= (std::size_t{1} << 31)) throw std::invalid_argument("hk_regions: too many vertices");
  h.verts.resize(n_verts);
  for (std::size_t v = 0; v < n_verts; ++v) h.verts[v] = make_double2(verts[2 * v], verts[2 * v + 1]);
  for (std::size_t p = 0; p < n_parts; ++p) {
    const std::size_t g0 = part_rings[p], g1 = part_rings[p + 1];
    if (g1 <= g0) throw std::invalid_argument("hk_regions: polygon part without an outer ring");
    double a = 0.0;
    for (std::size_t g = g0; g < g1; ++g) {
      const std::size_t nv = ring_verts[g + 1] - ring_verts[g];
      if (nv == 0) throw std::invalid_argument("hk_regions: empty ring");
      const double ra = ring_area(verts + 2 * ring_verts[g], nv);
      a = g == g0 ? ra : a - ra;  // polygon_area, geo.hpp:67-71
    }
    h.part_area[p] = a;
    const double* v0 = verts + 2 * ring_verts[g0];  // ring_bbox of the outer ring, geo.hpp:73-82
    double box[4] = {v0[0], v0[1], v0[0], v0[1]};
    for (std::size_t v = ring_verts[g0]; v < ring_verts[g0 + 1]; ++v) {
      box[0] = std::min(box[0], verts[2 * v]);
      box[1] = std::min(box[1], verts[2 * v + 1]);
      box[2] = std::max(box[2], verts[2 * v]);
      box[3] = std::max(box[3], verts[2 * v + 1]);
    }
    std::copy(box, box + 4, &h.part_box[4 * p]);
  }
  for (std::size_t r = 0; r < n_regions; ++r) {
    double total = 0.0;
    for (std::size_t p = region_parts[r]; p < region_parts[r + 1]; ++p) total += h.part_area[p];
    h.region_area[r] = total;
    h.kind[r] = is_point[r] ? kRegionPoint : (total > 0.0 ? kRegionPolygons : kRegionZeroArea);
  }
  h.event_region.assign(event_region, event_region + n_events);
  for (std::size_t e = 0; e < n_events; ++e)
    if (event_region[e] < 0 || static_cast<std::size_t>(event_region[e]) >= n_regions)
      throw std::invalid_argument("resample_locations: event " + std::to_string(e) +
                                  " has unresolvable region id");
  h.perm.resize(n_events);
  std::iota(h.perm.begin(), h.perm.end(), 0);
  std::stable_sort(h.perm.begin(), h.perm.end(),
                   [&](int a, int b) { return event_region[a] < event_region[b]; });
  return h;
}

RegionsDevice upload_regions(const RegionsHost& h, cudaStream_t s) {
  RegionsDevice d{};
  d.n_events = static_cast<int>(h.event_region.size());
  d.attempt_budget = 10000;  // sample_point_in_region's default, geo.hpp:139
  d.kind = upload(h.kind, s);
  d.point = upload(h.point, s);
  d.region_parts = upload(h.region_parts, s);
  d.region_area = upload(h.region_area, s);
  d.part_area = upload(h.part_area, s);
  d.part_box = upload(h.part_box, s);
  d.part_rings = upload(h.part_rings, s);
  d.ring_verts = upload(h.ring_verts, s);
  d.verts = upload(h.verts, s);
  d.event_region = upload(h.event_region, s);
  d.perm = upload(h.perm, s);
  if (cudaMalloc(&d.fail, sizeof(unsigned long long)) != cudaSuccess)
    throw std::runtime_error("hk_regions: cudaMalloc failed");
  return d;
}

void free_regions(RegionsDevice& d) {
  for (const void* p : {static_cast<const void*>(d.kind), static_cast<const void*>(d.point),
                        static_cast<const void*>(d.region_parts), static_cast<const void*>(d.region_area),
                        static_cast<const void*>(d.part_area), static_cast<const void*>(d.part_box),
                        static_cast<const void*>(d.part_rings), static_cast<const void*>(d.ring_verts),
                        static_cast<const void*>(d.verts), static_cast<const void*>(d.event_region),
                        static_cast<const void*>(d.perm), static_cast<const void*>(d.fail)})
    if (p) cudaFree(const_cast<void*>(p));
  d = RegionsDevice{};
}

void launch_sample(const RegionsDevice& d, unsigned long long seed, unsigned long long counter,
                   double* x, double* y, cudaStream_t s) {
  cudaMemsetAsync(d.fail, 0xff, sizeof(unsigned long long), s);
  if (d.n_events == 0) return;
  sample_kernel<<<(d.n_events + kSampleThreads - 1) / kSampleThreads, kSampleThreads, 0, s>>>(
      d, seed, counter, x, y, d.fail);
}

}  // namespace hk
