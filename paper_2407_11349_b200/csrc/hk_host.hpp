// Host-side logic behind the C ABI: validation with the reference's
// messages, the reference's synthetic catalog, partitions and shard plans,
// and the work-item planner for the pair kernel.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "hk_kernels.cuh"

namespace hk {

struct ParamsIn {
  double mu0, tau_t, xi0, sigma_x, sigma_t, area;
  int variant;
};

// Catalog invariants, types.hpp:43-57 (same checks, same messages);
// coarse_only skips the location check (Catalog(events, coarse_only)).
void validate_catalog(const double* t, const double* x, const double* y, const double* d,
                      std::size_t n, bool coarse_only = false);
// HawkesParams::validate, types.hpp:92-103.
void validate_params(const ParamsIn& p);

// benchmark_catalog(n, seed), engine.hpp:251-259.
void benchmark_catalog(std::size_t n, std::uint64_t seed, double* t, double* x, double* y,
                       double* d);

// Partition::make, engine.hpp:27-40, as g+1 boundaries.
std::vector<std::size_t> partition_make(std::size_t n, std::size_t g);

// count_before / upper_bound for every row of a sorted time array.
void tie_bounds(const std::vector<double>& t, std::vector<int>& lb, std::vector<int>& ub);

// Cost-balanced contiguous shards: row i costs alpha*(n-1) + kCostBeta*lb[i]
// FP64 instructions (ncu-measured per-pair costs of the pair kernel).  The
// background costs 13 per pair on the direct path but ~0.2 once the block
// expansion qualifies, which it does for catalogs dense in time (large N);
// alpha = background_cost(n) picks between the two.
constexpr double kCostAlphaDirect = 13.0;    // FP64 per background pair, direct
constexpr double kCostAlphaExpanded = 1.0;   // ... with the block expansion (rounded up)
constexpr double kCostBeta = 16.0;           // FP64 per trigger pair (direct background)
// With the background expanded, the measured per-row cost of the homogeneous
// kernel is a + b t_n/T with b/a = 46 (fit of sixteen 1/16 row ranges at
// N=1e6: 3.32 + 3.93 k ms): the trigger weighs 46 against 1 per background
// column.
constexpr double kCostBetaExpanded = 46.0;
constexpr std::size_t kExpansionRows = 32768;  // catalogs at least this large expand
// From this size the homogeneous trigger before each checkpoint and the
// background go through the Hermite expansions (hk_fgt.cu, on by default):
// every row then costs about the same (the expansion's row evaluation is
// independent of t_i and the direct remainder is bounded by a checkpoint's
// width), so homogeneous shards are planned with beta = 0 (equal rows).
constexpr std::size_t kFgtPlanRows = 131072;
constexpr double kCostBetaFgt = 0.0;
inline double background_cost(std::size_t n) {
  return n >= kExpansionRows ? kCostAlphaExpanded : kCostAlphaDirect;
}
// The density-scaled kernel culls its trigger spatially (cell tiles, the
// certified cut), so a row's cost is nearly proportional to its earlier
// sources: fit of the shard times at N=1e6 (g = 2, 4, 8) to f + b sum(lb):
// b = 18.1 ms per 1e12, the per-row part indistinguishable from 0; with
// beta = 20 the fitted model's max/mean is 1.02-1.03 (4.3 before the cells:
// measured 1.38 at g = 8).
constexpr double kCostBetaVarying = 20.0;
std::vector<std::size_t> plan_shards(const std::vector<int>& lb, std::size_t g,
                                     double beta = kCostBeta);

// Work items for rows [rb, re) of an n-event catalog: row blocks of
// rows_per_item rows times column chunks of whole tiles; heaviest first.  Returns the
// number of chunk slots per row.  window > 1: the rows are taken in windows
// of window * rows_per_item rows, classified against the whole window and
// read through the clustered order rperm[(window start - rb) + ...]
// (Item::pos; launch_cluster with the same window).
// cell_tiles > 0: the column space is that many spatial cell tiles
// (hk_cells.cu) instead of the time-ordered tiles.
int plan_items(const std::vector<int>& lb, const std::vector<int>& ub, int n, int rb, int re,
               int rows_per_item, std::vector<Item>& items, int window = 1, int cell_tiles = 0);

// The homogeneous plan when the pair kernel computes only the trigger and the
// Hermite expansion supplies every tile below each block's checkpoint: one
// item per row block (more only if a block's remaining band exceeds
// kMaxItemTiles tiles) over the tiles [checkpoint, last tile of the block's
// ties).  Returns the slots (chunks per block).
int plan_items_fgt(const std::vector<int>& lb, const std::vector<int>& ub, int n, int rb, int re,
                   int kBI, std::vector<Item>& items);

// Per-evaluation coefficients (types.hpp:105-109, model.hpp:202-210) and
// the host-side argument bound that selects the checked exp.
EvalCoef make_coef(const ParamsIn& p, double t_min, double t_max, double d2_max, double q_max);

}  // namespace hk
