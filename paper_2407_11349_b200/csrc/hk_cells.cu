// Spatial cell tiles for the density-scaled trigger (csrc/hk_kernels.cu,
// PairParams::cells).
//
// The density-scaled trigger reaches only a few hundredths of the domain
// per source (with the certified cut), yet in time order every 256-column
// tile holds columns from everywhere, so every warp had to test every
// earlier column against its box.  Here the columns are regrouped by
// spatial cell (a gc x gc grid over the locations' box), time-sorted within
// each cell, and each cell's list padded to whole 256-column "cell tiles".
// A cell tile then has a small spatial box and a time range, and a CTA
// skips every tile whose box is beyond the reach of all its rows (one test
// per tile instead of eight per warp) or whose times are all at or after its
// rows'.  Tiles entirely earlier than the CTA's rows keep the factorised
// temporal weight (t_ref = the tile's last time); the others evaluate the
// guard t_j < t_i per pair.
//
// The order is a deterministic stable counting sort by cell (one warp per
// 1024-column chunk ranks its columns with match_any in index order), so each
// cell's columns keep their time order.  Recomputed once per location set.
#include <cuda_runtime.h>

#include "hk_device.cuh"
#include "hk_kernels.cuh"

namespace hk {

namespace {

constexpr int kRankChunk = 1024;

__device__ __forceinline__ int cell_of(double x, double y, double q, const CellGrid& g) {
  const int cx = min(max(static_cast<int>(floor((x - g.x0) * g.inv_side)), 0), g.gc - 1);
  const int cy = min(max(static_cast<int>(floor((y - g.y0) * g.inv_side)), 0), g.gc - 1);
  const int cl = g.ncls > 1 ? min(max(static_cast<int>(floor((log(q) - g.lq0) * g.inv_lq)), 0), g.ncls - 1) : 0;
  return (cx + g.gc * cy) * g.ncls + cl;
}

// per chunk of kRankChunk columns: the count of each cell
__global__ void cells_count_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                   const double* __restrict__ q, int n, CellGrid g, int* cell, int* chunk_counts) {
  extern __shared__ int s_cnt[];
  const int ncell = g.gc * g.gc * g.ncls;
  for (int c = threadIdx.x; c < ncell; c += blockDim.x) s_cnt[c] = 0;
  __syncthreads();
  const int j0 = blockIdx.x * kRankChunk;
  for (int j = j0 + threadIdx.x; j < min(n, j0 + kRankChunk); j += blockDim.x) {
    const int c = cell_of(x[j], y[j], q[j], g);
    cell[j] = c;
    atomicAdd(&s_cnt[c], 1);  // integer counts: order-independent
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ncell; c += blockDim.x)
    chunk_counts[static_cast<size_t>(blockIdx.x) * ncell + c] = s_cnt[c];
}

// per cell (one warp each, a CTA of kScanWarps warps per kScanWarps cells):
// exclusive prefix over the chunks (in place) and the cell's count, 32
// chunks per step; then cells_start_kernel turns the counts into the cells'
// first cell-tile positions.
constexpr int kScanWarps = 4;
__global__ void __launch_bounds__(32 * kScanWarps) cells_scan_kernel(int n_chunks, int ncell, int* chunk_counts,
                                                                     int* cell_count) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * kScanWarps + (threadIdx.x >> 5);
  if (c >= ncell) return;
  int carry = 0;
  for (int k0 = 0; k0 < n_chunks; k0 += 32) {
    const int k = k0 + lane;
    int* slot = chunk_counts + static_cast<size_t>(k) * ncell + c;
    const int v = k < n_chunks ? *slot : 0;
    int inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, off);
      if (lane >= off) inc += t;
    }
    if (k < n_chunks) *slot = carry + inc - v;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) cell_count[c] = carry;
}

__global__ void cells_start_kernel(int ncell, int* cell_start, int* n_ctiles) {
  if (threadIdx.x != 0) return;
  int pos = 0;
  for (int c = 0; c < ncell; ++c) {
    const int cnt = cell_start[c];  // the count, in place
    cell_start[c] = pos;
    pos += (cnt + kBJ - 1) / kBJ * kBJ;  // whole cell tiles
  }
  cell_start[ncell] = pos;
  *n_ctiles = pos / kBJ;
}

// one warp per chunk: stable ranks within the chunk, in index order
__global__ void cells_rank_kernel(int n, int ncell, const int* __restrict__ cell,
                                  const int* __restrict__ chunk_base, const int* __restrict__ cell_start,
                                  int* perm) {
  extern __shared__ int s_run[];
  const int lane = threadIdx.x;
  for (int c = lane; c < ncell; c += 32) s_run[c] = chunk_base[static_cast<size_t>(blockIdx.x) * ncell + c];
  __syncwarp();
  const int j0 = blockIdx.x * kRankChunk;
  for (int s = j0; s < min(n, j0 + kRankChunk); s += 32) {
    const int j = s + lane;
    const bool ok = j < n;
    const int c = ok ? cell[j] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, c);
    const int before = __popc(peers & ((1u << lane) - 1u));
    if (ok) perm[cell_start[c] + s_run[c] + before] = j;
    __syncwarp();
    if (ok && before == 0) s_run[c] += __popc(peers);  // the group's first lane advances the cell
    __syncwarp();
  }
}

}  // namespace

void launch_cells(const double* x, const double* y, const double* q, int n, const CellGrid& g, int* cell, int* chunk_counts,
                  int* cell_start, int* perm, int perm_len, int* n_ctiles, cudaStream_t s) {
  const int ncell = g.gc * g.gc * g.ncls;
  const int n_chunks = (n + kRankChunk - 1) / kRankChunk;
  cudaMemsetAsync(perm, 0xff, static_cast<size_t>(perm_len) * sizeof(int), s);  // -1: padding
  cells_count_kernel<<<n_chunks, 256, ncell * sizeof(int), s>>>(x, y, q, n, g, cell, chunk_counts);
  cells_scan_kernel<<<(ncell + kScanWarps - 1) / kScanWarps, 32 * kScanWarps, 0, s>>>(n_chunks, ncell, chunk_counts,
                                                                                      cell_start);
  cells_start_kernel<<<1, 32, 0, s>>>(ncell, cell_start, n_ctiles);
  cells_rank_kernel<<<n_chunks, 32, ncell * sizeof(int), s>>>(n, ncell, cell, chunk_counts, cell_start, perm);
}

}  // namespace hk
