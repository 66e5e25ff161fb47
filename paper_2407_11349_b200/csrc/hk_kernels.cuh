// Launch-side view of the device kernels (shared by hk_kernels.cu and the
// context code in hk_capi.cu).  Plain structs only.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace hk {

// One work item = one CTA: up to kBI rows against column tiles [tb, te);
// its five per-row partial sums land in partial slot `slot`.  [rb, re) is
// the row block the column tiles are classified against.  pos < 0: the rows
// are rb, rb+1, ... (< re).  pos >= 0: the rows are rperm[pos .. pos+kBI)
// (-1 = none), a spatially clustered order of a row window (cluster_kernel)
// in which each warp's 32*NR consecutive positions form one cluster.
struct Item {
  int rb, re, tb, te, slot, pos;
  int xt;  // homogeneous plan: the trigger of tiles below xt comes from the Hermite expansion
           // (hk_fgt.cu) when the launch says so (PairParams::fgt); 0 otherwise
};
constexpr int kMaxItemTiles = 2048;  // te - tb (the pair kernel classifies them in shared memory)
// Work items per launch the planner aims for (~72 waves of 148 SMs x 3
// CTAs): measured at N=1e6 (tools/item_sweep.sh, profiles/r02_item_sweep.txt)
// the pair kernel keeps speeding up with more, smaller items up to here
// (3552 items: 543.5 ms, 7104: 522.9, 14208: 510.1, 31264: 503.9).
constexpr int kItemTarget = 148 * 3 * 72;
// The density-scaled (clustered, trigger-only) plan: half as many items are
// as fast there (N=1e6: 16000 items 17.48 ms = 31968 items; county catalog
// +0.5%) and halve its partial-sum traffic.  Over cell tiles (trigger ms,
// bench / county catalog): 6000 items 8.07 / 53.1, 12000 8.14 / 51.5,
// 16000 8.22 / 51.5.
constexpr int kItemTargetVarying = 12000;
// Column chunks per row block at most: the partial-sum buffer holds
// slots x 40 B per row.
constexpr int kMaxSlots = 64;

// Per-evaluation coefficients, all derived on the host in double exactly
// once (HawkesParams accessors, types.hpp:105-109; coefficients,
// model.hpp:202-210).
struct EvalCoef {
  double mu0, tau_t, xi0, sigma_x, sigma_t;
  double tau_prec, sx_prec, omega;
  double a;       // background_coefficient<double>
  double c;       // trigger_coefficient<double>
  double half_s2; // 0.5 * sx_prec * sx_prec (model.hpp:151)
  double Kb;      // -0.5 tau_prec^2 * 16/ln2   (background exponent per td^2)
  double Kq0;     // -half_s2 * 16/ln2           (trigger exponent per d^2, q = 1)
  double Kw;      // -omega * 16/ln2             (trigger exponent per td)
  double t_end;   // t[N-1]
  double u_scale; // 1 / (tau sqrt 2): background kernel = exp(-(u_i - u_j)^2)
  double two_tau2;// 2 tau^2
  int bg_expansion;  // 1: background by the exact block expansion where it qualifies
  double cx, cy;  // centre of the locations' bounding box (FP32 skip test frame)
  double f32_err; // bound on |FP32 distance - exact distance| in that frame
  int single_prec;   // Precision::single: FP32 trigger arithmetic, LL only
  int varying;
  int mode;       // ExpMode: kExact / kFlush / kChecked from the argument bound
  double tr_cut;  // density-scaled trigger: spatial exponent (ln2/kTab units) beyond which
                  // the candidate test drops a column (certified, hk_cert.cu); 0 = the flush
                  // threshold (only exact zeros dropped)
};

struct DeviceCatalog {
  int n, npad;
  const double* t;   // [npad], padded with t[n-1]
  const double* x;   // [npad], padded with 0
  const double* y;   // [npad]
  const double* q;   // density, [npad], padded with 1
  const int* lb;     // [n] count_before(t_i) (model.hpp:115-117)
  const int* ub;     // [n] upper_bound(t_i)
  double* K;         // prep: per-source trigger exponent coefficient  [npad]
  double* thr;       // prep: d^2 beyond which the spatial factor flushes [npad]
  double* w;         // prep: q_j exp(-omega (t_ref(J) - t_j))        [npad]
  double* v;         // prep: (t_ref(J) - t_j) w_j                    [npad]
  double* z;         // prep: q_j w_j                                 [npad]
  float4* fxy;       // prep: {x_j - cx, y_j - cy, thrf_j, 0} in FP32     [npad]
  float2* fkw;       // prep: {K_j log2(e)/(ln2-units), w_j} in FP32 (single precision) [npad]
  const int* rperm;  // clustered row order per row window (Item::pos), or null
  double2* xy;       // prep: {x_j, y_j}  \ interleaved copies for the trigger-only
  double2* wk;       // prep: {w_j, K_j}   > launches' compact stage layout: one
  double2* vz;       // prep: {v_j, z_j}  / 16-byte broadcast load per pair    [npad]
};

// Spatial cell tiles of the density-scaled trigger (hk_cells.cu): the grid
// and, per location set, the columns regrouped by cell (time order kept
// within a cell), each cell padded to whole kBJ-column cell tiles.
struct CellGrid {
  int gc;                       // cells per side
  double x0, y0, inv_side;      // grid origin, 1 / cell side
  int ncls;                     // reach classes per cell (log density bands), 1: none
  double lq0, inv_lq;           // class = floor((log q - lq0) * inv_lq)
};
struct CellLayout {
  const int* perm;              // [npos] position -> column (-1: padding)
  const int* n_ctiles;          // device: cell tiles in use
  int max_tiles;                // allocated tiles (npos = max_tiles * kBJ)
  // per evaluation (prep_cells_kernel), in cell-tile order
  double2 *xy, *wk, *vz;        // {x, y}, {w, K}, {v, z}: w relative to the tile's last time
  float4* fxy;                  // {x - cx, y - cy, thrf}
  double *t, *q;
  // per cell tile: FP32 box of its columns, largest thrf, first and last time
  float4* box;
  float* r2;
  double *tmin, *tmax;
};
void launch_cells(const double* x, const double* y, const double* q, int n, const CellGrid& g, int* cell, int* chunk_counts,
                  int* cell_start, int* perm, int perm_len, int* n_ctiles, cudaStream_t s);

// Row-sum halves: the background [B, B2] and the trigger [T, Td, Tq].
constexpr int kHalfBg = 1, kHalfTr = 2;

// The exp table (hk_device.cuh) of the current device; once per device
// before the first pair launch.
void upload_exp2_table(cudaStream_t s);
// 2^(j/n), j < n, each high word minus (j << (20 - log2 n)) (host).
void make_exp2_table(double* out, int n);
void launch_prep(const DeviceCatalog& d, const EvalCoef& c, cudaStream_t s);
// The cell-tile arrays of this evaluation (after launch_prep's coefficients).
void launch_prep_cells(const DeviceCatalog& d, const EvalCoef& c, const CellLayout& L, cudaStream_t s);
// Spatially clusters the rows [rows_base, rows_base + rows) window by window
// (k-d median splits down to `leaf` rows) into rperm, `window` (a power of
// two) slots per window; slots without a row hold -1.  The nblocks row blocks
// form n_windows windows of near-equal size (window_first_block): a window
// of few rows would cluster badly.  Any order gives bitwise the same per-row
// sums: the clustering only lets the density-scaled trigger skip columns per
// warp.
// block_rows: the row blocks windows are made of (0: the varying plan's).
// Windows of more than kClusterSplitTarget rows (up to kMaxSplitWindow) are
// first split at medians (x, then y, ...) into halves, which are clustered
// separately (scratch: 2 * n_windows * window + cluster_work_ints ints).
inline std::size_t cluster_work_ints(int n_windows, int window) {
  const std::size_t slots = static_cast<std::size_t>(n_windows) * window;
  // hist [256] + sel [4] for up to slots/4096 sub-windows, then 2 counts per 4096-slot chunk
  return slots / 4096 * 260 + slots / 2048 + 4096;
}
void launch_cluster(const double* x, const double* y, int* rperm, int rows_base, int rows,
                    int window, int n_windows, int leaf, double cx, double cy, double half_extent,
                    cudaStream_t s, int block_rows = 0, int* scratch = nullptr);
constexpr int kMaxClusterWindow = 32768;  // rows clustered in shared memory (6.25 bytes each: 200 KB)
constexpr int kMaxSplitWindow = 8 * kMaxClusterWindow;  // rows per window with median splits first
#ifndef HK_CLUSTER_SPLIT_TARGET
#define HK_CLUSTER_SPLIT_TARGET 8192
#endif
constexpr int kClusterSplitTarget = HK_CLUSTER_SPLIT_TARGET;  // split windows down to this many rows
// Windows of at most max_blocks row blocks covering nblocks: their number,
// the first block of window w, and the window of block b.
__host__ __device__ inline int window_count(int nblocks, int max_blocks) {
  return (nblocks + max_blocks - 1) / max_blocks;
}
__host__ __device__ inline int window_first_block(int w, int nblocks, int n_windows) {
  return static_cast<int>(static_cast<long long>(w) * nblocks / n_windows);
}
__host__ __device__ inline int window_of_block(int b, int nblocks, int n_windows) {
  return static_cast<int>((static_cast<long long>(b + 1) * n_windows - 1) / nblocks);
}
// fgt: the trigger of each item's tiles below Item::xt is left out (it is
// added by the Hermite expansion, hk_fgt.cu); homogeneous plan only.
// cells (density-scaled FP64 trigger-only launches): items index cell tiles.
void launch_pair(const DeviceCatalog& d, const EvalCoef& c, const Item* items, int n_items,
                 double* partial, int rows_base, int rows_total, bool with_grad, int halves,
                 cudaStream_t s, bool fgt = false, const CellLayout* cells = nullptr);
// Sums the partial slots per row (fixed order) into the background plane
// pair [B, B2] and/or the trigger planes [T, Td, Tq] (either may be null).
void launch_collapse(const double* partial, int slots, int rows_total, double* bg_sums,
                     double* tr_sums, cudaStream_t s);
// Forms ell_n and its gradient from the row sums and reduces to one
// 6-vector per block; writes per-row outputs when the pointers are non-null.
int launch_finish(const DeviceCatalog& d, const EvalCoef& c, const double* bg_sums,
                  const double* tr_sums, int rows_base, int rows_total, bool with_grad,
                  double* ell_rows, double* grad_rows, double* blockpart, cudaStream_t s);
void launch_reduce(const double* blockpart, int n_blocks, double* out6, cudaStream_t s);
// Certification of the density-scaled trigger's spatial cut (EvalCoef::tr_cut):
// per row Q_i = sum_{j < lb_i} q_j exp(-omega (t_i - t_j)) bounds the weight of
// every dropped source, so the dropped terms are at most Q_i 2^{-tr_cut/kTab};
// a row where c x that exceeds row_tol x S_i sets *flag.  scratch: 4 x
// ceil(n / kCertChunk) doubles.
constexpr int kCertChunk = 1024;
void launch_tr_cut_cert(const DeviceCatalog& d, const EvalCoef& c, const double* bg_sums,
                        const double* tr_sums, int rows_base, int rows_total, double* scratch,
                        double row_tol, unsigned* flag, cudaStream_t s, int lb_last = -1);
// (lb_last: count_before of the shard's last row; the later chunks are left
// out, -1: every chunk)
// Bounding box and finiteness of n locations: out5 = {xmin, xmax, ymin, ymax,
// index of the first non-finite location or n}, on the device; scratch holds
// bbox_scratch_doubles() doubles.
int bbox_scratch_doubles();
void launch_bbox(const double* x, const double* y, int n, double* scratch, double* out5,
                 cudaStream_t s);
// total[k] = sum over d < n_dev of parts[6 d + k], in ascending d.
void launch_sum6(const double* parts, int n_dev, double* total, cudaStream_t s);
double measure_fp64_peak(int device, double* ms);

}  // namespace hk
