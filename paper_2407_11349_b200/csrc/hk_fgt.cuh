// Launch-side view of the homogeneous-trigger Hermite expansion (hk_fgt.cu).
#pragma once

#include <cuda_runtime.h>

namespace hk {

constexpr int kFgtP = 30;              // Hermite terms per dimension (a, b < kFgtP)
constexpr double kFgtGamma = 1.4142135623730951;  // box side / sqrt(delta): rho = 1
constexpr int kFgtBlocks = 4;          // homogeneous row blocks per checkpoint
constexpr int kFgtRowBlock = 512;      // rows per block of the homogeneous plan (rows_per_item(false))
#ifndef HK_FGT_THREADS
#define HK_FGT_THREADS 64
#endif
#ifndef HK_FGT_MINB
#define HK_FGT_MINB 6
#endif
constexpr int kFgtEvalThreads = HK_FGT_THREADS;  // threads per evaluation CTA (the warps share the staged moments)
constexpr int kFgtEvalMinBlocks = HK_FGT_MINB;   // __launch_bounds__ minimum resident CTAs per SM
#ifndef HK_FGT_RPT
#define HK_FGT_RPT 1
#endif
constexpr int kFgtRowsPerThread = HK_FGT_RPT;  // rows per thread (kFgtEvalThreads x this divides kFgtRowBlock)
constexpr int kFgtCkRows = kFgtBlocks * kFgtRowBlock;  // rows per checkpoint (a power of two)
constexpr int kFgtLeaf = 32 * kFgtRowsPerThread;       // one warp's rows: a k-d leaf
static_assert(kFgtCkRows % (kFgtRowsPerThread * kFgtEvalThreads) == 0,
              "an evaluation CTA's rows lie inside one checkpoint");
constexpr double kFgtCut = 36.0;       // boxes farther than 6 scaled units are skipped (<= e^-36 per unit weight)
constexpr double kFgtRowTol = 1e-13;   // certified per-row relative error bound, else recompute directly
constexpr int kFgtMaxBoxes = 1024;     // larger grids (small sigma_x / wide catalogs): direct path
// Per (warp, box) truncation by the distance of the warp's nearest row from
// the box centre: buckets of r^2 (scaled units) -> the kept set {a < a1,
// b < p} u {a1 <= a < p, b < 2 np2} (fgt_truncation_table)
constexpr int kFgtR2Buckets = 256;
constexpr double kFgtR2Step = 0.25;

struct FgtParams {
  int n, ncols;                 // catalog size; columns below the last prefix
  const double *t, *x, *y;
  int nck;                      // checkpoints (ck_off virtual ones, then nck_rows with rows)
  int ck_off, nck_rows;
  const int* P;                 // [nck] prefix boundaries (columns [0, P_k)), nondecreasing
  double* tR;                   // [nck] reference times t[P_k]
  double* decay;                // [nck] exp(-omega (tR_k - tR_{k-1}))
  double* dt;                   // [nck] tR_k - tR_{k-1}
  int nb, nbox;                 // boxes per side, boxes
  double x0, y0, L, inv_sqd;    // grid origin, box side, 1 / sqrt(delta)
  double omega, delta;          // 1 / sigma_t, 2 sigma_x^2
  double eps;                   // truncation bound per unit of box weight
  double row_tol;               // certified per-row relative bound (kFgtRowTol)
  int grad;
  int* box;                     // [ncols]
  double *u, *v;                // [ncols] scaled offsets from the box centre
  double* mom;                  // [nck][nbox][2][kFgtP^2]: A (and B) moments
  double* wsum;                 // [nck] total prefix weight (sum over boxes of A_00)
  const int* perm;              // [nck * kFgtCkRows] each checkpoint's rows in spatial (k-d) order, -1: none
  unsigned short pn[kFgtR2Buckets];  // per r^2 bucket: p | a1 << 5 | np2 << 10
};

// The background's 1-D expansion in time (hk_fgt.cu, both variants).
constexpr int kBgFgtMaxBoxes = 1 << 16;
struct BgFgtParams {
  int n;                        // catalog size
  const double* t;              // sorted times
  const int *lb, *ub;           // tie bounds (count_before / upper_bound)
  int nbt;                      // time boxes
  double t0, L, inv_sqd;        // first time, box side gamma sqrt(2 tau^2), 1/sqrt(2 tau^2)
  double delta;                 // 2 tau^2
  double eps, row_tol;          // truncation bound per unit weight; certified relative bound
  double* mom;                  // [nbt][kFgtP] moments
  int* count;                   // [nbt] columns per box
};
double bg_fgt_truncation_bound(int p, double gamma);
// moments (of the boxes within reach of times [t_first, t_last]: the rows'
// first and last) + the rows [rows_base, rows_base + rows_total): bg_sums
// planes B, B2.
// part: scratch of boxes x bg_fgt_parts(n, boxes) x kFgtP doubles (boxes: at
// most nbt).
void launch_bg_fgt(const BgFgtParams& F, int rows_base, int rows_total, double* bg_sums, unsigned* flag,
                   cudaStream_t s, double t_first, double t_last, double* part);
int bg_fgt_parts(int n, int boxes);

// eps_p of hk_fgt.cu for p terms and box side gamma sqrt(delta).
double fgt_truncation_bound(int p, double gamma);
// Per r^2 bucket k (r^2 >= k kFgtR2Step): the kept set {a < a1, b < p} u
// {a1 <= a < p, b < 2 np2}, p <= kFgtP, with the fewest multiply-adds whose
// dropped terms are bounded by `target` per unit of box weight for every row
// at least sqrt(k kFgtR2Step) from the box centre.
void fgt_truncation_table(double gamma, double target, unsigned short* pn);
// reference times, box assignment, increment moments and their scan.
void launch_fgt_prepare(const FgtParams& F, cudaStream_t s);
// adds the expansion's trigger sums into tr_sums (planes T, Td, Tq of
// rows_total rows); sets *flag when a row's certified bound fails.
void launch_fgt_eval(const FgtParams& F, int rows_base, int rows_total, const double* bg_sums,
                     double* tr_sums, double coef_a, double coef_c, unsigned* flag, cudaStream_t s);

}  // namespace hk
