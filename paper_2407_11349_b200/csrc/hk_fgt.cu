// Homogeneous trigger by a Hermite (fast Gauss transform) expansion.
//
// The homogeneous pair kernel spends ~all of its time on the dense O(N^2/2)
// trigger of its BT tiles: for a row i and every earlier column j
//   g_ij = exp(-omega (t_i - t_j)) exp(-|x_i - x_j|^2 / delta),  delta = 2 sigma_x^2
// (model.hpp:146-170 with q_j = 1).  With a reference time t_R no later than
// the row and no earlier than the columns, the temporal factor splits into a
// row factor E_i = exp(-omega (t_i - t_R)) and a column weight
// W_j = exp(-omega (t_R - t_j)), so the BT part of T_i is E_i times a 2-D
// Gauss transform of the earlier columns with weights W_j.  Spatial boxes of
// side L = gamma sqrt(delta) and, in 1-D with s = (x - c)/sqrt(delta),
// u = (x_j - c)/sqrt(delta) about the box centre c,
//   exp(-(s - u)^2) = sum_n u^n / n! h_n(s),   h_n(s) = H_n(s) e^{-s^2}
// (Hermite functions), so per box and per checkpoint (a prefix of the
// columns) the moments
//   A_ab = sum_j W_j u_j^a v_j^b / (a! b!),  B_ab = sum_j (t_R - t_j) W_j u_j^a v_j^b / (a! b!)
// give, for every later row,
//   T  += E_i sum_ab A_ab h_a(X) h_b(Y)
//   Td += E_i [(t_i - t_R) sum_ab A_ab h_a h_b + sum_ab B_ab h_a h_b]
//   Tq += E_i delta [ sum_ab A_ab h_a h_b + (sum_ab A_ab h_{a+2} h_b + A_ab h_a h_{b+2}) / 4 ]
// (Tq: d^2 e^{-d^2/delta} with s^2 e^{-s^2} = (h_2(s) + 2 h_0(s)) / 4 and the
// Taylor series of h_2).  Truncation at a, b < kFgtP: with rho = sqrt(2) *
// max|u| = gamma / sqrt(2) and Cramer's bound |h_n(s)| <= K 2^{n/2} sqrt(n!)
// (K < 1.0865), the dropped terms are below
//   eps_p = 2 K^2 C(rho) rho^p / sqrt(p!) / (1 - rho / sqrt(p+1))
// per unit of box weight (gamma = sqrt 2, p = 30: 6.1e-16).  The same bound
// carries a factor e^{-r^2/2} for a row at scaled distance r from the box
// centre (Cramer: |h_n(s)| <= K 2^{n/2} sqrt(n!) e^{-s^2/2}, in both
// dimensions), so a farther box needs fewer terms: per warp and box the
// evaluation keeps two rectangles {a < a1, b < p} u {a1 <= a < p, b < b2}
// (each a rolled loop over a with a fully unrolled b loop) with the fewest
// terms whose dropped terms, summed exactly (fgt_truncation_table), stay
// below eps_30 at the warp's nearest row (every box within eps_30).  Boxes whose
// nearest point is more than sqrt(kFgtCut) scaled units from the row are
// skipped (weight factor <= e^{-46}).  Both bounds, per row, are compared
// with the row's rate S_i after the sum: a row whose certified error could
// exceed kFgtRowTol relative raises a flag and the host recomputes the
// evaluation on the direct path (hk_capi.cu).
//
// Checkpoints: every kFgtBlocks row blocks of the homogeneous plan (512 rows
// each) share one prefix P_k = floor(lb(first row) / 256) * 256 of columns;
// the pair kernel evaluates the trigger of the tiles below P_k / 256 no more
// (Item::xt), so the columns [P_k, lb_i) stay on the direct path.  Per
// evaluation: box assignment O(N), per-checkpoint increment moments (one CTA
// per checkpoint, sources summed per box in column order), a scan over the
// checkpoints (decay to the new reference time), then the evaluation (one
// thread per row, moments staged per box by bulk async copies) adds E_i x
// (box sums) into the trigger row sums.  No floating-point atomics: bitwise
// deterministic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "hk_device.cuh"
#include "hk_fgt.cuh"

namespace hk {

namespace {

constexpr int P = kFgtP;
constexpr int PP = kFgtP * kFgtP;

// 1 / (n + 1), n < P: the power tables u^n / n! by multiplications (an FP64
// division is a long instruction sequence on the GPU)
struct Recip {
  double v[P];
};
constexpr Recip make_recip() {
  Recip r{};
  for (int n = 0; n < P; ++n) r.v[n] = 1.0 / (n + 1);
  return r;
}
__constant__ Recip c_recip = make_recip();

// ---------------------------------------------------------------------------
// per checkpoint: reference time, decay from the previous one

__global__ void fgt_refs_kernel(const FgtParams F) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= F.nck) return;
  const double tr = F.t[F.P[k]];
  F.tR[k] = tr;
  if (k == 0) {
    F.decay[0] = 0.0;
    F.dt[0] = 0.0;
  } else {
    const double dt = tr - F.t[F.P[k - 1]];
    F.dt[k] = dt;
    F.decay[k] = exp(-F.omega * dt);
  }
}

// per column below the last prefix: box and scaled offsets from its centre
__global__ void fgt_assign_kernel(const FgtParams F) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= F.ncols) return;
  const double x = F.x[j], y = F.y[j];
  const int bx = min(max(static_cast<int>(floor((x - F.x0) / F.L)), 0), F.nb - 1);
  const int by = min(max(static_cast<int>(floor((y - F.y0) / F.L)), 0), F.nb - 1);
  F.box[j] = bx + F.nb * by;
  HK_ASSERT(bx + F.nb * by < F.nbox && F.nbox <= kFgtMaxBoxes);
  F.u[j] = (x - (F.x0 + (bx + 0.5) * F.L)) * F.inv_sqd;
  F.v[j] = (y - (F.y0 + (by + 0.5) * F.L)) * F.inv_sqd;
}

// ---------------------------------------------------------------------------
// increment moments of checkpoint k: sources [P_{k-1}, P_k), weights relative
// to t_R(k).  One warp per box (boxes strided over the CTA's warps); the
// box's sources are compacted in column order, their power tables u^a/a!,
// v^b/b! staged in shared memory, and each lane sums its coefficients over
// the sources in that order.

constexpr int kMomThreads = 256;
constexpr int kMomWarps = kMomThreads / 32;
constexpr int kMomBatch = 16;   // sources per batch and warp
constexpr int kMomSort = 2048;  // sources sorted by box per pass (a power of two)
// dynamic shared memory: per warp kMomBatch x 3P doubles (W u^a/a!, (t_R - t) W u^a/a!, v^b/b!),
// then the pass's sort keys and each box's first position
constexpr int kMomSmem = kMomWarps * kMomBatch * (3 * P) * static_cast<int>(sizeof(double)) +
                         kMomSort * static_cast<int>(sizeof(unsigned)) +
                         (kFgtMaxBoxes + 1) * static_cast<int>(sizeof(int));

// adds the batch's sources (in batch order) to the box's coefficients held
// in registers: lane b (< P) owns the coefficients (a, b) of both sets for
// every a, so per source it reads its v^b/b! once and the broadcast u^a/a!
// weights
__device__ __forceinline__ void fgt_accumulate(double (&accA)[P], double (&accB)[P], bool grad, int nb,
                                               const double* wpu, const double* pv, int lane) {
  if (lane >= P) return;
  for (int s = 0; s < nb; ++s) {
    const double vb = pv[s * P + lane];
    const double* wa = wpu + s * 2 * P;  // [W u^a / a!, (t_R - t) W u^a / a!]
#pragma unroll
    for (int a = 0; a < P; ++a) {
      accA[a] = fma(wa[a], vb, accA[a]);
      if (grad) accB[a] = fma(wa[P + a], vb, accB[a]);
    }
  }
}

// One CTA per checkpoint interval [P_{k-1}, P_k): its sources are sorted by
// (box, column) in shared memory (bitonic, kMomSort per pass), so every box's
// sources are one contiguous run, summed in column order by one warp.
__global__ void __launch_bounds__(kMomThreads) fgt_moments_kernel(const FgtParams F) {
  extern __shared__ __align__(16) double s_dyn[];
  const int k = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* wpu = s_dyn + warp * kMomBatch * (3 * P);  // [s][2][P]
  double* pv = wpu + kMomBatch * 2 * P;              // [s][P]
  unsigned* keys = reinterpret_cast<unsigned*>(s_dyn + kMomWarps * kMomBatch * 3 * P);
  int* start = reinterpret_cast<int*>(keys + kMomSort);
  const int j0 = k ? F.P[k - 1] : 0, j1 = F.P[k];
  const double tR = F.tR[k];
  const bool grad = F.grad != 0;
  double* out = F.mom + static_cast<size_t>(k) * F.nbox * 2 * PP;
  if (j1 <= j0)  // an empty interval: zero increments
    for (int c = threadIdx.x; c < F.nbox * 2 * PP; c += kMomThreads)
      if (grad || c % (2 * PP) < PP) out[c] = 0.0;
  for (int p0 = j0; p0 < j1; p0 += kMomSort) {
    const int cnt = min(kMomSort, j1 - p0);
    __syncthreads();  // the previous pass is done with keys / start and its stores are visible
    for (int i = threadIdx.x; i < kMomSort; i += kMomThreads)
      keys[i] = i < cnt ? (static_cast<unsigned>(F.box[p0 + i]) << 12) | static_cast<unsigned>(i) : 0xffffffffu;
    HK_ASSERT(j1 <= F.ncols && kMomSort <= 4096);
    __syncthreads();
    for (int kk = 2; kk <= kMomSort; kk <<= 1)
      for (int jj = kk >> 1; jj > 0; jj >>= 1) {
        for (int i = threadIdx.x; i < kMomSort; i += kMomThreads) {
          const int l = i ^ jj;
          if (l > i) {
            const unsigned x = keys[i], y = keys[l];
            if ((x > y) == ((i & kk) == 0)) {
              keys[i] = y;
              keys[l] = x;
            }
          }
        }
        __syncthreads();
      }
    for (int B = threadIdx.x; B <= F.nbox; B += kMomThreads) {  // first position of box B
      int lo = 0, hi = cnt;
      const unsigned kb = static_cast<unsigned>(B) << 12;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (keys[mid] < kb) lo = mid + 1;
        else hi = mid;
      }
      start[B] = lo;
    }
    __syncthreads();
    for (int B = warp; B < F.nbox; B += kMomWarps) {
      double* ob = out + static_cast<size_t>(B) * 2 * PP;
      // the box's coefficients stay in registers over its sources: written
      // once per pass (the first pass starts from zero: no fill, no reload)
      double accA[P], accB[P];
      const bool first = p0 == j0;
#pragma unroll
      for (int a = 0; a < P; ++a) {
        accA[a] = (first || lane >= P) ? 0.0 : ob[a * P + lane];
        accB[a] = (first || lane >= P || !grad) ? 0.0 : ob[PP + a * P + lane];
      }
      for (int s0 = start[B]; s0 < start[B + 1]; s0 += kMomBatch) {
        const int nb = min(kMomBatch, start[B + 1] - s0);
        if (lane < nb) {
          const int j = p0 + static_cast<int>(keys[s0 + lane] & 0xfffu);
          const double u = F.u[j], v = F.v[j];
          const double dtj = tR - F.t[j];
          const double wj = exp(-F.omega * dtj);
          double a1 = wj, a2 = dtj * wj, b1 = 1.0;
#pragma unroll 1
          for (int n = 0; n < P; ++n) {
            wpu[lane * 2 * P + n] = a1;
            wpu[lane * 2 * P + P + n] = a2;
            pv[lane * P + n] = b1;
            const double f = c_recip.v[n];
            a1 = a1 * u * f;
            a2 = a2 * u * f;
            b1 = b1 * v * f;
          }
        }
        __syncwarp();
        fgt_accumulate(accA, accB, grad, nb, wpu, pv, lane);
        __syncwarp();
      }
      if (lane < P)
#pragma unroll
        for (int a = 0; a < P; ++a) {
          ob[a * P + lane] = accA[a];
          if (grad) ob[PP + a * P + lane] = accB[a];
        }
    }
  }
}

// prefix moments over the checkpoints, in place: M_A[k] = d_k M_A[k-1] +
// inc_A[k], M_B[k] = d_k (M_B[k-1] + dt_k M_A[k-1]) + inc_B[k]
__global__ void fgt_scan_kernel(const FgtParams F) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;  // (box, a, b)
  if (c >= F.nbox * PP) return;
  const int B = c / PP, ab = c % PP;
  double ma = 0.0, mb = 0.0;
#pragma unroll 4
  for (int k = 0; k < F.nck; ++k) {
    double* m = F.mom + (static_cast<size_t>(k) * F.nbox + B) * 2 * PP + ab;
    const double d = F.decay[k], dt = F.dt[k];
    const double ia = m[0];
    const double na = fma(d, ma, ia);
    if (F.grad) {
      const double nbv = fma(d, fma(dt, ma, mb), m[PP]);
      m[PP] = nbv;
      mb = nbv;
    }
    m[0] = na;
    ma = na;
  }
}

// ---------------------------------------------------------------------------
// evaluation: one thread per row, kFgtEvalThreads rows per CTA (inside one
// checkpoint's row blocks); every box's moments are staged in shared memory
// by a bulk async copy (double-buffered, mbarrier-tracked).

template <bool kGrad>
__device__ __forceinline__ void hermite(double s, double (&h)[P + 2]) {
  h[0] = exp(-s * s);
  h[1] = 2.0 * s * h[0];
#pragma unroll
  for (int n = 1; n < P + 1; ++n) h[n + 1] = fma(2.0 * s, h[n], -2.0 * n * h[n - 1]);
}

// sA += sum_{b < 2 NP} A_ab h_b (and the gradient chains) for the
// kFgtRowsPerThread rows: NP pairs of b, fully unrolled.
template <int NP, bool kGrad>
__device__ __forceinline__ void row_pairs(const double* __restrict__ Ar, const double (&hy)[kFgtRowsPerThread][P + 2],
                                          double (&sA)[kFgtRowsPerThread], double (&sA2)[kFgtRowsPerThread],
                                          double (&sB)[kFgtRowsPerThread]) {
  static_assert(2 * NP <= P, "pairs of b below P");
  constexpr int R = kFgtRowsPerThread;
#pragma unroll
  for (int b = 0; b < 2 * NP; b += 2) {
    const double2 ab = *reinterpret_cast<const double2*>(Ar + b);
    double2 bb;
    if (kGrad) bb = *reinterpret_cast<const double2*>(Ar + PP + b);
    // the b terms of every chain first, then the b+1 terms: each
    // accumulator's dependent multiply-adds are 2 R (grad: 3 R) - 1
    // independent ones apart (the DFMA latency is hidden in-thread)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      sA[r] = fma(ab.x, hy[r][b], sA[r]);
      if (kGrad) {
        sA2[r] = fma(ab.x, hy[r][b + 2], sA2[r]);
        sB[r] = fma(bb.x, hy[r][b], sB[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      sA[r] = fma(ab.y, hy[r][b + 1], sA[r]);
      if (kGrad) {
        sA2[r] = fma(ab.y, hy[r][b + 3], sA2[r]);
        sB[r] = fma(bb.y, hy[r][b + 1], sB[r]);
      }
    }
  }
}

// Moment rows [a0, a_end) over b < 2 NP: t0 += sum_a h_a(X) S_a, S_a =
// sum_b A_ab h_b(Y), and the gradient sums; h_a by the running three-term
// recurrence (ha = h_a, ha1 = h_{a+1}, ha2 = h_{a+2} on entry and exit).
template <int NP, bool kGrad>
__device__ __forceinline__ void rect_rows(const double* __restrict__ A, int a0, int a_end,
                                          const double (&hy)[kFgtRowsPerThread][P + 2],
                                          const double (&X2)[kFgtRowsPerThread], double (&ha)[kFgtRowsPerThread],
                                          double (&ha1)[kFgtRowsPerThread], double (&ha2)[kFgtRowsPerThread],
                                          double (&t0)[kFgtRowsPerThread], double (&q1)[kFgtRowsPerThread],
                                          double (&q2)[kFgtRowsPerThread], double (&b0)[kFgtRowsPerThread]) {
  constexpr int R = kFgtRowsPerThread;
#pragma unroll 1
  for (int a = a0; a < a_end; ++a) {
    double sA[R], sA2[R], sB[R];
#pragma unroll
    for (int r = 0; r < R; ++r) sA[r] = sA2[r] = sB[r] = 0.0;
    row_pairs<NP, kGrad>(A + a * P, hy, sA, sA2, sB);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      t0[r] = fma(ha[r], sA[r], t0[r]);
      if (kGrad) {
        q1[r] = fma(ha2[r], sA[r], q1[r]);
        q2[r] = fma(ha[r], sA2[r], q2[r]);
        b0[r] = fma(ha[r], sB[r], b0[r]);
      }
      const double ha3 = fma(X2[r], ha2[r], -2.0 * (a + 2) * ha1[r]);  // h_{a+3}
      ha[r] = ha1[r];
      ha1[r] = ha2[r];
      ha2[r] = ha3;
    }
  }
}

// rect_rows for a run-time pair count (warp-uniform; once per rectangle)
template <bool kGrad>
__device__ __forceinline__ void rect_dispatch(int np, const double* __restrict__ A, int a0, int a_end,
                                              const double (&hy)[kFgtRowsPerThread][P + 2],
                                              const double (&X2)[kFgtRowsPerThread], double (&ha)[kFgtRowsPerThread],
                                              double (&ha1)[kFgtRowsPerThread], double (&ha2)[kFgtRowsPerThread],
                                              double (&t0)[kFgtRowsPerThread], double (&q1)[kFgtRowsPerThread],
                                              double (&q2)[kFgtRowsPerThread], double (&b0)[kFgtRowsPerThread]) {
  if (a0 >= a_end) return;
  static_assert(P == 30, "the cases below cover 15 pairs");
  switch (np) {
#define HK_FGT_CASE(k) \
  case k:              \
    rect_rows<k, kGrad>(A, a0, a_end, hy, X2, ha, ha1, ha2, t0, q1, q2, b0); \
    break;
    HK_FGT_CASE(1) HK_FGT_CASE(2) HK_FGT_CASE(3) HK_FGT_CASE(4) HK_FGT_CASE(5)
    HK_FGT_CASE(6) HK_FGT_CASE(7) HK_FGT_CASE(8) HK_FGT_CASE(9) HK_FGT_CASE(10)
    HK_FGT_CASE(11) HK_FGT_CASE(12) HK_FGT_CASE(13) HK_FGT_CASE(14) HK_FGT_CASE(15)
#undef HK_FGT_CASE
    default: break;
  }
}

// kFgtRowsPerThread rows per thread (rows li and li + kFgtEvalThreads of the
// CTA's 2 x kFgtEvalThreads rows): every moment pair read from shared memory
// feeds both rows' multiply-adds (half the loads per FMA, twice the
// independent accumulation chains per warp).
template <bool kGrad>
__global__ void __launch_bounds__(kFgtEvalThreads, kFgtEvalMinBlocks)
    fgt_eval_kernel(const FgtParams F, int rows_base, int rows_total, const double* __restrict__ bg_sums,
                    double* __restrict__ tr_sums, double coef_a, double coef_c, unsigned* flag) {
  constexpr int R = kFgtRowsPerThread;
  constexpr int kSets = kGrad ? 2 : 1;
  constexpr unsigned kBoxBytes = kSets * PP * sizeof(double);
  __shared__ __align__(128) double s_m[2][kSets * PP];
  __shared__ __align__(8) uint64_t s_bar[2];
  // positions in the checkpoint's spatially clustered order (cluster_kernel,
  // windows = checkpoints, leaves = one warp's kFgtLeaf rows): a warp's rows
  // are close together, so boxes beyond the cut-off of all of them are skipped
  const int cta_rows = R * kFgtEvalThreads;
  const int k = F.ck_off + (blockIdx.x * cta_rows) / kFgtCkRows;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int li[R];
  bool valid[R];
  double xi[R], yi[R], ti[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int pos = blockIdx.x * cta_rows + warp * kFgtLeaf + r * 32 + lane;
    HK_ASSERT(pos < F.nck_rows * kFgtCkRows && k < F.nck);
    const int row = F.perm[pos];
    HK_ASSERT(row < 0 || (row >= rows_base && row < rows_base + rows_total));
    valid[r] = row >= 0;
    li[r] = valid[r] ? row - rows_base : 0;
    const int rr = valid[r] ? row : rows_base;
    xi[r] = F.x[rr];
    yi[r] = F.y[rr];
    ti[r] = F.t[rr];
  }
  const double* mk = F.mom + static_cast<size_t>(k) * F.nbox * 2 * PP;
  if (threadIdx.x == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_fence_init();
  }
  // the boxes some row of the CTA can use (the per-row test below, on the
  // CTA's bounding box with a margin): the others are neither staged nor
  // visited.  A skipped box changes no row's sums.
  __shared__ int s_boxes[kFgtMaxBoxes];
  __shared__ int s_nboxes;
  __shared__ double s_bb[4][kFgtEvalThreads / 32];
  {
    const double kInfD = __longlong_as_double(0x7ff0000000000000LL);
    double x0 = kInfD, x1 = -kInfD, y0 = kInfD, y1 = -kInfD;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (valid[r]) {
        x0 = fmin(x0, xi[r]);
        x1 = fmax(x1, xi[r]);
        y0 = fmin(y0, yi[r]);
        y1 = fmax(y1, yi[r]);
      }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      x0 = fmin(x0, __shfl_xor_sync(0xffffffffu, x0, off));
      x1 = fmax(x1, __shfl_xor_sync(0xffffffffu, x1, off));
      y0 = fmin(y0, __shfl_xor_sync(0xffffffffu, y0, off));
      y1 = fmax(y1, __shfl_xor_sync(0xffffffffu, y1, off));
    }
    if (lane == 0) {
      s_bb[0][warp] = x0;
      s_bb[1][warp] = x1;
      s_bb[2][warp] = y0;
      s_bb[3][warp] = y1;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int w = 1; w < kFgtEvalThreads / 32; ++w) {
        x0 = fmin(x0, s_bb[0][w]);
        x1 = fmax(x1, s_bb[1][w]);
        y0 = fmin(y0, s_bb[2][w]);
        y1 = fmax(y1, s_bb[3][w]);
      }
      int base = 0;
      for (int B0 = 0; B0 < F.nbox; B0 += 32) {
        const int B = B0 + lane;
        bool keep = false;
        if (B < F.nbox) {
          const double cxB = F.x0 + (B % F.nb + 0.5) * F.L, cyB = F.y0 + (B / F.nb + 0.5) * F.L;
          const double gx = fmax(fmax(x0 - cxB, cxB - x1) * F.inv_sqd - 0.5 * F.L * F.inv_sqd, 0.0);
          const double gy = fmax(fmax(y0 - cyB, cyB - y1) * F.inv_sqd - 0.5 * F.L * F.inv_sqd, 0.0);
          keep = fma(gx, gx, gy * gy) <= kFgtCut * (1.0 + 1e-9) + 1e-9;  // margin: a superset of the rows' tests
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (keep) s_boxes[base + __popc(m & ((1u << lane) - 1u))] = B;
        base += __popc(m);
      }
      if (lane == 0) s_nboxes = base;
    }
  }
  __syncthreads();
  const int nbx = s_nboxes;
  const bool any = F.P[k] > 0;  // checkpoint with no earlier columns: nothing to add
  double T[R], Td[R], Tq[R], Tq2[R], w_used[R];  // w_used: box weights (A_00 = sum W) evaluated
#pragma unroll
  for (int r = 0; r < R; ++r) T[r] = Td[r] = Tq[r] = Tq2[r] = w_used[r] = 0.0;
  const double hs = 0.5 * F.L * F.inv_sqd;  // half box side, scaled
  if (any && nbx > 0) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(&s_bar[0], kBoxBytes);
      bulk_g2s(s_m[0], mk + static_cast<size_t>(s_boxes[0]) * 2 * PP, kBoxBytes, &s_bar[0]);
    }
    unsigned phases = 0u;
    for (int ib = 0; ib < nbx; ++ib) {
      const int B = s_boxes[ib];
      const int st = ib & 1;
      if (ib + 1 < nbx && threadIdx.x == 0) {
        mbar_expect_tx(&s_bar[st ^ 1], kBoxBytes);
        bulk_g2s(s_m[st ^ 1], mk + static_cast<size_t>(s_boxes[ib + 1]) * 2 * PP, kBoxBytes, &s_bar[st ^ 1]);
      }
      mbar_wait(&s_bar[st], (phases >> st) & 1u);
      phases ^= 1u << st;
      const double* A = s_m[st];
      const int bx = B % F.nb, by = B / F.nb;
      const double cxB = F.x0 + (bx + 0.5) * F.L, cyB = F.y0 + (by + 0.5) * F.L;
      double X[R], Y[R];
      bool use[R], any_use = false;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        X[r] = (xi[r] - cxB) * F.inv_sqd;
        Y[r] = (yi[r] - cyB) * F.inv_sqd;
        const double dx = fmax(fabs(X[r]) - hs, 0.0), dy = fmax(fabs(Y[r]) - hs, 0.0);
        use[r] = valid[r] && fma(dx, dx, dy * dy) <= kFgtCut;
        if (use[r]) w_used[r] += A[0];  // sum of the box's weights (>= 0)
        any_use = any_use || use[r];
      }
      if (__any_sync(0xffffffffu, any_use)) {
        // the truncation for the warp's nearest row that uses the box
        double r2m = 1e300;
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (use[r]) r2m = fmin(r2m, fma(X[r], X[r], Y[r] * Y[r]));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) r2m = fmin(r2m, __shfl_xor_sync(0xffffffffu, r2m, off));
        const int kb = static_cast<int>(fmin(r2m * (1.0 / kFgtR2Step), kFgtR2Buckets - 1.0));
        const unsigned pn = F.pn[kb];
        const int p = static_cast<int>(pn & 31u), a1 = static_cast<int>((pn >> 5) & 31u),
                  np2 = static_cast<int>(pn >> 10);
        HK_ASSERT(p >= 1 && p <= P && a1 <= p && np2 >= 1 && np2 <= (p + 1) / 2);
        // h_b(Y) for every b (register arrays, static indices); h_a(X) by the
        // running three-term recurrence inside the a loop (the loop stays
        // rolled: a fully unrolled P x P body overflows the instruction cache)
        double hy[R][P + 2];
        double X2[R], ha[R], ha1[R], ha2[R];
        double t0[R], q1[R], q2[R], b0[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          hermite<kGrad>(Y[r], hy[r]);
          X2[r] = 2.0 * X[r];
          ha[r] = exp(-X[r] * X[r]);
          ha1[r] = X2[r] * ha[r];
          ha2[r] = fma(X2[r], ha1[r], -2.0 * ha[r]);
          t0[r] = q1[r] = q2[r] = b0[r] = 0.0;
        }
        // rows a < a1 over b < p, rows a1 <= a < p over b < 2 np2 (pairs
        // of b; with p odd the extra column b = p only shrinks the bound)
        rect_dispatch<kGrad>((p + 1) >> 1, A, 0, a1, hy, X2, ha, ha1, ha2, t0, q1, q2, b0);
        rect_dispatch<kGrad>(np2, A, a1, p, hy, X2, ha, ha1, ha2, t0, q1, q2, b0);
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (use[r]) {
            T[r] += t0[r];
            if (kGrad) {
              Td[r] += b0[r];
              Tq[r] += q1[r];
              Tq2[r] += q2[r];
            }
          }
      }
      __syncthreads();  // every warp is done with this stage before it is refilled
    }
  }
  if (!any) return;
  const double tR = F.tR[k];
  double* trT = tr_sums;
  double* trTd = tr_sums + rows_total;
  double* trTq = tr_sums + 2 * static_cast<size_t>(rows_total);
  // the boxes not evaluated are farther than sqrt(kFgtCut) scaled units:
  // their total weight (the prefix's, sum_B A_00, minus the evaluated boxes')
  // contributes at most e^{-kFgtCut} per unit
  const double w_all = F.wsum[k];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (!valid[r]) continue;
    const double E = exp(-F.omega * (ti[r] - tR));
    const double Ttot = trT[li[r]] + E * T[r];
    trT[li[r]] = Ttot;
    if (kGrad) {
      trTd[li[r]] += E * fma(ti[r] - tR, T[r], Td[r]);
      trTq[li[r]] += E * F.delta * fma(0.25, Tq[r] + Tq2[r], T[r]);
    }
    // certification: what the expansion may have dropped (truncation per
    // unit weight of the boxes used, the cut boxes' weight bound) against
    // the row's rate S_i = a B_i + c T_i (gradient terms: same weights, the
    // h_{n+2} terms inflate the truncation bound by at most 2 (p + 1))
    const double err = coef_c * E * (F.eps * w_used[r] + fmax(w_all - w_used[r], 0.0) * exp(-kFgtCut));
    const double S = coef_a * bg_sums[li[r]] + coef_c * Ttot;
    if (!(err <= F.row_tol * S)) atomicOr(flag, 1u);
  }
}

// the total weight of each checkpoint's prefix (sum over boxes of A_00)
__global__ void fgt_wsum_kernel(const FgtParams F) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= F.nck) return;
  double w = 0.0;
  for (int B = 0; B < F.nbox; ++B) w += F.mom[(static_cast<size_t>(k) * F.nbox + B) * 2 * PP];
  F.wsum[k] = w;
}

// ---------------------------------------------------------------------------
// The background as a 1-D Hermite expansion in time (both variants):
//   B_i  = sum_{t_j != t_i} exp(-(t_i - t_j)^2 / delta_t),  delta_t = 2 tau^2
//   B2_i = sum_{t_j != t_i} (t_i - t_j)^2 exp(...)
// (model.hpp:124-140 and the gradient's B2).  Time boxes of side
// gamma sqrt(delta_t) are contiguous index ranges of the sorted times; with
// unit weights A_n = sum_{j in box} u_j^n / n! the full sums over every j are
//   Bfull_i  = sum_box sum_n A_n h_n(X),
//   B2full_i = delta_t [ sum_box sum_n A_n h_{n+2}(X) / 4 + Bfull_i / 2 ],
// and the tied columns (self included) add exactly 1 each to Bfull and 0 to
// B2full: B_i = Bfull_i - (ub_i - lb_i).  Certification per row: truncation
// eps per unit weight x the counts of the boxes used, the cut boxes' counts x
// e^{-d^2}, and the rounding of Bfull against B_i itself (S_i >= a B_i).

constexpr int kBgThreads = 256;

// box ranges (binary search of each box's first time) and moments: CTA
// (b, s) sums the s-th of gridDim.y equal parts of box b's columns into
// part[(b - b_lo) gridDim.y + s] (thread-strided partial sums, warp
// butterflies, warps in order); bg_fgt_reduce_kernel adds the parts in order.
// Deterministic for a fixed part count.
__global__ void __launch_bounds__(kBgThreads) bg_fgt_moments_kernel(const BgFgtParams F, int b_lo, double* part) {
  __shared__ double s_w[kBgThreads / 32][P];
  __shared__ int s_range[2];
  const int b = b_lo + blockIdx.x, S = gridDim.y, sidx = blockIdx.y;
  if (threadIdx.x < 2) {
    const int box = b + threadIdx.x;  // first index whose box >= `box`
    int lo = 0, hi = F.n;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const int bx = min(max(static_cast<int>(floor((F.t[mid] - F.t0) / F.L)), 0), F.nbt - 1);
      if (bx < box) lo = mid + 1;
      else hi = mid;
    }
    s_range[threadIdx.x] = box >= F.nbt ? F.n : lo;
  }
  __syncthreads();
  const int b0 = s_range[0], b1 = s_range[1];
  const long long len = b1 - b0;
  const int j0 = b0 + static_cast<int>(len * sidx / S), j1 = b0 + static_cast<int>(len * (sidx + 1) / S);
  const double c = F.t0 + (b + 0.5) * F.L;
  double acc[P];
#pragma unroll
  for (int n = 0; n < P; ++n) acc[n] = 0.0;
  for (int j = j0 + threadIdx.x; j < j1; j += kBgThreads) {
    const double u = (F.t[j] - c) * F.inv_sqd;
    double pw = 1.0;
#pragma unroll
    for (int n = 0; n < P; ++n) {
      acc[n] += pw;
      pw = pw * u * c_recip.v[n];
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int n = 0; n < P; ++n) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc[n] += __shfl_xor_sync(0xffffffffu, acc[n], off);
    if (lane == 0) s_w[warp][n] = acc[n];
  }
  __syncthreads();
  if (threadIdx.x < P) {
    double v = s_w[0][threadIdx.x];
#pragma unroll
    for (int w = 1; w < kBgThreads / 32; ++w) v += s_w[w][threadIdx.x];
    part[(static_cast<size_t>(blockIdx.x) * S + sidx) * P + threadIdx.x] = v;
  }
  if (threadIdx.x == 0 && sidx == 0) F.count[b] = b1 - b0;
}

__global__ void bg_fgt_reduce_kernel(const BgFgtParams F, int b_lo, int S, const double* __restrict__ part) {
  const int n = threadIdx.x, bi = blockIdx.x;
  if (n >= P) return;
  double v = 0.0;
  for (int s = 0; s < S; ++s) v += part[(static_cast<size_t>(bi) * S + s) * P + n];
  F.mom[(b_lo + bi) * P + n] = v;
}

__global__ void __launch_bounds__(kBgThreads) bg_fgt_eval_kernel(const BgFgtParams F, int rows_base,
                                                                  int rows_total, double* bg_sums,
                                                                  unsigned* flag) {
  const int li = blockIdx.x * kBgThreads + threadIdx.x;
  if (li >= rows_total) return;
  const int row = rows_base + li;
  const double ti = F.t[row];
  const double reach = sqrt(kFgtCut) / F.inv_sqd + 0.5 * F.L;  // box centres farther: cut
  const int b0 = max(0, static_cast<int>(floor((ti - reach - F.t0) / F.L)));
  const int b1 = min(F.nbt - 1, static_cast<int>(floor((ti + reach - F.t0) / F.L)));
  const double hs = 0.5 * F.L * F.inv_sqd;
  // every box outside [b0, b1] is farther than sqrt(kFgtCut) scaled units:
  // its columns add at most e^{-kFgtCut} each (the `cut` bound below)
  double Bf = 0.0, Q = 0.0, used = 0.0;
  for (int b = b0; b <= b1; ++b) {
    const double X = (ti - (F.t0 + (b + 0.5) * F.L)) * F.inv_sqd;
    const double d = fmax(fabs(X) - hs, 0.0);
    if (d * d > kFgtCut) continue;
    used += F.count[b];
    HK_ASSERT(b >= 0 && b < F.nbt);
  const double* A = F.mom + b * P;
    const double X2 = 2.0 * X;
    double h0 = exp(-X * X), h1 = X2 * h0;
    double h2 = fma(X2, h1, -2.0 * h0);
    double s0 = 0.0, s2 = 0.0;
#pragma unroll
    for (int n = 0; n < P; ++n) {
      s0 = fma(A[n], h0, s0);
      s2 = fma(A[n], h2, s2);
      const double h3 = fma(X2, h2, -2.0 * (n + 2) * h1);
      h0 = h1;
      h1 = h2;
      h2 = h3;
    }
    Bf += s0;
    Q += s2;
  }
  const double ties = static_cast<double>(F.ub[row] - F.lb[row]);
  const double B = Bf - ties;
  const double B2 = F.delta * fma(0.25, Q, 0.5 * Bf);
  bg_sums[li] = B;
  bg_sums[rows_total + li] = B2;
  const double cut = (F.n - used) * exp(-kFgtCut);
  const double err = F.eps * used + cut + 2.3e-16 * (Bf + ties);
  if (!(err <= F.row_tol * B)) atomicOr(flag, 1u);
}

}  // namespace

double fgt_truncation_bound(int p, double gamma) {
  const double K2 = 1.0865 * 1.0865;
  const double rho = gamma / std::sqrt(2.0);
  double C = 0.0, term = 1.0;  // C(rho) = sum rho^n / sqrt(n!)
  for (int n = 0; n < 200; ++n) {
    C += term;
    term *= rho / std::sqrt(static_cast<double>(n + 1));
  }
  double tail = 1.0;  // rho^p / sqrt(p!)
  for (int n = 1; n <= p; ++n) tail *= rho / std::sqrt(static_cast<double>(n));
  return 2.0 * K2 * C * tail / (1.0 - rho / std::sqrt(p + 1.0));
}

void fgt_truncation_table(double gamma, double target, unsigned short* pn) {
  // term(a, b) = K^2 rho^{a+b} / sqrt(a! b!) = K^2 e_a e_b: the bound of the
  // (a, b) term per unit weight at r = 0 (hk_fgt.cu header).  The kept set
  // {a < a1, b < p} u {a1 <= a < p, b < b2} (b2 = 2 np2, or p) drops
  //   out(p) = the terms with a >= p or b >= p
  //   + (sum_{a1 <= a < p} e_a) (sum_{b2 <= b < p} e_b) K^2,
  // every sum of positive terms taken from suffix sums (no cancellation;
  // beyond kM the terms are below 1e-100).
  constexpr int kM = 160;
  const double K2 = 1.0865 * 1.0865;
  const double rho = gamma / std::sqrt(2.0);
  double e[kM], tail[kM + 1];
  for (int a = 0; a < kM; ++a) e[a] = std::exp(a * std::log(rho) - 0.5 * std::lgamma(a + 1.0));
  tail[kM] = 0.0;
  for (int a = kM - 1; a >= 0; --a) tail[a] = tail[a + 1] + e[a];  // sum_{b >= a}
  const double C = tail[0];
  static_assert(kFgtP < 32 && kFgtP / 2 < 64, "p, a1 and np2 are packed in 5 + 5 + 6 bits");
  for (int k = 0; k < kFgtR2Buckets; ++k) {
    const double allowed = target * std::exp(0.5 * k * kFgtR2Step);  // rows at r^2 >= k step
    int best = 1 << 30;
    unsigned short code = static_cast<unsigned short>(kFgtP | (kFgtP << 5) | ((kFgtP / 2) << 10));  // the full square
    for (int p = 1; p <= kFgtP; ++p) {
      const double out = K2 * (C * tail[p] + (C - tail[p]) * tail[p]);
      if (out > allowed) continue;
      const int np1 = (p + 1) / 2;
      for (int a1 = 0; a1 <= p; ++a1) {
        const double rows = tail[a1] - tail[p];  // sum_{a1 <= a < p} e_a
        for (int np2 = 1; np2 <= np1; ++np2) {
          const int b2 = std::min(2 * np2, p);
          if (out + K2 * rows * (tail[b2] - tail[p]) > allowed) continue;
          const int cost = a1 * np1 + (p - a1) * np2;  // pairs of b
          if (cost < best) {
            best = cost;
            code = static_cast<unsigned short>(p | (a1 << 5) | (np2 << 10));
          }
          break;  // larger np2: more pairs
        }
      }
    }
    pn[k] = code;
  }
}

void launch_fgt_prepare(const FgtParams& F, cudaStream_t s) {
  fgt_refs_kernel<<<(F.nck + 127) / 128, 128, 0, s>>>(F);
  if (F.ncols > 0) fgt_assign_kernel<<<(F.ncols + 255) / 256, 256, 0, s>>>(F);
  cudaFuncSetAttribute(fgt_moments_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMomSmem);
  fgt_moments_kernel<<<F.nck, kMomThreads, kMomSmem, s>>>(F);
  fgt_scan_kernel<<<(F.nbox * PP + 255) / 256, 256, 0, s>>>(F);
  fgt_wsum_kernel<<<(F.nck + 127) / 128, 128, 0, s>>>(F);
}

double bg_fgt_truncation_bound(int p, double gamma) {
  const double K = 1.0865;
  const double rho = gamma / std::sqrt(2.0);
  double tail = 1.0;  // rho^p / sqrt(p!)
  for (int n = 1; n <= p; ++n) tail *= rho / std::sqrt(static_cast<double>(n));
  return K * tail / (1.0 - rho / std::sqrt(p + 1.0));
}

int bg_fgt_parts(int n, int boxes) {
  // about 4096 columns per part, at most 64 parts per box
  return std::max(1, std::min(64, n / (4096 * std::max(1, boxes))));
}

void launch_bg_fgt(const BgFgtParams& F, int rows_base, int rows_total, double* bg_sums, unsigned* flag,
                   cudaStream_t s, double t_first, double t_last, double* part) {
  // only the boxes the rows can reach (bg_fgt_eval_kernel's [b0, b1] for the
  // first and last row; a shard's rows span part of the catalog)
  const double reach = std::sqrt(kFgtCut) / F.inv_sqd + 0.5 * F.L;
  const int b_lo = std::max(0, static_cast<int>(std::floor((t_first - reach - F.t0) / F.L)));
  const int b_hi = std::min(F.nbt - 1, static_cast<int>(std::floor((t_last + reach - F.t0) / F.L)));
  if (b_hi >= b_lo) {
    const int nb = b_hi - b_lo + 1;
    const int S = bg_fgt_parts(F.n, nb);
    bg_fgt_moments_kernel<<<dim3(nb, S), kBgThreads, 0, s>>>(F, b_lo, part);
    bg_fgt_reduce_kernel<<<nb, 32, 0, s>>>(F, b_lo, S, part);
  }
  bg_fgt_eval_kernel<<<(rows_total + kBgThreads - 1) / kBgThreads, kBgThreads, 0, s>>>(F, rows_base, rows_total,
                                                                                     bg_sums, flag);
}

void launch_fgt_eval(const FgtParams& F, int rows_base, int rows_total, const double* bg_sums,
                     double* tr_sums, double coef_a, double coef_c, unsigned* flag, cudaStream_t s) {
  const int rows_per_cta = kFgtRowsPerThread * kFgtEvalThreads;
  const int blocks = F.nck_rows * (kFgtCkRows / rows_per_cta);  // the permutation's positions
  if (F.grad)
    fgt_eval_kernel<true><<<blocks, kFgtEvalThreads, 0, s>>>(F, rows_base, rows_total, bg_sums, tr_sums,
                                                             coef_a, coef_c, flag);
  else
    fgt_eval_kernel<false><<<blocks, kFgtEvalThreads, 0, s>>>(F, rows_base, rows_total, bg_sums, tr_sums,
                                                              coef_a, coef_c, flag);
}

}  // namespace hk
