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
// per unit of box weight (gamma = sqrt 2, p = 30: 6.1e-16).  Boxes whose
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

#include <cmath>
#include <cstdint>

#include "hk_device.cuh"
#include "hk_fgt.cuh"

namespace hk {

namespace {

constexpr int P = kFgtP;
constexpr int PP = kFgtP * kFgtP;

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
  F.u[j] = (x - (F.x0 + (bx + 0.5) * F.L)) * F.inv_sqd;
  F.v[j] = (y - (F.y0 + (by + 0.5) * F.L)) * F.inv_sqd;
}

// ---------------------------------------------------------------------------
// increment moments of checkpoint k: sources [P_{k-1}, P_k), weights relative
// to t_R(k).  One warp per box (boxes strided over the CTA's warps); the
// box's sources are compacted in column order, their power tables u^a/a!,
// v^b/b! staged in shared memory, and each lane sums its coefficients over
// the sources in that order.

constexpr int kMomThreads = 128;
constexpr int kMomWarps = kMomThreads / 32;
constexpr int kMomBatch = 32;  // sources per batch and warp (one 32-column chunk fits)
// dynamic shared memory: per warp kMomBatch x (P + P + 2) doubles
constexpr int kMomSmem = kMomWarps * kMomBatch * (2 * P + 2) * static_cast<int>(sizeof(double));

// adds the batch's sources (in batch order) to the box's coefficients
__device__ __forceinline__ void fgt_flush(double* ob, int sets, int nb, const double* pu, const double* pv,
                                          const double* w, int lane) {
  for (int c = lane; c < sets * PP; c += 32) {
    const int set = c / PP, a = (c % PP) / P, b = c % P;
    double acc = ob[c];
    for (int s = 0; s < nb; ++s) acc = fma(w[2 * s + set] * pu[s * P + a], pv[s * P + b], acc);
    ob[c] = acc;
  }
}

constexpr int kMomBoxesPerCta = 16;  // grid: (checkpoint, group of 16 boxes)

__global__ void __launch_bounds__(kMomThreads) fgt_moments_kernel(const FgtParams F) {
  extern __shared__ __align__(16) double s_dyn[];
  const int k = blockIdx.x;
  const int B_end = min(F.nbox, (static_cast<int>(blockIdx.y) + 1) * kMomBoxesPerCta);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* pu = s_dyn + warp * kMomBatch * (2 * P + 2);
  double* pv = pu + kMomBatch * P;
  double* w = pv + kMomBatch * P;
  const int j0 = k ? F.P[k - 1] : 0, j1 = F.P[k];
  const double tR = F.tR[k];
  const int sets = F.grad ? 2 : 1;
  double* out = F.mom + static_cast<size_t>(k) * F.nbox * 2 * PP;
  for (int B = blockIdx.y * kMomBoxesPerCta + warp; B < B_end; B += kMomWarps) {
    double* ob = out + static_cast<size_t>(B) * 2 * PP;
    for (int c = lane; c < sets * PP; c += 32) ob[c] = 0.0;
    int nb = 0;
    for (int c0 = j0; c0 < j1; c0 += 32) {
      const int j = c0 + lane;
      const bool in = j < j1 && F.box[j] == B;
      const unsigned m = __ballot_sync(0xffffffffu, in);
      const int cnt = __popc(m);
      if (cnt == 0) continue;
      if (nb + cnt > kMomBatch) {
        __syncwarp();
        fgt_flush(ob, sets, nb, pu, pv, w, lane);
        __syncwarp();
        nb = 0;
      }
      if (in) {
        const int s = nb + __popc(m & ((1u << lane) - 1u));
        const double u = F.u[j], v = F.v[j];
        const double wj = exp(-F.omega * (tR - F.t[j]));
        w[2 * s] = wj;
        w[2 * s + 1] = (tR - F.t[j]) * wj;
        double a1 = 1.0, b1 = 1.0;
#pragma unroll 1
        for (int n = 0; n < P; ++n) {
          pu[s * P + n] = a1;
          pv[s * P + n] = b1;
          a1 = a1 * u / (n + 1);
          b1 = b1 * v / (n + 1);
        }
      }
      nb += cnt;
    }
    __syncwarp();
    if (nb) fgt_flush(ob, sets, nb, pu, pv, w, lane);
    __syncwarp();
  }
}

// prefix moments over the checkpoints, in place: M_A[k] = d_k M_A[k-1] +
// inc_A[k], M_B[k] = d_k (M_B[k-1] + dt_k M_A[k-1]) + inc_B[k]
__global__ void fgt_scan_kernel(const FgtParams F) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;  // (box, a, b)
  if (c >= F.nbox * PP) return;
  const int B = c / PP, ab = c % PP;
  double ma = 0.0, mb = 0.0;
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

template <bool kGrad>
__global__ void __launch_bounds__(kFgtEvalThreads, 4)
    fgt_eval_kernel(const FgtParams F, int rows_base, int rows_total, const double* __restrict__ bg_sums,
                    double* __restrict__ tr_sums, double coef_a, double coef_c, unsigned* flag) {
  constexpr int kSets = kGrad ? 2 : 1;
  constexpr unsigned kBoxBytes = kSets * PP * sizeof(double);
  __shared__ __align__(128) double s_m[2][kSets * PP];
  __shared__ __align__(8) uint64_t s_bar[2];
  const int li = blockIdx.x * kFgtEvalThreads + threadIdx.x;
  const int row_block = (blockIdx.x * kFgtEvalThreads) / kFgtRowBlock;
  const int k = row_block / kFgtBlocks;
  const bool valid = li < rows_total;
  const int row = rows_base + (valid ? li : rows_total - 1);
  const double xi = F.x[row], yi = F.y[row], ti = F.t[row];
  const double* mk = F.mom + static_cast<size_t>(k) * F.nbox * 2 * PP;
  if (threadIdx.x == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const bool any = F.P[k] > 0;  // checkpoint with no earlier columns: nothing to add
  double T = 0.0, Td = 0.0, Tq = 0.0, Tq2 = 0.0;
  double w_used = 0.0, w_cut = 0.0;  // box weights (A_00 = sum W) used / skipped with their bound
  const double hs = 0.5 * F.L * F.inv_sqd;  // half box side, scaled
  if (any) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(&s_bar[0], kBoxBytes);
      bulk_g2s(s_m[0], mk, kBoxBytes, &s_bar[0]);
    }
    unsigned phases = 0u;
    for (int B = 0; B < F.nbox; ++B) {
      const int st = B & 1;
      if (B + 1 < F.nbox && threadIdx.x == 0) {
        mbar_expect_tx(&s_bar[st ^ 1], kBoxBytes);
        bulk_g2s(s_m[st ^ 1], mk + static_cast<size_t>(B + 1) * 2 * PP, kBoxBytes, &s_bar[st ^ 1]);
      }
      mbar_wait(&s_bar[st], (phases >> st) & 1u);
      phases ^= 1u << st;
      const double* A = s_m[st];
      const int bx = B % F.nb, by = B / F.nb;
      const double X = (xi - (F.x0 + (bx + 0.5) * F.L)) * F.inv_sqd;
      const double Y = (yi - (F.y0 + (by + 0.5) * F.L)) * F.inv_sqd;
      const double dx = fmax(fabs(X) - hs, 0.0), dy = fmax(fabs(Y) - hs, 0.0);
      const double d2 = fma(dx, dx, dy * dy);
      const bool use = valid && d2 <= kFgtCut;
      const double wB = A[0];  // sum of the box's weights (>= 0)
      if (use) w_used += wB;
      else if (valid) w_cut += wB * exp(-d2);
      if (__any_sync(0xffffffffu, use)) {
        // h_b(Y) for every b (register array, static indices); h_a(X) by the
        // running three-term recurrence inside the a loop (the loop stays
        // rolled: a fully unrolled P x P body overflows the instruction cache)
        double hy[P + 2];
        hermite<kGrad>(Y, hy);
        const double X2 = 2.0 * X;
        double ha = exp(-X * X), ha1 = X2 * ha;
        double ha2 = fma(X2, ha1, -2.0 * ha);
        double t0 = 0.0, q1 = 0.0, q2 = 0.0, b0 = 0.0;
#pragma unroll 2
        for (int a = 0; a < P; ++a) {
          const double* Ar = A + a * P;
          double sA = 0.0, sA2 = 0.0, sB = 0.0;
#pragma unroll
          for (int b = 0; b < P; b += 2) {
            const double2 ab = *reinterpret_cast<const double2*>(Ar + b);
            sA = fma(ab.x, hy[b], sA);
            sA = fma(ab.y, hy[b + 1], sA);
            if (kGrad) {
              sA2 = fma(ab.x, hy[b + 2], sA2);
              sA2 = fma(ab.y, hy[b + 3], sA2);
              const double2 bb = *reinterpret_cast<const double2*>(Ar + PP + b);
              sB = fma(bb.x, hy[b], sB);
              sB = fma(bb.y, hy[b + 1], sB);
            }
          }
          t0 = fma(ha, sA, t0);
          if (kGrad) {
            q1 = fma(ha2, sA, q1);
            q2 = fma(ha, sA2, q2);
            b0 = fma(ha, sB, b0);
          }
          const double ha3 = fma(X2, ha2, -2.0 * (a + 2) * ha1);  // h_{a+3}
          ha = ha1;
          ha1 = ha2;
          ha2 = ha3;
        }
        if (use) {
          T += t0;
          if (kGrad) {
            Td += b0;
            Tq += q1;
            Tq2 += q2;
          }
        }
      }
      __syncthreads();  // every warp is done with this stage before it is refilled
    }
  }
  if (!valid || !any) return;
  const double tR = F.tR[k];
  const double E = exp(-F.omega * (ti - tR));
  double* trT = tr_sums;
  double* trTd = tr_sums + rows_total;
  double* trTq = tr_sums + 2 * static_cast<size_t>(rows_total);
  const double addT = E * T;
  const double Ttot = trT[li] + addT;
  trT[li] = Ttot;
  if (kGrad) {
    trTd[li] += E * fma(ti - tR, T, Td);
    trTq[li] += E * F.delta * fma(0.25, Tq + Tq2, T);
  }
  // certification: the bound on what the expansion may have dropped, against
  // the row's rate S_i = a B_i + c T_i (gradient terms: same weights, the
  // h_{n+2} terms inflate the truncation bound by F.eps_grad / F.eps)
  const double err = coef_c * E * (F.eps * w_used + w_cut);
  const double S = coef_a * bg_sums[li] + coef_c * Ttot;
  if (!(err <= F.row_tol * S)) atomicOr(flag, 1u);
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

// box ranges (binary search of each box's first time) and moments: one CTA
// per box; thread-strided partial sums reduced in a fixed tree order
__global__ void __launch_bounds__(kBgThreads) bg_fgt_moments_kernel(const BgFgtParams F) {
  __shared__ double s_red[kBgThreads];
  __shared__ int s_range[2];
  const int b = blockIdx.x;
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
  const int j0 = s_range[0], j1 = s_range[1];
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
      pw = pw * u / (n + 1);
    }
  }
  for (int n = 0; n < P; ++n) {
    s_red[threadIdx.x] = acc[n];
    __syncthreads();
    for (int h = kBgThreads / 2; h > 0; h >>= 1) {
      if (threadIdx.x < h) s_red[threadIdx.x] += s_red[threadIdx.x + h];
      __syncthreads();
    }
    if (threadIdx.x == 0) F.mom[b * P + n] = s_red[0];
    __syncthreads();
  }
  if (threadIdx.x == 0) F.count[b] = j1 - j0;
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

void launch_fgt_prepare(const FgtParams& F, cudaStream_t s) {
  fgt_refs_kernel<<<(F.nck + 127) / 128, 128, 0, s>>>(F);
  if (F.ncols > 0) fgt_assign_kernel<<<(F.ncols + 255) / 256, 256, 0, s>>>(F);
  cudaFuncSetAttribute(fgt_moments_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMomSmem);
  const dim3 grid(F.nck, (F.nbox + kMomBoxesPerCta - 1) / kMomBoxesPerCta);
  fgt_moments_kernel<<<grid, kMomThreads, kMomSmem, s>>>(F);
  fgt_scan_kernel<<<(F.nbox * PP + 255) / 256, 256, 0, s>>>(F);
}

double bg_fgt_truncation_bound(int p, double gamma) {
  const double K = 1.0865;
  const double rho = gamma / std::sqrt(2.0);
  double tail = 1.0;  // rho^p / sqrt(p!)
  for (int n = 1; n <= p; ++n) tail *= rho / std::sqrt(static_cast<double>(n));
  return K * tail / (1.0 - rho / std::sqrt(p + 1.0));
}

void launch_bg_fgt(const BgFgtParams& F, int rows_base, int rows_total, double* bg_sums, unsigned* flag,
                   cudaStream_t s) {
  bg_fgt_moments_kernel<<<F.nbt, kBgThreads, 0, s>>>(F);
  bg_fgt_eval_kernel<<<(rows_total + kBgThreads - 1) / kBgThreads, kBgThreads, 0, s>>>(F, rows_base, rows_total,
                                                                                     bg_sums, flag);
}

void launch_fgt_eval(const FgtParams& F, int rows_base, int rows_total, const double* bg_sums,
                     double* tr_sums, double coef_a, double coef_c, unsigned* flag, cudaStream_t s) {
  const int blocks = (rows_total + kFgtEvalThreads - 1) / kFgtEvalThreads;
  if (F.grad)
    fgt_eval_kernel<true><<<blocks, kFgtEvalThreads, 0, s>>>(F, rows_base, rows_total, bg_sums, tr_sums,
                                                             coef_a, coef_c, flag);
  else
    fgt_eval_kernel<false><<<blocks, kFgtEvalThreads, 0, s>>>(F, rows_base, rows_total, bg_sums, tr_sums,
                                                              coef_a, coef_c, flag);
}

}  // namespace hk
