// Device-side constants and the FP64 exponential used inside the pair loops.
//
// The reference evaluates every pair term with libm `exp`
// (model.hpp:181 `detail::exp_nonpos`).  There is no FP64 MUFU on B200, so
// exp is a DFMA polynomial and it dominates the FP64 pipe.  This exp works in
// units of log2(e)/16: the caller folds the 16/ln2 factor into the per-
// evaluation coefficient K, so the range reduction is fused with the
// argument product:
//
//   t  = fma(x, K, MAGIC)       k = round(x*K)      (k in the low word of t)
//   kd = t - MAGIC
//   r  = fma(x, K, -kd)         |r| <= 1/2, one rounding
//   2^((k + r)/16) = [2^(k>>4) * TAB[k & 15]] * (1 + r*g(r))
//
// g is a degree-4 Chebyshev fit of (2^(r/16)-1)/r on [-1/2, 1/2]
// (tools/exp2_poly.py; max relative error of the whole evaluation, table
// rounding included, 9.3e-15).  The 16-entry table occupies exactly the 32
// shared-memory banks, so the per-lane lookup never bank-conflicts.  Each
// entry's high word is stored minus (j << 16), so the power-of-two scale is
// ONE integer multiply-add on the looked-up entry:
//   hi(2^(j/16)) + ((k>>4) << 20) == stored_hi[j] + (k << 16).
//
// Three argument regimes, chosen per evaluation on the host from bounds on
// the data (hk_host.cpp make_coef), uniform over a launch:
//   kExact   |x*K| < 16320 for every evaluated term: no flush/validity test.
//   kFlush   |x*K| < 2^30: results below 2^-1021 flush to +0 (the reference
//            keeps subnormals; the difference is < 2.3e-308 absolute, far
//            under the 1e-40 rate clip of model.hpp:144).
//   kChecked anything else: also rejects arguments whose k left int32.
#pragma once

#include <cstdint>

namespace hk {

// Kernel shape (overridable at build time for tuning experiments).
#ifndef HK_THREADS
#define HK_THREADS 128
#endif
#ifndef HK_ROWS_PER_THREAD
#define HK_ROWS_PER_THREAD 2
#endif
#ifndef HK_UNROLL
#define HK_UNROLL 2
#endif
#ifndef HK_MIN_BLOCKS
#define HK_MIN_BLOCKS 4
#endif
constexpr int kThreads = HK_THREADS;             // threads per CTA
constexpr int kRowsPerThread = HK_ROWS_PER_THREAD;
constexpr int kBI = kThreads * kRowsPerThread;   // rows per work item (one CTA)
constexpr int kBJ = 256;                         // columns per shared-memory tile
constexpr int kUnroll = HK_UNROLL;               // column-loop unroll of the fast tiles

constexpr double kMagic = 6755399441055744.0;      // 1.5 * 2^52
constexpr double kLog2e16 = 23.083120654223414;    // 16 / ln 2
constexpr double kFlushArg = 16400.0;              // |x*K| beyond which 2^(x*K/16) flushes
constexpr double kExactArg = 16320.0;              // |x*K| below which no term under/overflows
constexpr double kCheckArg = 1073741824.0;         // 2^30
constexpr double kRateClip = 1e-40;                // model.hpp:144
constexpr double kInvSqrt2Pi = 0.3989422804014327;  // model.hpp:149
constexpr double kInv2Pi = 0.15915494309189535;     // model.hpp:150

enum ExpMode { kExact = 0, kFlush = 1, kChecked = 2 };

// g(r) = c1 + c2 r + c3 r^2 + c4 r^3 + c5 r^4
constexpr double kC1 = 0.04332169878499658;
constexpr double kC2 = 0.0009383847926296646;
constexpr double kC3 = 1.3550807778387664e-05;
constexpr double kC4 = 1.4676387238435006e-07;
constexpr double kC5 = 1.2716049516906705e-09;

#ifdef __CUDACC__
// 2^(j/16) with (j << 16) subtracted from the high word.
__device__ __constant__ static const double kExp2Tab16[16] = {
    1.0,
    0.9908868912137069,
    0.9827538663326288,
    0.9756443173783458,
    0.9696035575013605,
    0.964678906036742,
    0.9609197773255048,
    0.9583777734684463,
    0.9571067811865476,
    0.9571630729697497,
    0.9586054127039704,
    0.9614951659746271,
    0.9658964152537145,
    0.9718760801866497,
    0.9795040432046712,
    0.9888532806985737,
};

// The per-CTA copy of the table (file-scope static shared: the lookup
// address is an immediate).  Kernels that call exp2_16* must run
// load_exp2_table() and a barrier first.
__shared__ double s_exp2_tab[16];

__device__ __forceinline__ void load_exp2_table() {
  if (threadIdx.x < 16) s_exp2_tab[threadIdx.x] = kExp2Tab16[threadIdx.x];
}

// Completes 2^((k + r)/16) given t = MAGIC + k and the reduced r.
template <int kMode>
__device__ __forceinline__ double exp2_16_finish(double t, double r) {
  const int k = __double2loint(t);
  const double T = s_exp2_tab[k & 15];
  int hi = __double2hiint(T) + (k << 16);
  int lo = __double2loint(T);
  if (kMode != kExact) {
    bool ok = k >= -16336;  // (k >> 4) > -1022: the scaled entry stays normal
    // For x*K <= 0, t = MAGIC + k has high word 0x43380000 + (k < 0 ? -1 : 0)
    // exactly when -2^32 <= k <= 0; requiring that offset to equal the sign
    // of the low-word k also rejects k < -2^31, where the low word wraps.
    if (kMode == kChecked) ok = ok && (__double2hiint(t) - 0x43380000 == (k >> 31));
    hi = ok ? hi : 0;
    lo = ok ? lo : 0;
  }
  double p = kC5;
  p = fma(p, r, kC4);
  p = fma(p, r, kC3);
  p = fma(p, r, kC2);
  p = fma(p, r, kC1);
  const double y = fma(p, r, 1.0);
  return y * __hiloint2double(hi, lo);
}

// 2^(x*K/16) for x*K <= 0 (x >= 0, K < 0 at every call site).
template <int kMode>
__device__ __forceinline__ double exp2_16(double x, double K) {
  const double t = fma(x, K, kMagic);
  const double kd = t - kMagic;
  const double r = fma(x, K, -kd);
  return exp2_16_finish<kMode>(t, r);
}

// 2^(A/16) for an argument A that is already formed.
template <int kMode>
__device__ __forceinline__ double exp2_16_arg(double A) {
  const double t = A + kMagic;
  const double kd = t - kMagic;
  const double r = A - kd;
  return exp2_16_finish<kMode>(t, r);
}

#endif  // __CUDACC__

}  // namespace hk
