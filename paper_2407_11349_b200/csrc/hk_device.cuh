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

// Kernel shape (overridable at build time for tuning experiments).  Rows
// per thread differ by variant (measured, tools/tune_shapes.sh): the
// constant kernel amortises each staged column over 4 rows; the varying
// kernel keeps 2 so its per-row-slot skip votes stay cheap.
#ifndef HK_THREADS
#define HK_THREADS 128
#endif
#ifndef HK_ROWS_CONST
#define HK_ROWS_CONST 4
#endif
#ifndef HK_ROWS_VAR
#define HK_ROWS_VAR 2
#endif
#ifndef HK_UNROLL
#define HK_UNROLL 2
#endif
constexpr int kThreads = HK_THREADS;  // threads per CTA
__host__ __device__ constexpr int rows_per_thread(bool varying) {
  return varying ? HK_ROWS_VAR : HK_ROWS_CONST;
}
// rows per work item (one CTA)
__host__ __device__ constexpr int rows_per_item(bool varying) {
  return kThreads * rows_per_thread(varying);
}
// resident CTAs per SM the register budget is sized for (64K regs)
__host__ __device__ constexpr int min_blocks(int rows) { return rows >= 4 ? 2 : (rows == 3 ? 2 : 4); }
constexpr int kBJ = 256;                         // columns per shared-memory tile
constexpr int kUnroll = HK_UNROLL;               // column-loop unroll of the fast tiles

#ifndef HK_TAB_BITS
#define HK_TAB_BITS 6
#endif
constexpr int kTabBits = HK_TAB_BITS;              // table of 2^(j/kTab), j < kTab
constexpr int kTab = 1 << kTabBits;

constexpr double kMagic = 6755399441055744.0;      // 1.5 * 2^52
constexpr double kRateClip = 1e-40;                // model.hpp:144
constexpr double kInvSqrt2Pi = 0.3989422804014327;  // model.hpp:149
constexpr double kInv2Pi = 0.15915494309189535;     // model.hpp:150
// Argument bounds in units of ln2/kTab: below kExactArg no term can leave
// the normal range (|k >> kTabBits| < 1021); beyond kFlushArg every term
// flushes to 0; below kCheckArg k stays far inside int32.
constexpr double kExactArg = 1020.0 * kTab;
constexpr double kFlushArg = 1025.0 * kTab;
constexpr double kCheckArg = 1073741824.0;         // 2^30

enum ExpMode { kExact = 0, kFlush = 1, kChecked = 2 };

// (2^(r/kTab) - 1)/r on [-1/2, 1/2]: Chebyshev fits from tools/exp2_poly.py;
// max relative error of the whole evaluation incl. table rounding in [].
#if HK_TAB_BITS == 4
constexpr double kLog2eT = 23.083120654223414;  // 16 / ln 2
constexpr int kPolyTerms = 5;                   // [9.3e-15]
#define HK_POLY {0.04332169878499658, 0.0009383847926296646, 1.3550807778387664e-05, \
                 1.4676387238435006e-07, 1.2716049516906705e-09}
#elif HK_TAB_BITS == 5
constexpr double kLog2eT = 46.16624130844683;   // 32 / ln 2
constexpr int kPolyTerms = 4;                   // [1.6e-13]
#define HK_POLY {0.021660849392187844, 0.00023459619820112603, 1.6938609067364198e-06, \
                 9.172598566029335e-09}
#elif HK_TAB_BITS == 6
constexpr double kLog2eT = 92.33248261689366;   // 64 / ln 2
constexpr int kPolyTerms = 4;                   // [5.0e-15]
#define HK_POLY {0.010830424696239445, 5.864904955054418e-05, 2.1173168200092995e-07, \
                 5.732857292414682e-10}
#else
#error "HK_TAB_BITS must be 4, 5 or 6"
#endif
__host__ __device__ constexpr double poly_coef(int i) {
  constexpr double c[kPolyTerms] = HK_POLY;
  return c[i];
}

#ifdef __CUDACC__
// 2^(j/kTab) with (j << (20 - kTabBits)) subtracted from the high word.
__device__ __constant__ static const double kExp2Tab[kTab] = {
#if HK_TAB_BITS == 4
    1.0, 0.9908868912137069, 0.9827538663326288,
    0.9756443173783458, 0.9696035575013605, 0.964678906036742,
    0.9609197773255048, 0.9583777734684463, 0.9571067811865476,
    0.9571630729697497, 0.9586054127039704, 0.9614951659746271,
    0.9658964152537145, 0.9718760801866497, 0.9795040432046712,
    0.9888532806985737,
#elif HK_TAB_BITS == 5
    1.0, 0.9953235743270583, 0.9908868912137069,
    0.9866952003384118, 0.9827538663326288, 0.9790683712979462,
    0.9756443173783458, 0.9724874293887887, 0.9696035575013605,
    0.9669986799902345, 0.964678906036742, 0.9626504785958666,
    0.9609197773255048, 0.9594933215798707, 0.9583777734684463,
    0.957579940981916, 0.9571067811865476, 0.9569654034885233,
    0.9571630729697497, 0.9577072137967114, 0.9586054127039704,
    0.9598654225539432, 0.9614951659746271, 0.9635027390769825,
    0.9658964152537145, 0.968684649061239, 0.9718760801866497,
    0.9754795375015536, 0.9795040432046712, 0.98395881705515,
    0.9888532806985737, 0.9941970620877001,
#else
    1.0, 0.9976321430258502, 0.9953235743270583,
    0.9930749395106142, 0.9908868912137069, 0.9887600891802786,
    0.9866952003384118, 0.9846928988785599, 0.9827538663326288,
    0.9808787916539204, 0.9790683712979462, 0.9773233093041209,
    0.9756443173783458, 0.9740321149764913, 0.9724874293887887,
    0.9710109958251406, 0.9696035575013605, 0.9682658657263515,
    0.9669986799902345, 0.965802768053435, 0.964678906036742,
    0.9636278785123455, 0.9626504785958666, 0.9617475080393891,
    0.9609197773255048, 0.9601681057623822, 0.9594933215798707,
    0.9588962620266515, 0.9583777734684463, 0.9579387114872953,
    0.957579940981916, 0.9573023362691556, 0.9571067811865476,
    0.956994169195985, 0.9569654034885233, 0.9570213970903235,
    0.9571630729697497, 0.9573913641456324, 0.9577072137967114,
    0.9581115753722692, 0.9586054127039704, 0.9591897001189185,
    0.9598654225539432, 0.9606335756711335, 0.9614951659746271,
    0.9624512109286739, 0.9635027390769825, 0.9646507901633682,
    0.9658964152537145, 0.9672406768592617, 0.968684649061239,
    0.9702294176368531, 0.9718760801866497, 0.9736257462632606,
    0.9754795375015536, 0.9774385877501994, 0.9795040432046712,
    0.9816770625416927, 0.98395881705515, 0.9863504907934828,
    0.9888532806985737, 0.9914683967461472, 0.9941970620877001,
    0.9970405131939755,
#endif
};

// The per-CTA copy of the table (file-scope static shared: the lookup
// address is an immediate).  Kernels that call exp2_16* must run
// load_exp2_table() and a barrier first.
__shared__ double s_exp2_tab[kTab];

__device__ __forceinline__ void load_exp2_table() {
  if (threadIdx.x < kTab) s_exp2_tab[threadIdx.x] = kExp2Tab[threadIdx.x];
}

// Polynomial coefficients in the constant bank: DFMA reads them as c[][]
// operands instead of rematerialising 64-bit immediates into registers.
__device__ __constant__ static double c_poly[kPolyTerms] = HK_POLY;  // non-const: not folded

// Table entry k & (kTab-1): one mask + one multiply-add for the address.
__device__ __forceinline__ double exp2_table(int k) {
  unsigned addr;
  asm("{\n"
      ".reg .u32 i;\n"
      "and.b32 i, %1, %2;\n"
      "mad.lo.u32 %0, i, 8, %3;\n"
      "}\n"
      : "=r"(addr)
      : "r"(k), "n"(kTab - 1), "r"(static_cast<unsigned>(__cvta_generic_to_shared(s_exp2_tab))));
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

// Completes 2^((k + r)/kTab) given t = MAGIC + k and the reduced r.
template <int kMode>
__device__ __forceinline__ double exp2_16_finish(double t, double r) {
  const int k = __double2loint(t);
  const double T = exp2_table(k);
  int hi = __double2hiint(T) + (k << (20 - kTabBits));
  int lo = __double2loint(T);
  if (kMode != kExact) {
    bool ok = k >= -1021 * kTab;  // (k >> kTabBits) > -1022: the scaled entry stays normal
    // For x*K <= 0, t = MAGIC + k has high word 0x43380000 + (k < 0 ? -1 : 0)
    // exactly when -2^32 <= k <= 0; requiring that offset to equal the sign
    // of the low-word k also rejects k < -2^31, where the low word wraps.
    if (kMode == kChecked) ok = ok && (__double2hiint(t) - 0x43380000 == (k >> 31));
    hi = ok ? hi : 0;
    lo = ok ? lo : 0;
  }
  double p = c_poly[kPolyTerms - 1];
#pragma unroll
  for (int i = kPolyTerms - 2; i >= 0; --i) p = fma(p, r, c_poly[i]);
  const double y = fma(p, r, 1.0);
  return y * __hiloint2double(hi, lo);
}

// 2^(x*K/kTab) for x*K <= 0 (x >= 0, K < 0 at every call site).
template <int kMode>
__device__ __forceinline__ double exp2_16(double x, double K) {
  const double t = fma(x, K, kMagic);
  const double kd = t - kMagic;
  const double r = fma(x, K, -kd);
  return exp2_16_finish<kMode>(t, r);
}

// 2^(A/kTab) for an argument A that is already formed.
template <int kMode>
__device__ __forceinline__ double exp2_16_arg(double A) {
  const double t = A + kMagic;
  const double kd = t - kMagic;
  const double r = A - kd;
  return exp2_16_finish<kMode>(t, r);
}

#endif  // __CUDACC__

}  // namespace hk
