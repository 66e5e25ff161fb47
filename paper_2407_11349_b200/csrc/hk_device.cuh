// Device-side constants and the FP64 exponential used inside the pair loops.
//
// The reference evaluates every pair term with libm `exp`
// (model.hpp:55 `detail::exp_nonpos`).  There is no FP64 MUFU on B200, so
// exp is a DFMA polynomial and it dominates the FP64 pipe.  This exp works in
// units of ln2/kTab: the caller folds the kTab/ln2 factor into the per-
// evaluation coefficient K, so the range reduction is fused with the
// argument product:
//
//   t  = fma(x, K, MAGIC)       k = round(x*K)      (k in the low word of t)
//   kd = t - MAGIC
//   r  = fma(x, K, -kd)         |r| <= 1/2, one rounding
//   2^((k + r)/kTab) = [2^(k>>b) * TAB[k & (kTab-1)]] * (1 + r*g(r))
//
// g is a Chebyshev fit of (2^(r/kTab)-1)/r on [-1/2, 1/2]
// (tools/exp2_poly.py).  Default kTab = 256 (HK_TAB_BITS = 8): g of degree 2,
// i.e. 3 DFMA for the polynomial, max relative error of the whole evaluation
// (table rounding included) 3.5e-14.  The table lives in dynamic shared
// memory.  Measured alternatives: 64 entries (degree 3, 5.0e-15) 5% slower;
// 4096 entries (degree 1, 5.1e-14, 32 KB) no faster for the homogeneous
// kernel (latency-, not pipe-bound) and it costs the density-scaled kernel
// a resident CTA.  Each entry's high word is stored minus (j << (20 - b)), so the
// power-of-two scale is ONE integer multiply-add on the looked-up entry:
//   hi(2^(j/kTab)) + ((k>>b) << 20) == stored_hi[j] + (k << (20 - b)).
//
// Three argument regimes, chosen per evaluation on the host from bounds on
// the data (hk_host.cpp make_coef), uniform over a launch:
//   kExact   |x*K| < 1020 kTab for every evaluated term: no flush/validity test.
//   kFlush   |x*K| < 2^30: results below 2^-1021 flush to +0 (the reference
//            keeps subnormals; the difference is < 2.3e-308 absolute, far
//            under the 1e-40 rate clip of model.hpp:18).
//   kChecked anything else: also rejects arguments whose k left int32.
#pragma once

#include <cassert>
#include <cstdint>

// Device-side bounds checks of the debug build (make debug: -DHK_DEBUG);
// compiled out otherwise.
#ifdef HK_DEBUG
#define HK_ASSERT(x) assert(x)
#else
#define HK_ASSERT(x) ((void)0)
#endif

namespace hk {

// Kernel shape (overridable at build time for tuning experiments).  Rows
// per thread (measured, tools/tune_shapes.sh, tools/tune_trig.sh): the
// constant kernel amortises each staged column over 4 rows; the varying
// kernel also uses 4 since round 2: with the certified spatial cut its
// candidates are rare and the per-32-column box tests dominate, which 4
// rows amortise over 128-row warp clusters (N=1e6 trigger launch 19.3 ->
// 17.5 ms on the bench catalog, county catalog +1.5%).
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
#define HK_UNROLL 4
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
#ifndef HK_MIN_BLOCKS_TRIG
#define HK_MIN_BLOCKS_TRIG 5  // density-scaled trigger-only launches
#endif
#ifndef HK_MIN_BLOCKS_CONST
#define HK_MIN_BLOCKS_CONST 3
#endif
__host__ __device__ constexpr int min_blocks(int rows) {
  return rows >= 4 ? HK_MIN_BLOCKS_CONST : (rows == 3 ? 2 : 4);
}
constexpr int kBJ = 256;                         // columns per shared-memory tile
constexpr int kUnroll = HK_UNROLL;               // column-loop unroll of the fast tiles

#ifndef HK_TAB_BITS
#define HK_TAB_BITS 8
#endif
constexpr int kTabBits = HK_TAB_BITS;              // table of 2^(j/kTab), j < kTab
constexpr int kTab = 1 << kTabBits;

constexpr double kMagic = 6755399441055744.0;      // 1.5 * 2^52
constexpr double kRateClip = 1e-40;                // model.hpp:18
constexpr double kInvSqrt2Pi = 0.3989422804014327;  // model.hpp:23
constexpr double kInv2Pi = 0.15915494309189535;     // model.hpp:24
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
#elif HK_TAB_BITS == 12
constexpr double kLog2eT = 5909.278887481194;  // 4096 / ln 2
constexpr int kPolyTerms = 2;                   // [5.1e-14]
#define HK_POLY {0.00016922538597985429, 1.431861561720141e-08}
#elif HK_TAB_BITS == 8
constexpr double kLog2eT = 369.3299304675746;  // 256 / ln 2
constexpr int kPolyTerms = 3;                   // [3.5e-14]
#define HK_POLY {0.0027076061740622863, 3.6655660167967235e-06, 3.308302907918888e-09}
#else
#error "HK_TAB_BITS must be 4, 5, 6, 8 or 12"
#endif
__host__ __device__ constexpr double poly_coef(int i) {
  constexpr double c[kPolyTerms] = HK_POLY;
  return c[i];
}

#ifdef __CUDACC__
// 2^(j/kTab) with (j << (20 - kTabBits)) subtracted from the high word,
// generated on the host (hk::make_exp2_table) and uploaded per device
// (hk::upload_exp2_table, hk_kernels.cu).
static __device__ double g_exp2_tab[kTab];

// The per-CTA copy of the table, in dynamic shared memory (kTab * 8 bytes
// per launch of a kernel that calls exp2_16*; such kernels must run
// load_exp2_table() and a barrier first).
extern __shared__ __align__(16) double s_exp2_tab[];

__device__ __forceinline__ void load_exp2_table() {
  for (int i = threadIdx.x; i < kTab; i += blockDim.x) s_exp2_tab[i] = g_exp2_tab[i];
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

// mbarrier + 1-D bulk async copies (TMA engine, SASS UBLKCP): the staging
// of every pair / FGT kernel.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "HK_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra HK_WAIT;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// 1-D bulk async copy global -> shared (TMA engine; SASS UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

#endif  // __CUDACC__

}  // namespace hk
