// Device-side constants and the FP64 exponential used inside the pair loops.
//
// The reference evaluates every pair term with libm `exp`
// (model.hpp:181 `detail::exp_nonpos`).  There is no FP64 MUFU on B200, so
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
// (table rounding included) 3.5e-14 -- measured 5% faster than 64 entries
// (degree 3, 5.0e-15) despite shared-memory bank conflicts on the 2 KB
// table.  Each entry's high word is stored minus (j << (20 - b)), so the
// power-of-two scale is ONE integer multiply-add on the looked-up entry:
//   hi(2^(j/kTab)) + ((k>>b) << 20) == stored_hi[j] + (k << (20 - b)).
//
// Three argument regimes, chosen per evaluation on the host from bounds on
// the data (hk_host.cpp make_coef), uniform over a launch:
//   kExact   |x*K| < 1020 kTab for every evaluated term: no flush/validity test.
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
#elif HK_TAB_BITS == 8
constexpr double kLog2eT = 369.3299304675746;  // 256 / ln 2
constexpr int kPolyTerms = 3;                   // [3.5e-14]
#define HK_POLY {0.0027076061740622863, 3.6655660167967235e-06, 3.308302907918888e-09}
#else
#error "HK_TAB_BITS must be 4, 5, 6 or 8"
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
#elif HK_TAB_BITS == 6
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
#else
    1.0, 0.9994025125251013, 0.9988087005564014, 0.9982185740592088,
    0.9976321430258502, 0.9970494174757447, 0.9964704074554765, 0.995895123038869,
    0.9953235743270583, 0.9947557714485679, 0.9941917245593819, 0.9936314438430205,
    0.9930749395106142, 0.9925222218009786, 0.9919733009806894, 0.991428187344158,
    0.9908868912137069, 0.9903494229396449, 0.9898157929003436, 0.9892860115023132,
    0.9887600891802786, 0.9882380363972564, 0.987719863644631, 0.9872055814422322,
    0.9866952003384118, 0.9861887309101209, 0.9856861837629878, 0.9851875695313955,
    0.9846928988785599, 0.9842021824966076, 0.9837154311066546, 0.9832326554588848,
    0.9827538663326288, 0.9822790745364429, 0.9818082909081884, 0.981341526315111,
    0.9808787916539204, 0.9804200978508706, 0.9799654558618394, 0.9795148766724088,
    0.9790683712979462, 0.9786259507836846, 0.9781876262048034, 0.97775340866651,
    0.9773233093041209, 0.976897339283144, 0.9764755097993596, 0.9760578320789027,
    0.9756443173783458, 0.9752349769847808, 0.9748298222159021, 0.9744288644200895,
    0.9740321149764913, 0.973639585295108, 0.9732512868168756, 0.9728672310137494,
    0.9724874293887887, 0.9721118934762408, 0.9717406348416251, 0.9713736650818187,
    0.9710109958251406, 0.9706526387314379, 0.9702986054921705, 0.9699489078304969,
    0.9696035575013605, 0.9692625662915756, 0.9689259460199137, 0.9685937085371903,
    0.9682658657263515, 0.9679424295025619, 0.9676234118132908, 0.9673088246384006,
    0.9669986799902345, 0.9666929899137042, 0.9663917664863788, 0.9660950218185728,
    0.965802768053435, 0.9655150173670379, 0.9652317819684667, 0.9649530740999083,
    0.964678906036742, 0.964409290087629, 0.9641442385946024, 0.9638837639331581,
    0.9636278785123455, 0.9633765947748583, 0.9631299251971254, 0.9628878822894031,
    0.9626504785958666, 0.9624177266947014, 0.962189639198196, 0.9619662287528347,
    0.9617475080393891, 0.9615334897730128, 0.9613241867033329, 0.9611196116145447,
    0.9609197773255048, 0.9607246966898253, 0.9605343825959679, 0.9603488479673387,
    0.9601681057623822, 0.9599921689746773, 0.959821050633032, 0.9596547638015788,
    0.9594933215798707, 0.9593367371029772, 0.9591850235415808, 0.9590381941020729,
    0.9588962620266515, 0.9587592405934177, 0.9586271431164729, 0.9584999829460172,
    0.9583777734684463, 0.9582605281064506, 0.9581482603191124, 0.958040983602006,
    0.9579387114872953, 0.9578414575438342, 0.9577492353772651, 0.957662058630119,
    0.957579940981916, 0.9575028961492645, 0.9574309378859631, 0.9573640799831001,
    0.9573023362691556, 0.9572457206101024, 0.9571942469095077, 0.9571479291086353,
    0.9571067811865476, 0.9570708171602076, 0.9570400510845828, 0.9570144970527471,
    0.956994169195985, 0.9569790816838945, 0.9569692487244912, 0.9569646845643128,
    0.9569654034885233, 0.9569714198210175, 0.9569827479245263, 0.9569994022007219,
    0.9570213970903235, 0.9570487470732029, 0.9570814666684909, 0.9571195704346838,
    0.9571630729697497, 0.9572119889112359, 0.9572663329363762, 0.9573261197621985,
    0.9573913641456324, 0.9574620808836177, 0.9575382848132128, 0.9576199908117032,
    0.9577072137967114, 0.9577999687263049, 0.9578982705991074, 0.9580021344544073,
    0.9581115753722692, 0.9582266084736435, 0.958347248920478, 0.9584735119158284,
    0.9586054127039704, 0.9587429665705107, 0.9588861888425, 0.9590350948885443,
    0.9591897001189185, 0.9593500199856788, 0.9595160699827765, 0.9596878656461707,
    0.9598654225539432, 0.9600487563264123, 0.9602378826262469, 0.960432817158582,
    0.9606335756711335, 0.9608401739543135, 0.9610526278413467, 0.9612709532083855,
    0.9614951659746271, 0.9617252821024304, 0.9619613175974319, 0.9622032885086644,
    0.9624512109286739, 0.9627051009936375, 0.9629649748834822, 0.9632308488220032,
    0.9635027390769825, 0.9637806619603089, 0.9640646338280972, 0.9643546710808081,
    0.9646507901633682, 0.9649530075652912, 0.9652613398207983, 0.9655758035089392,
    0.9658964152537145, 0.9662231917241967, 0.9665561496346526, 0.9668953057446663,
    0.9672406768592617, 0.9675922798290256, 0.9679501315502315, 0.968314248964963,
    0.968684649061239, 0.969061348873137, 0.9694443654809188, 0.9698337160111555,
    0.9702294176368531, 0.9706314875775782, 0.9710399430995845, 0.9714548015159391,
    0.9718760801866497, 0.972303796518792, 0.9727379679666364, 0.9731786120317774,
    0.9736257462632606, 0.9740793882577122, 0.9745395556594675, 0.9750062661607005,
    0.9754795375015536, 0.9759593874702676, 0.976445833903312, 0.976938894685516,
    0.9774385877501994, 0.9779449310793042, 0.9784579427035267, 0.9789776407024486,
    0.9795040432046712, 0.9800371683879469, 0.980577034479313, 0.9811236597552254,
    0.9816770625416927, 0.9822372612144102, 0.9828042741988945, 0.9833781199706193,
    0.98395881705515, 0.9845463840282801, 0.9851408395161673, 0.9857422021954696,
    0.9863504907934828, 0.9869657240882777, 0.9875879209088371, 0.9882171001351949,
    0.9888532806985737, 0.9894964815815237, 0.9901467218180625, 0.9908040204938136,
    0.9914683967461472, 0.9921398697643202, 0.9928184587896166, 0.9935041831154892,
    0.9941970620877001, 0.9948971151044637, 0.9956043616165879, 0.9963188211276172,
    0.9970405131939755, 0.9977694574251097, 0.9985056734836332, 0.9992491810854701,
#endif
};

// The per-CTA copy of the table (file-scope static shared: the lookup
// address is an immediate).  Kernels that call exp2_16* must run
// load_exp2_table() and a barrier first.
__shared__ double s_exp2_tab[kTab];

__device__ __forceinline__ void load_exp2_table() {
  for (int i = threadIdx.x; i < kTab; i += blockDim.x) s_exp2_tab[i] = kExp2Tab[i];
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
