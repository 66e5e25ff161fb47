/* TEST INFRASTRUCTURE ONLY: a checker, never linked into the product.
 *
 * Double-precision whole-catalog log-likelihood, gradient and conditioning
 * scale (sum_n |d ell_n / d theta_k|) for catalogs too large for the
 * long-double path of hawkes_oracle.c (N = 1e6: tests/golden/full_1m.json).
 * Same formulas as ld_row (hawkes_oracle.c; the reference's likelihood,
 * model.hpp:123-223, plus the gradient of SURVEY.md 8(a)), with the value
 * guards as loop bounds over the sorted times: sources j < count_before(t_i)
 * carry background + trigger (t_j < t_i), j >= upper_bound(t_i) background
 * only, ties nothing (model.hpp:137, :152).  The inner loops are branch
 * free so the compiler vectorises them (libmvec exp, <= 4 ulp); each row sum
 * is accumulated in plain double over blocks of kBlock sources and the
 * block sums are added with Neumaier compensation, so a row sum is good to
 * ~1e-14 relative in the worst case (the parity gate is 1e-10). */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define DBL_CLIP 1e-40 /* kRateClip, model.hpp:18 */
#define DBL_INV_SQRT_2PI 0.39894228040143267794
#define DBL_INV_2PI 0.15915494309189533577

enum { kBlock = 1024 };

typedef struct {
  double s, c;
} nsum;

static void nadd(nsum* a, double v) {
  const double t = a->s + v;
  if (fabs(a->s) >= fabs(v)) a->c += (a->s - t) + v;
  else a->c += (v - t) + a->s;
  a->s = t;
}

static double nval(const nsum* a) { return a->s + a->c; }

typedef struct {
  const double *t, *x, *y, *q;
  size_t n;
  double mu0, tau, xi0, sx, st, area;
  size_t first, stride;
  double* ell; /* [n] */
  double* g;   /* [5n] */
} job;

static size_t lower(const double* t, size_t n, double v) {
  size_t lo = 0, hi = n;
  while (lo < hi) {
    const size_t m = lo + (hi - lo) / 2;
    if (t[m] < v) lo = m + 1;
    else hi = m;
  }
  return lo;
}

static size_t upper(const double* t, size_t n, double v) {
  size_t lo = 0, hi = n;
  while (lo < hi) {
    const size_t m = lo + (hi - lo) / 2;
    if (t[m] <= v) lo = m + 1;
    else hi = m;
  }
  return lo;
}

/* background sums over sources [b, e) */
static void bg_range(const double* t, double ti, double kb, size_t b, size_t e, nsum* B, nsum* B2) {
  for (size_t j0 = b; j0 < e; j0 += kBlock) {
    const size_t j1 = j0 + kBlock < e ? j0 + kBlock : e;
    double sb = 0.0, sb2 = 0.0;
    for (size_t j = j0; j < j1; ++j) {
      const double td = ti - t[j];
      const double b1 = exp(kb * td * td);
      sb += b1;
      sb2 += td * td * b1;
    }
    nadd(B, sb);
    nadd(B2, sb2);
  }
}

static void row(const job* J, size_t i) {
  const double* t = J->t;
  const size_t n = J->n;
  const double tau = J->tau, sx = J->sx, st = J->st, mu0 = J->mu0, xi0 = J->xi0;
  const double omega = 1.0 / st, s2 = 1.0 / (sx * sx);
  const double a = mu0 / (J->area * tau) * DBL_INV_SQRT_2PI;
  const double c = xi0 * omega * s2 * DBL_INV_2PI;
  const double kb = -0.5 / (tau * tau), kq = -0.5 * s2;
  const double ti = t[i], xi = J->x[i], yi = J->y[i];
  const size_t lb = lower(t, n, ti), ub = upper(t, n, ti);
  nsum B = {0, 0}, B2 = {0, 0}, T = {0, 0}, Td = {0, 0}, Tq = {0, 0};
  bg_range(t, ti, kb, 0, lb, &B, &B2);
  bg_range(t, ti, kb, ub, n, &B, &B2);
  for (size_t j0 = 0; j0 < lb; j0 += kBlock) {
    const size_t j1 = j0 + kBlock < lb ? j0 + kBlock : lb;
    double sT = 0.0, sTd = 0.0, sTq = 0.0;
    for (size_t j = j0; j < j1; ++j) {
      const double td = ti - t[j];
      const double dx = xi - J->x[j], dy = yi - J->y[j];
      const double d2 = dx * dx + dy * dy, q = J->q[j];
      const double g = q * exp(-omega * td + kq * q * d2);
      sT += g;
      sTd += td * g;
      sTq += q * d2 * g;
    }
    nadd(&T, sT);
    nadd(&Td, sTd);
    nadd(&Tq, sTq);
  }
  const double Bv = nval(&B), B2v = nval(&B2), Tv = nval(&T), Tdv = nval(&Td), Tqv = nval(&Tq);
  const double S = a * Bv + c * Tv;
  const double lg = log(S > DBL_CLIP ? S : DBL_CLIP);
  const double r = t[n - 1] - ti;
  const double cdf_r = 0.5 * erfc(-(r / tau) * 0.7071067811865475244);
  const double cdf_0 = 0.5 * erfc((ti / tau) * 0.7071067811865475244);
  const double dPhi = cdf_r - cdf_0;
  const double er = exp(-r / st);
  J->ell[i] = lg - (mu0 * dPhi + xi0 * (1.0 - er));
  const double inv = S >= DBL_CLIP ? 1.0 / S : 0.0;
  const double pdf_r = DBL_INV_SQRT_2PI * exp(-0.5 * (r / tau) * (r / tau));
  const double pdf_0 = DBL_INV_SQRT_2PI * exp(-0.5 * (ti / tau) * (ti / tau));
  double* g5 = J->g + 5 * i;
  g5[0] = (a * Bv / mu0) * inv - dPhi;
  g5[1] = (a * (B2v / (tau * tau) - Bv) / tau) * inv + mu0 * (pdf_r * r + pdf_0 * ti) / (tau * tau);
  g5[2] = (c * Tv / xi0) * inv - (1.0 - er);
  g5[3] = (c * (s2 * Tqv - 2.0 * Tv) / sx) * inv;
  g5[4] = -omega * omega * ((c * Tv / omega - c * Tdv) * inv - xi0 * r * er);
}

static void* worker(void* arg) {
  const job* J = (const job*)arg;
  for (size_t i = J->first; i < J->n; i += J->stride) row(J, i);
  return NULL;
}

/* p6 = {mu0, tau_t, xi0, sigma_x, sigma_t, area}; variant 1 = q_j = density. */
int orc_ll_grad_dbl(const double* t, const double* x, const double* y, const double* d, size_t n,
                    const double* p6, int variant, size_t threads, double* ll, double* grad5,
                    double* scale5) {
  for (int k = 0; k < 6; ++k)
    if (!(p6[k] > 0.0) || !isfinite(p6[k])) return 1;
  if (n == 0) return 1;
  double* q = (double*)malloc(n * sizeof(double));
  double* ell = (double*)malloc(n * sizeof(double));
  double* g = (double*)malloc(5 * n * sizeof(double));
  for (size_t i = 0; i < n; ++i) q[i] = variant ? d[i] : 1.0;
  if (threads == 0) threads = 1;
  job* jobs = (job*)calloc(threads, sizeof(job));
  pthread_t* tids = (pthread_t*)calloc(threads, sizeof(pthread_t));
  for (size_t w = 0; w < threads; ++w) {
    job j = {t, x, y, q, n, p6[0], p6[1], p6[2], p6[3], p6[4], p6[5], w, threads, ell, g};
    jobs[w] = j;
    if (w > 0) pthread_create(&tids[w], NULL, worker, &jobs[w]);
  }
  worker(&jobs[0]);
  for (size_t w = 1; w < threads; ++w) pthread_join(tids[w], NULL);
  nsum acc[6];
  double sc[5] = {0, 0, 0, 0, 0};
  memset(acc, 0, sizeof acc);
  for (size_t i = 0; i < n; ++i) {
    nadd(&acc[0], ell[i]);
    for (int k = 0; k < 5; ++k) {
      nadd(&acc[1 + k], g[5 * i + k]);
      sc[k] += fabs(g[5 * i + k]);
    }
  }
  *ll = nval(&acc[0]);
  for (int k = 0; k < 5; ++k) {
    if (grad5) grad5[k] = nval(&acc[1 + k]);
    if (scale5) scale5[k] = sc[k];
  }
  free(tids);
  free(jobs);
  free(q);
  free(ell);
  free(g);
  return 0;
}
