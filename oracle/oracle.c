/*
 * oracle.c — CPU ORACLE (test infrastructure only; see oracle.h header for the
 * pinning statement).  Plain sequential loops, one row at a time, restating
 * SPEC.md / PAPER.md.  Compiled with -ffp-contract=off so every a*b+c below is
 * two roundings unless written as fma().
 */
#include "oracle.h"
#include "../paper_2509_08383_b200/csrc/pam_logexp_tables.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ scalars */

/* z^p by right-to-left square-and-multiply (pin A6; addition-chain order of
 * SPEC.md:279-284). */
double orc_ipow(double z, int p) {
  double acc = 0.0, sq = z;
  int have = 0;
  while (p > 0) {
    if (p & 1) {
      if (have) acc = acc * sq; else { acc = sq; have = 1; }
    }
    p >>= 1;
    if (p) sq = sq * sq;
  }
  return have ? acc : 1.0;
}

float orc_ipowf(float z, int p) {
  float acc = 0.0f, sq = z;
  int have = 0;
  while (p > 0) {
    if (p & 1) {
      if (have) acc = acc * sq; else { acc = sq; have = 1; }
    }
    p >>= 1;
    if (p) sq = sq * sq;
  }
  return have ? acc : 1.0f;
}

/* Newton invsqrt y <- y (1.5 - 0.5 x y^2), y0 = 1.5 - 0.5 x. */
double orc_invsqrt_newton(double x, int iters) {
  double half = 0.5 * x;
  double y = 1.5 - half;
  int i;
  for (i = 0; i < iters; ++i) {
    double y2 = y * y;
    double corr = fma(-half, y2, 1.5);
    y = y * corr;
  }
  return y;
}

/* Goldschmidt inverse f(x) = prod_{i=0}^{d} (1 + (1-x)^(2^i)). */
double orc_goldschmidt_inv(double x, int d) {
  double t = 1.0 - x;
  double f = 1.0 + t;
  int i;
  for (i = 1; i <= d; ++i) {
    t = t * t;
    f = f * (1.0 + t);
  }
  return f;
}

/* Rescaled forms (SPEC.md:205 with the /sqrt(b) correction). */
int orc_invsqrt_cfg(double x, const pam_approx_config* cfg, double* out) {
  *out = 0.0;
  if (!(x > 0.0) || !isfinite(x)) return PAM_ERR_RANGE;
  if (cfg->rescale == PAM_RESCALE_AUTO) {
    int e;
    (void)frexp(x, &e);
    int k = (e + 1) >> 1;
    double xs = ldexp(x, -2 * k);
    *out = ldexp(orc_invsqrt_newton(xs, cfg->iterations), -k);
    return PAM_OK;
  }
  int k = 0;
  double xs = x;
  if (cfg->rescale == PAM_RESCALE_STATIC) { k = cfg->scale_log2 / 2; xs = ldexp(x, -2 * k); }
  if (!(xs >= cfg->lo && xs <= cfg->hi)) return PAM_ERR_RANGE;
  *out = ldexp(orc_invsqrt_newton(xs, cfg->iterations), -k);
  return PAM_OK;
}

int orc_inv_cfg(double x, const pam_approx_config* cfg, double* out) {
  *out = 0.0;
  if (!(x > 0.0) || !isfinite(x)) return PAM_ERR_RANGE;
  if (cfg->rescale == PAM_RESCALE_AUTO) {
    int e;
    double m = frexp(x, &e);
    *out = ldexp(orc_goldschmidt_inv(m, cfg->iterations), -e);
    return PAM_OK;
  }
  int k = 0;
  double xs = x;
  if (cfg->rescale == PAM_RESCALE_STATIC) { k = cfg->scale_log2; xs = ldexp(x, -k); }
  if (!(xs >= cfg->lo && xs <= cfg->hi) || !(xs > 0.0 && xs < 2.0)) return PAM_ERR_RANGE;
  *out = ldexp(orc_goldschmidt_inv(xs, cfg->iterations), -k);
  return PAM_OK;
}

/* Portable exp (pin A6): x = k ln2 + r, Taylor to r^13 by Horner with fma. */
static const double ORC_LN2_HI = 0x1.62e42fefa3800p-1;
static const double ORC_LN2_LO = 0x1.ef35793c76730p-45;

double orc_exp(double x) {
  static const double c[14] = {
      1.0, 1.0, 0.5, 0x1.5555555555555p-3, 0x1.5555555555555p-5, 0x1.1111111111111p-7,
      0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19,
      0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26, 0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33};
  if (isnan(x)) return x;
  if (x > 709.782712893383973096) return INFINITY;
  if (x < -708.3964185322641) return 0.0;
  double k = rint(x * 0x1.71547652b82fep+0);
  double r = fma(-k, ORC_LN2_HI, x);
  r = fma(-k, ORC_LN2_LO, r);
  double poly = c[13];
  int j;
  for (j = 12; j >= 0; --j) poly = fma(poly, r, c[j]);
  int ki = (int)k;
  if (ki < -1021) {
    double t = ldexp(poly, ki + 60);
    return (t < 0x1p-962) ? 0.0 : ldexp(t, -60);
  }
  return ldexp(poly, ki);
}

/* Portable log (pin A6): m in [sqrt(1/2), sqrt(2)), 2 atanh((m-1)/(m+1)). */
double orc_log(double x) {
  static const double inv_odd[12] = {
      1.0, 0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3, 0x1.c71c71c71c71cp-4,
      0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4, 0x1.e1e1e1e1e1e1ep-5,
      0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5};
  if (isnan(x)) return x;
  if (x < 0.0) return NAN;
  if (x == 0.0) return -INFINITY;
  if (isinf(x)) return x;
  int e;
  double m = frexp(x, &e);
  if (m < 0x1.6a09e667f3bcdp-1) { m = m + m; e = e - 1; }
  double f = (m - 1.0) / (m + 1.0);
  double s = f * f;
  double q = inv_odd[11];
  int j;
  for (j = 10; j >= 1; --j) q = fma(q, s, inv_odd[j]);
  double twof = f + f;
  double lm = fma(twof * s, q, twof);
  double ed = (double)e;
  return fma(ed, ORC_LN2_HI, fma(ed, ORC_LN2_LO, lm));
}

/* Philox4x32-10 (Salmon et al. 2011), the named counter-based generator of SPEC.md:466. */
void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  int round;
  for (round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* U_i for element i of row `row`, draw `draw` (Alg. 3 line 3, PAPER.md:229;
 * per-prompt seed ^ index). */
double orc_uniform(uint64_t seed, uint64_t row, uint64_t draw, uint64_t i) {
  uint64_t key64 = seed ^ row;
  uint64_t j = i >> 1;
  uint32_t ctr[4] = {(uint32_t)j, (uint32_t)(j >> 32), (uint32_t)draw, (uint32_t)(draw >> 32)};
  uint32_t key[2] = {(uint32_t)key64, (uint32_t)(key64 >> 32)};
  uint32_t o[4];
  orc_philox(ctr, key, o);
  uint32_t lo = (i & 1) ? o[2] : o[0];
  uint32_t hi = (i & 1) ? o[3] : o[1];
  uint64_t bits = ((uint64_t)hi << 32) | lo;
  return ((double)(bits >> 12) + 0.5) * 0x1p-52;
}

/* Table-driven log / exp of the sampler's noise and nucleus test (the kernel's
 * pam_scalar.h log_t / exp_t, restated operation for operation; tables from
 * tools/gen_logexp_tables.py, 50-digit decimal, correctly rounded).
 * log: x = 2^e m, m in [1,2); i = top 7 mantissa bits; m/2, e+1 for i >= 53;
 * r = m * invc[i] - 1 (one rounding), log1p(r) to degree 8; + logc[i] + e ln2.
 * exp: x = (128 q + j) ln2/128 + r (two-step Cody-Waite), exp(r)-1 to degree 5,
 * 2^(j/128) (1 + (exp(r)-1)) with one rounding, times 2^q. */
static const double orc_logt_invc[128] = {PAM_LOGT_INVC_VALUES};
static const double orc_logt_logc[128] = {PAM_LOGT_LOGC_VALUES};
static const double orc_expt_e2[128] = {PAM_EXPT_E2_VALUES};

static double orc_bits_to_double(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }
static uint64_t orc_double_to_bits(double d) { uint64_t b; memcpy(&b, &d, 8); return b; }

double orc_log_t(double x) {
  if (x != x) return x;
  if (x < 0.0) return NAN;
  if (x == 0.0) return -INFINITY;
  if (x > 1.79769313486231570815e308) return x;
  uint64_t xb = orc_double_to_bits(x);
  if ((xb >> 52) == 0) return orc_log(x);                     /* subnormal */
  uint64_t mb = xb & 0x000fffffffffffffULL;
  int i = (int)(mb >> 45);
  int half = i >= 53;
  int e = (int)(xb >> 52) - 1023 + (half ? 1 : 0);
  double m = orc_bits_to_double(mb | 0x3ff0000000000000ULL);
  if (half) m = m * 0.5;
  double r = fma(m, orc_logt_invc[i], -1.0);
  double a = fma(r, -0.125, 0x1.2492492492492p-3);
  a = fma(a, r, -0x1.5555555555555p-3);
  a = fma(a, r, 0x1.999999999999ap-3);
  a = fma(a, r, -0.25);
  a = fma(a, r, 0x1.5555555555555p-2);
  a = fma(a, r, -0.5);
  double lp = fma(r * r, a, r);
  double t = orc_logt_logc[i] + lp;
  double ed = (double)e;
  return fma(ed, ORC_LN2_HI, fma(ed, ORC_LN2_LO, t));
}

double orc_exp_t(double x) {
  if (x != x) return x;
  if (x > 709.782712893383973096) return INFINITY;
  if (x < -708.3964185322641) return 0.0;
  double k = rint(x * 0x1.71547652b82fep+7);
  double r = fma(-k, PAM_EXPT_LN2N_HI, x);
  r = fma(-k, PAM_EXPT_LN2N_LO, r);
  double p = fma(r, 0x1.1111111111111p-7, 0x1.5555555555555p-5);
  p = fma(p, r, 0x1.5555555555555p-3);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  double em1 = r * p;
  int ki = (int)k;
  double tj = orc_expt_e2[ki & 127];
  double y = fma(tj, em1, tj);
  int q = ki >> 7;
  if (q < -1021) {                       /* result may be subnormal: flush (as orc_exp) */
    double tt = ldexp(y, q + 60);
    return (tt < 0x1p-962) ? 0.0 : ldexp(tt, -60);
  }
  if (q > 1023) return ldexp(y, q - 1) * 2.0;
  return ldexp(y, q);
}

/* betaInverseCdf u^(1/alpha) (Lemma 2 proof PAPER.md:208). */
double orc_beta_icdf(double u, double alpha) {
  double inv_alpha = 1.0 / alpha;
  if (!(u > 0.0)) return 0.0;
  if (u >= 1.0) return 1.0;
  if (inv_alpha == 1.0) return u;
  return orc_exp_t(orc_log_t(u) * inv_alpha);
}

/* gumbelFromUniform -log(-log u) (Definition 1). */
double orc_gumbel(double u) { return -orc_log_t(-orc_log_t(u)); }

/* nucleusAlpha ln(1-q)/ln(p) (Observation 1 PAPER.md:212-215). */
double orc_nucleus_alpha(double p, double q) {
  if (!(p > 0.0 && p < 1.0 && q > 0.0 && q < 1.0)) return NAN;
  return orc_log(1.0 - q) / orc_log(p);
}

/* --------------------------------------------------------------- core ---- */

static int orc_validate(const pam_cutmax_params* prm, int64_t n) {
  int t;
  if (n < 2) return PAM_ERR_INVALID_PARAMS;
  if (prm->T < 1 || prm->T > PAM_MAX_T) return PAM_ERR_INVALID_PARAMS;
  if (!(prm->eps_var >= 0.0)) return PAM_ERR_INVALID_PARAMS;
  for (t = 0; t < prm->T; ++t) {
    int p = prm->p[t];
    double c = prm->c[t];
    if (p < 1 || p > 63) return PAM_ERR_INVALID_PARAMS;
    if (!(prm->flags & PAM_F_UNCHECKED) && (p < 3 || (p % 2) == 0)) return PAM_ERR_INVALID_PARAMS;
    if (!(c > 0.0) || !isfinite(c)) return PAM_ERR_INVALID_PARAMS;
    if ((prm->flags & PAM_F_GUARANTEE) && !(c > sqrt((double)(n - 1)))) return PAM_ERR_INVALID_PARAMS;
    if (prm->invsqrt_mode == PAM_MODE_POLY &&
        (prm->invsqrt[t].iterations < 0 || prm->invsqrt[t].iterations > 64)) return PAM_ERR_INVALID_PARAMS;
  }
  if (prm->inv_mode == PAM_MODE_POLY && (prm->inv.iterations < 0 || prm->inv.iterations > 64))
    return PAM_ERR_INVALID_PARAMS;
  return PAM_OK;
}

/* TieWarning: top-2 gap of the input below 1e-9. */
int orc_tie_warning(const double* x, int64_t n) {
  double m1 = -INFINITY, m2 = -INFINITY;
  int64_t i;
  for (i = 0; i < n; ++i) {
    if (x[i] > m1) { m2 = m1; m1 = x[i]; }
    else if (x[i] > m2) m2 = x[i];
  }
  return (m1 - m2 < 1e-9) ? PAM_ROW_FLAG_TIE : 0;
}

/* cutmax(x, params) -> Z (Alg. 1).  z doubles as
 * the working buffer Y.  stats (nullable) receives {mu_t, s2_t} for t < T. */
int orc_cutmax(const double* x, int64_t n, const pam_cutmax_params* prm,
               double* z, int32_t* argmax, double* stats, int32_t* iters_run) {
  int st = orc_validate(prm, n);
  int64_t i;
  int t;
  if (argmax) *argmax = -1;
  if (st) return st;
  for (i = 0; i < n; ++i)
    if (!isfinite(x[i])) return PAM_ERR_NON_FINITE;            /* LogitVector invariant SPEC.md:33 */
  for (i = 0; i < n; ++i) z[i] = x[i];                          /* Y^(1) = X */
  int ran = 0;
  for (t = 0; t < prm->T; ++t) {
    double sum = 0.0;
    for (i = 0; i < n; ++i) sum += z[i];
    double mu = sum / (double)n;
    double ss = 0.0;
    for (i = 0; i < n; ++i) { double d = z[i] - mu; ss += d * d; }
    double s2 = ss / (double)n;                                 /* PAPER.md:63, population variance */
    if (!isfinite(mu) || !isfinite(s2)) return PAM_ERR_RANGE;
    if (stats) { stats[2 * t] = mu; stats[2 * t + 1] = s2; }
    if (s2 < prm->eps_var) return PAM_ERR_DEGENERATE_INPUT;
    double inv_sigma;
    if (prm->invsqrt_mode == PAM_MODE_POLY) {
      int rs = orc_invsqrt_cfg(s2, &prm->invsqrt[t], &inv_sigma);
      if (rs) return rs;
    } else {
      inv_sigma = 1.0 / sqrt(s2);
    }
    double k = inv_sigma * (1.0 / prm->c[t]);
    int p = prm->p[t];
    for (i = 0; i < n; ++i) {
      double u = (z[i] - mu) * k + 1.0;
      z[i] = orc_ipow(u, p);
    }
    ran = t + 1;
    if (prm->eps_stop > 0.0 && t + 1 < prm->T) {
      double s = 0.0, m = -INFINITY;
      for (i = 0; i < n; ++i) { s += z[i]; if (z[i] > m) m = z[i]; }
      if (m / s >= 1.0 - prm->eps_stop) break;
    }
  }
  if (iters_run) *iters_run = ran;
  /* argmax of the final iterate Y^(T+1) (pin A7): equal to argmax Z for the
   * positive normaliser required below, without the spurious ties the
   * rounding of Y*inv(sum Y) can create.  Lowest index among maxima. */
  int64_t best = 0;
  for (i = 1; i < n; ++i) if (z[i] > z[best]) best = i;
  double total = 0.0;
  for (i = 0; i < n; ++i) total += z[i];
  if (!isfinite(total)) return PAM_ERR_RANGE;
  if (!(prm->flags & PAM_F_NO_NORMALIZE)) {
    double r;
    if (!(total > 0.0)) return PAM_ERR_RANGE;                   /* Z must be a distribution */
    if (prm->inv_mode == PAM_MODE_POLY) {
      int rs = orc_inv_cfg(total, &prm->inv, &r);
      if (rs) return rs;
    } else {
      r = 1.0 / total;
    }
    for (i = 0; i < n; ++i) z[i] = z[i] * r;                    /* PAPER.md:69 / :163 */
  }
  if (argmax) *argmax = (int32_t)best;
  return orc_tie_warning(x, n);                                 /* PAM_OK | TieWarning flag */
}

/* TieWarning on an fp32 input: the top-2 gap of the float values, taken in
 * fp64 (exact: the difference of two floats fits a double). */
static int orc_tie_warning_f32(const float* x, int64_t n) {
  double m1 = -INFINITY, m2 = -INFINITY;
  int64_t i;
  for (i = 0; i < n; ++i) {
    double v = (double)x[i];
    if (v > m1) { m2 = m1; m1 = v; }
    else if (v > m2) m2 = v;
  }
  return (m1 - m2 < 1e-9) ? PAM_ROW_FLAG_TIE : 0;
}

/* fp32 path: fp32 storage and elementwise math, fp64 statistics and scalars. */
int orc_cutmax_f32(const float* x, int64_t n, const pam_cutmax_params* prm,
                   float* z, int32_t* argmax, double* stats) {
  int st = orc_validate(prm, n);
  int64_t i;
  int t;
  if (argmax) *argmax = -1;
  if (st) return st;
  for (i = 0; i < n; ++i)
    if (!isfinite(x[i])) return PAM_ERR_NON_FINITE;
  for (i = 0; i < n; ++i) z[i] = x[i];
  for (t = 0; t < prm->T; ++t) {
    double sum = 0.0;
    for (i = 0; i < n; ++i) sum += (double)z[i];
    double mu = sum / (double)n;
    double ss = 0.0;
    for (i = 0; i < n; ++i) { double d = (double)z[i] - mu; ss += d * d; }
    double s2 = ss / (double)n;
    if (!isfinite(mu) || !isfinite(s2)) return PAM_ERR_RANGE;
    if (stats) { stats[2 * t] = mu; stats[2 * t + 1] = s2; }
    if (s2 < prm->eps_var) return PAM_ERR_DEGENERATE_INPUT;
    double inv_sigma;
    if (prm->invsqrt_mode == PAM_MODE_POLY) {
      int rs = orc_invsqrt_cfg(s2, &prm->invsqrt[t], &inv_sigma);
      if (rs) return rs;
    } else {
      inv_sigma = 1.0 / sqrt(s2);
    }
    double k = inv_sigma * (1.0 / prm->c[t]);
    float muf = (float)mu, kf = (float)k;
    int p = prm->p[t];
    for (i = 0; i < n; ++i) {
      float u = (z[i] - muf) * kf + 1.0f;
      z[i] = orc_ipowf(u, p);
    }
    if (prm->eps_stop > 0.0 && t + 1 < prm->T) {                 /* SPEC.md:126, as the fp64 path */
      double s = 0.0, m = -INFINITY;
      for (i = 0; i < n; ++i) { s += (double)z[i]; if ((double)z[i] > m) m = (double)z[i]; }
      if (m / s >= 1.0 - prm->eps_stop) break;
    }
  }
  int64_t best = 0;
  for (i = 1; i < n; ++i) if (z[i] > z[best]) best = i;        /* argmax of Y^(T+1), pin A7 */
  double total = 0.0;
  for (i = 0; i < n; ++i) total += (double)z[i];
  if (!isfinite(total)) return PAM_ERR_RANGE;
  if (!(prm->flags & PAM_F_NO_NORMALIZE)) {
    double r;
    if (!(total > 0.0)) return PAM_ERR_RANGE;
    if (prm->inv_mode == PAM_MODE_POLY) {
      int rs = orc_inv_cfg(total, &prm->inv, &r);
      if (rs) return rs;
    } else {
      r = 1.0 / total;
    }
    float rf = (float)r;
    for (i = 0; i < n; ++i) z[i] = z[i] * rf;
  }
  if (argmax) *argmax = (int32_t)best;
  return orc_tie_warning_f32(x, n);
}

int64_t orc_cutmax_batch(const double* x, int64_t ld, int64_t B, int64_t n,
                         const pam_cutmax_params* prm, double* z, int64_t ldz,
                         int32_t* argmax, int32_t* status, int nthreads) {
  int64_t bad = 0, r;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(+ : bad)
#endif
  for (r = 0; r < B; ++r) {
    int32_t am = -1;
    int st = orc_cutmax(x + r * ld, n, prm, z + r * ldz, &am, NULL, NULL);
    if (argmax) argmax[r] = am;
    if (status) status[r] = st;
    if (st & 0xff) bad++;                                       /* the TieWarning bit is not a failure */
  }
  (void)nthreads;
  return bad;
}

int64_t orc_cutmax_batch_f32(const float* x, int64_t ld, int64_t B, int64_t n,
                             const pam_cutmax_params* prm, float* z, int64_t ldz,
                             int32_t* argmax, int32_t* status, int nthreads) {
  int64_t bad = 0, r;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(+ : bad)
#endif
  for (r = 0; r < B; ++r) {
    int32_t am = -1;
    int st = orc_cutmax_f32(x + r * ld, n, prm, z + r * ldz, &am, NULL);
    if (argmax) argmax[r] = am;
    if (status) status[r] = st;
    if (st & 0xff) bad++;                                       /* the TieWarning bit is not a failure */
  }
  (void)nthreads;
  return bad;
}

/* cutmaxStep (Appendix E). */
int orc_cutmax_step(const double* y, int64_t n, int p, double c, double eps_var,
                    double* next, double* residuals, double* mu_out, double* s2_out, double* disp_out) {
  int64_t i, top = 0;
  if (n < 2 || p < 1 || !(c > 0.0)) return PAM_ERR_INVALID_PARAMS;
  double sum = 0.0;
  for (i = 0; i < n; ++i) sum += y[i];
  double mu = sum / (double)n;
  double ss = 0.0;
  for (i = 0; i < n; ++i) { double d = y[i] - mu; ss += d * d; }
  double s2 = ss / (double)n;
  if (mu_out) *mu_out = mu;
  if (s2_out) *s2_out = s2;
  if (!(s2 >= eps_var)) return PAM_ERR_DEGENERATE_INPUT;
  double inv_s = 1.0 / sqrt(s2);
  double k = inv_s * (1.0 / c);
  for (i = 1; i < n; ++i) if (y[i] > y[top]) top = i;
  /* dispersion U = sum_{j != top} (r_j - rbar)^2 */
  double rs = 0.0;
  for (i = 0; i < n; ++i) if (i != top) rs += (y[i] - mu) * inv_s;
  double rbar = rs / (double)(n - 1);
  double disp = 0.0;
  for (i = 0; i < n; ++i) {
    double r = (y[i] - mu) * inv_s;
    if (residuals) residuals[i] = r;
    if (i != top) disp += (r - rbar) * (r - rbar);
  }
  if (disp_out) *disp_out = disp;
  if (next)
    for (i = 0; i < n; ++i) next[i] = orc_ipow((y[i] - mu) * k + 1.0, p);
  return PAM_OK;
}

/* fixedPointTarget (eq. fixed-two-level).  Top index 0. */
int orc_fixed_point_target(int64_t n, int p, double c, double* out, double* s_star) {
  int64_t i;
  if (n < 2 || !(c > sqrt((double)(n - 1)))) return PAM_ERR_INVALID_PARAMS;
  double sq = sqrt((double)(n - 1));
  double a = orc_ipow(1.0 + sq / c, p);
  double b = orc_ipow(1.0 - 1.0 / (c * sq), p);
  double s = a / (a + (double)(n - 1) * b);
  if (s_star) *s_star = s;
  if (out) {
    out[0] = s;
    for (i = 1; i < n; ++i) out[i] = (1.0 - s) / (double)(n - 1);
  }
  return PAM_OK;
}

/* contractionFactor kappa (eq. kappa-def). */
int orc_contraction_factor(int64_t n, int p, double c, double* kappa) {
  if (n < 2 || !(c > sqrt((double)(n - 1)))) return PAM_ERR_INVALID_PARAMS;
  double sq = sqrt((double)(n - 1));
  double num = (p / c) * (p / c) * orc_ipow(1.0 + sq / c, 2 * (p - 1));
  double den = (double)n * (double)n * orc_ipow(1.0 - sq / c, 2 * p);
  *kappa = num / den;
  return PAM_OK;
}

/* convergenceTrace: {mu, s2, dispersion, frac below mean} per iteration. */
int orc_convergence_trace(const double* x, int64_t n, const pam_cutmax_params* prm, double* out) {
  int st = orc_validate(prm, n);
  if (st) return st;
  double* y = (double*)malloc(sizeof(double) * (size_t)n);
  double* nx = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t i;
  int t;
  for (i = 0; i < n; ++i) y[i] = x[i];
  for (t = 0; t < prm->T; ++t) {
    double mu, s2, disp;
    st = orc_cutmax_step(y, n, prm->p[t], prm->c[t], prm->eps_var, nx, NULL, &mu, &s2, &disp);
    if (st) break;
    int64_t below = 0;
    for (i = 0; i < n; ++i) if (y[i] < mu) below++;
    out[4 * t + 0] = mu;
    out[4 * t + 1] = s2;
    out[4 * t + 2] = disp;
    out[4 * t + 3] = (double)below / (double)n;
    for (i = 0; i < n; ++i) y[i] = nx[i];
  }
  free(y);
  free(nx);
  return st;
}

/* cutmaxJvp (§3.4): directional derivative of
 * cutmax at x in direction v by forward-mode dual arithmetic through the mean,
 * the population variance, 1/sqrt, the odd power and the normalisation:
 *   mu' = mean(y'),  s2' = 2 mean((y - mu) y'),  k = 1/(c sqrt(s2)),
 *   k' = -k s2' / (2 s2),  u = k (y - mu) + 1,  u' = k' (y - mu) + k (y' - mu'),
 *   y_next = u^p,  y_next' = p u^(p-1) u',
 *   Z = Y / S,  Z' = Y'/S - Y S'/S^2  (S = sum Y, S' = sum Y').
 * s2 < eps_var anywhere on the path is the SingularityError (errors.hpp:55). */
int orc_cutmax_jvp(const double* x, const double* v, int64_t n, const pam_cutmax_params* prm, double* z,
                   double* dz) {
  int st = orc_validate(prm, n);
  if (st) return st;
  if (prm->eps_stop > 0.0) return PAM_ERR_UNSUPPORTED;
  double* y = (double*)malloc(sizeof(double) * (size_t)n);
  double* dy = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t i;
  int t;
  for (i = 0; i < n; ++i) {
    if (!isfinite(x[i]) || !isfinite(v[i])) { free(y); free(dy); return PAM_ERR_NON_FINITE; }
    y[i] = x[i];
    dy[i] = v[i];
  }
  for (t = 0; t < prm->T && st == PAM_OK; ++t) {
    double sum = 0.0, dsum = 0.0;
    for (i = 0; i < n; ++i) { sum += y[i]; dsum += dy[i]; }
    const double mu = sum / (double)n, dmu = dsum / (double)n;
    double ss = 0.0, dss = 0.0;
    for (i = 0; i < n; ++i) {
      const double d = y[i] - mu;
      ss += d * d;
      dss += d * dy[i];
    }
    const double s2 = ss / (double)n, ds2 = 2.0 * dss / (double)n;
    if (!(s2 >= prm->eps_var)) { st = PAM_ERR_SINGULAR; break; }
    const double k = (1.0 / sqrt(s2)) * (1.0 / prm->c[t]);
    const double dk = -k * ds2 / (2.0 * s2);
    const int p = prm->p[t];
    for (i = 0; i < n; ++i) {
      const double d = y[i] - mu;
      const double u = d * k + 1.0;
      const double du = dk * d + k * (dy[i] - dmu);
      y[i] = orc_ipow(u, p);
      dy[i] = (double)p * orc_ipow(u, p - 1) * du;
    }
  }
  if (st == PAM_OK) {
    double S = 0.0, dS = 0.0;
    for (i = 0; i < n; ++i) { S += y[i]; dS += dy[i]; }
    if (!(S > 0.0) || !isfinite(S)) st = PAM_ERR_RANGE;
    else {
      const double r = 1.0 / S;
      for (i = 0; i < n; ++i) {
        if (z) z[i] = y[i] * r;
        dz[i] = dy[i] * r - y[i] * dS * r * r;
      }
    }
  }
  free(y);
  free(dy);
  return st;
}

/* ---------------------------------------------------------- sampling ----- */

/* Nucleus membership ground truth (top-p definition):
 * inside(tok) <=> sum_{k: x_k > x_tok} softmax(x)_k < p  (ties included). */
int orc_nucleus_inside(const double* x, int64_t n, double p, int64_t tok) {
  int64_t i;
  double m = x[0];
  for (i = 1; i < n; ++i) if (x[i] > m) m = x[i];
  double total = 0.0, above = 0.0, xt = x[tok];
  for (i = 0; i < n; ++i) {
    double e = orc_exp_t(x[i] - m);
    total += e;
    if (x[i] > xt) above += e;
  }
  return above < p * total;
}

/* The top-p nucleus itself (softmax probabilities sorted descending,
 * smallest prefix with cumulative mass >= p, ties included), as the
 * set form of orc_nucleus_inside: v is inside <=> mass strictly above v < p.
 * Masses are 40-bit fixed-point integers w_i = floor(exp_t(x_i - m) 2^40 + 1/2)
 * (0 below m - 64), so the sums are exact and order-free and the GPU's histogram
 * scan (csrc/nucleus_set.cu) reproduces this sort-and-walk bit for bit:
 *   inside(v) <=> (double)A(v) < p * (double)W,  A(v) = sum of w over {x > v}.
 * Outputs: cutoff = smallest inside logit, size = entries >= cutoff, mass =
 * their share of W.  Non-finite input: PAM_ERR_NON_FINITE, NaN / 0 / NaN. */
typedef struct { double x; uint64_t q; } orc_nw;
static int orc_nw_desc(const void* a, const void* b) {
  const double xa = ((const orc_nw*)a)->x, xb = ((const orc_nw*)b)->x;
  return xa > xb ? -1 : (xa < xb ? 1 : 0);
}
int orc_nucleus_set(const double* x, int64_t n, double p, double* cutoff, int32_t* size, double* mass) {
  int64_t i;
  *cutoff = NAN; *size = 0; *mass = NAN;
  if (n < 1) return PAM_ERR_BAD_ARGUMENT;
  if (!(p > 0.0 && p < 1.0)) return PAM_ERR_DOMAIN;
  for (i = 0; i < n; ++i) if (!isfinite(x[i])) return PAM_ERR_NON_FINITE;
  double m = x[0];
  for (i = 1; i < n; ++i) if (x[i] > m) m = x[i];
  m = m + 0.0;
  orc_nw* e = (orc_nw*)malloc((size_t)n * sizeof(orc_nw));
  if (!e) return PAM_ERR_BAD_ARGUMENT;
  uint64_t W = 0;
  for (i = 0; i < n; ++i) {
    const double xi = x[i] + 0.0;  /* -0 -> +0, as the kernel's key does */
    const double t = xi - m;
    e[i].x = xi;
    e[i].q = t < -64.0 ? 0 : (uint64_t)(orc_exp_t(t) * 0x1p40 + 0.5);
    W += e[i].q;
  }
  qsort(e, (size_t)n, sizeof(orc_nw), orc_nw_desc);
  const double pW = p * (double)W;
  uint64_t above = 0, mq = 0;
  int64_t cnt = 0;
  i = 0;
  while (i < n) {
    int64_t j = i;
    uint64_t gw = 0;
    while (j < n && e[j].x == e[i].x) { gw += e[j].q; ++j; }
    if (e[i].q == 0 || !((double)above < pW)) break;
    *cutoff = e[i].x;
    cnt += j - i;
    mq = above + gw;
    above += gw;
    i = j;
  }
  *size = (int32_t)cnt;
  *mass = (double)mq / (double)W;
  free(e);
  return PAM_OK;
}
int64_t orc_nucleus_set_batch(const double* x, int64_t ld, int64_t B, int64_t n, double p, double* cutoff,
                              int32_t* size, double* mass, int32_t* status) {
  int64_t r, bad = 0;
  for (r = 0; r < B; ++r) {
    status[r] = orc_nucleus_set(x + r * ld, n, p, &cutoff[r], &size[r], &mass[r]);
    bad += status[r] != PAM_OK;
  }
  return bad;
}

/* nucleusOneShotSample (Alg. 3) and, with
 * gumbel != 0, gumbelMaxSample. */
int orc_sample(const double* x, int64_t n, const pam_sampler_cfg* cfg, const pam_cutmax_params* prm,
               uint64_t row, int gumbel, int32_t* token, uint8_t* inside, double* onehot) {
  int64_t i;
  *token = -1;
  *inside = 0;
  if (!(cfg->p > 0.0 && cfg->p < 1.0)) return PAM_ERR_DOMAIN;
  double alpha = cfg->alpha;
  if (!gumbel && !(alpha > 0.0)) {
    alpha = orc_nucleus_alpha(cfg->p, cfg->q);                  /* Alg. 3 line 1 */
    if (!(alpha > 0.0)) return PAM_ERR_DOMAIN;
  }
  for (i = 0; i < n; ++i)
    if (!isfinite(x[i])) return PAM_ERR_NON_FINITE;
  double* xt = (double*)malloc(sizeof(double) * (size_t)n);
  double* zz = onehot ? onehot : (double*)malloc(sizeof(double) * (size_t)n);
  for (i = 0; i < n; ++i) {
    double u = orc_uniform(cfg->seed, row, cfg->draw, (uint64_t)i);   /* line 3 */
    double g = gumbel ? orc_gumbel(u) : orc_beta_icdf(u, alpha);       /* line 4 */
    xt[i] = x[i] + g;                                                  /* line 5 */
  }
  int32_t am = -1;
  int st = orc_cutmax(xt, n, prm, zz, &am, NULL, NULL);                /* line 6; TieWarning on x~ */
  if ((st & 0xff) == PAM_OK) {
    *token = am;
    *inside = (uint8_t)orc_nucleus_inside(x, n, cfg->p, am);
  }
  free(xt);
  if (!onehot) free(zz);
  return st;
}

int64_t orc_sample_batch(const double* x, int64_t ld, int64_t B, int64_t n, const pam_sampler_cfg* cfg,
                         const pam_cutmax_params* prm, int gumbel, int32_t* token, uint8_t* inside,
                         int32_t* status, int nthreads) {
  int64_t bad = 0, r;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(+ : bad)
#endif
  for (r = 0; r < B; ++r) {
    int st = orc_sample(x + r * ld, n, cfg, prm, (uint64_t)r, gumbel, &token[r], &inside[r], NULL);
    if (status) status[r] = st;
    if (st & 0xff) bad++;                                       /* the TieWarning bit is not a failure */
  }
  (void)nthreads;
  return bad;
}
