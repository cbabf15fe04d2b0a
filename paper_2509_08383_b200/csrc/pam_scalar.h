// pam_scalar.h — pinned scalar numerics shared by the host C ABI and the
// sm_100a kernels (__host__ __device__), so host-side scalars and device-side
// scalars are bit-identical.  Every expression is written with explicit fma()
// where a fused multiply-add is intended; the library is compiled with
// --fmad=false (device) and -ffp-contract=off (host) so nothing else fuses.
//
// Pins (the reference leaves all of these open):
//   ipow          fixed right-to-left square-and-multiply (SPEC.md:276-284 chain)
//   invsqrt       Newton y <- y*(1.5 - (x/2)*y^2) from y0 = 1.5 - x/2
//                 d iterations after y0 (Table 3)
//   inverse       Goldschmidt prod_{i=0..d} (1 + (1-x)^(2^i))
//   rescale       x/4^k for invsqrt, x/2^k for inv, result * 2^-k     (SPEC.md:205 corrected to /sqrt(b))
//   RNG           Philox4x32-10, key = seed ^ row, counter = (i/2, draw)
//   u in (0,1)    ((bits >> 12) + 0.5) * 2^-52
//   exp / log     portable range-reduced polynomials (not libm), so host and
//                 device agree bit for bit; accuracy ~1 ulp (tests check vs libm)
#ifndef PAM_SCALAR_H
#define PAM_SCALAR_H

#include <stdint.h>
#include <math.h>
#include "pam_logexp_tables.h"
#include <string.h>

#if defined(__CUDACC__)
#define PAM_HD __host__ __device__ __forceinline__
#else
#define PAM_HD static inline
#endif

namespace pam {

// ------------------------------------------------------------------ ipow --
// y = z^p, p >= 1.  Right-to-left binary powering; p = 3 gives z * (z*z).
PAM_HD double ipow(double z, int p) {
  double result = 1.0, base = z;
  bool first = true;
  while (p > 0) {
    if (p & 1) { result = first ? base : result * base; first = false; }
    p >>= 1;
    if (p) base = base * base;
  }
  return result;
}
PAM_HD float ipowf(float z, int p) {
  float result = 1.0f, base = z;
  bool first = true;
  while (p > 0) {
    if (p & 1) { result = first ? base : result * base; first = false; }
    p >>= 1;
    if (p) base = base * base;
  }
  return result;
}

// --------------------------------------------------- Newton invsqrt core --
// Approximates 1/sqrt(x) for x in (0, 2]; x == 1 returns exactly 1.
PAM_HD double invsqrt_newton(double x, int iters) {
  const double h = 0.5 * x;
  double y = 1.5 - h;
  for (int i = 0; i < iters; ++i) {
    const double w = y * y;
    y = y * fma(-h, w, 1.5);
  }
  return y;
}

// ------------------------------------------------- Goldschmidt inverse ---
// f(x) = prod_{i=0}^{d} (1 + (1-x)^(2^i)),  x in (0, 2); x == 1 returns 1.
PAM_HD double goldschmidt_inv_core(double x, int d) {
  double e = 1.0 - x;
  double prod = 1.0 + e;
  for (int i = 1; i <= d; ++i) {
    e = e * e;
    prod = prod * (1.0 + e);
  }
  return prod;
}

// Status values shared with pam_c_api.h (kept numeric here so the header is
// usable without the C API include).
enum : int { S_OK = 0, S_INVALID = 1, S_DEGENERATE = 2, S_RANGE = 3, S_DOMAIN = 4, S_NONFINITE = 5 };
enum : int { RESCALE_AUTO = 0, RESCALE_STATIC = 1, RESCALE_NONE = 2 };

// Rescaled Newton invsqrt.  Returns status; *out = approx 1/sqrt(x).
PAM_HD int invsqrt_rescaled(double x, int iters, int rescale, int scale_log2,
                            double lo, double hi, double* out) {
  if (!(x > 0.0) || !(x <= 1.79e308)) { *out = 0.0; return S_RANGE; }
  if (rescale == RESCALE_AUTO) {
    int e;
    const double m = frexp(x, &e);           // x = m 2^e, m in [0.5, 1)
    (void)m;
    const int k = (e + 1) >> 1;              // ceil(e/2) (arithmetic shift)
    const double xs = ldexp(x, -2 * k);      // in [1/4, 1), exact
    *out = ldexp(invsqrt_newton(xs, iters), -k);
    return S_OK;
  }
  double xs = x;
  int k = 0;
  if (rescale == RESCALE_STATIC) { k = scale_log2 / 2; xs = ldexp(x, -2 * k); }
  if (!(xs >= lo && xs <= hi)) { *out = 0.0; return S_RANGE; }
  *out = ldexp(invsqrt_newton(xs, iters), -k);
  return S_OK;
}

// Rescaled Goldschmidt inverse.  Returns status; *out = approx 1/x.
PAM_HD int inv_rescaled(double x, int iters, int rescale, int scale_log2,
                        double lo, double hi, double* out) {
  if (!(x > 0.0) || !(x <= 1.79e308)) { *out = 0.0; return S_RANGE; }
  if (rescale == RESCALE_AUTO) {
    int e;
    const double m = frexp(x, &e);           // m in [0.5, 1)
    *out = ldexp(goldschmidt_inv_core(m, iters), -e);
    return S_OK;
  }
  double xs = x;
  int k = 0;
  if (rescale == RESCALE_STATIC) { k = scale_log2; xs = ldexp(x, -k); }
  if (!(xs >= lo && xs <= hi) || !(xs > 0.0 && xs < 2.0)) { *out = 0.0; return S_RANGE; }
  *out = ldexp(goldschmidt_inv_core(xs, iters), -k);
  return S_OK;
}

// ------------------------------------------------------------ Philox ------
struct u32x4 { uint32_t x, y, z, w; };

PAM_HD uint32_t mulhi32(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * (uint64_t)b) >> 32);
#endif
}

PAM_HD u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = mulhi32(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = mulhi32(M1, c.z), lo1 = M1 * c.z;
    u32x4 n;
    n.x = hi1 ^ c.y ^ k0;
    n.y = lo1;
    n.z = hi0 ^ c.w ^ k1;
    n.w = lo0;
    c = n;
    k0 += W0;
    k1 += W1;
  }
  return c;
}

// 64 random bits -> double in (0,1), never 0 or 1.
PAM_HD double u01_from_bits(uint32_t lo, uint32_t hi) {
  const uint64_t b = ((uint64_t)hi << 32) | (uint64_t)lo;
  return ((double)(b >> 12) + 0.5) * 0x1p-52;
}

// Uniforms for elements 2j and 2j+1 of (row key, draw).
PAM_HD void uniform_pair(uint64_t key, uint64_t draw, uint64_t j, double* u_even, double* u_odd) {
  u32x4 c;
  c.x = (uint32_t)j; c.y = (uint32_t)(j >> 32);
  c.z = (uint32_t)draw; c.w = (uint32_t)(draw >> 32);
  const u32x4 r = philox4x32_10(c, (uint32_t)key, (uint32_t)(key >> 32));
  *u_even = u01_from_bits(r.x, r.y);
  *u_odd = u01_from_bits(r.z, r.w);
}

PAM_HD double uniform_at(uint64_t seed, uint64_t row, uint64_t draw, uint64_t i) {
  double a, b;
  uniform_pair(seed ^ row, draw, i >> 1, &a, &b);
  return (i & 1) ? b : a;
}

// ------------------------------------------------------- exp / log -------
// Exponent-field helpers: exact replacements for ldexp / frexp on the normal
// range (scaling by 2^k is exact there, so results are bit-identical to the
// library calls the oracle uses); the library calls remain for subnormals.
PAM_HD double pam_bits_to_double(uint64_t b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  double d;
  memcpy(&d, &b, 8);
  return d;
#endif
}
PAM_HD uint64_t pam_double_to_bits(double d) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t b;
  memcpy(&b, &d, 8);
  return b;
#endif
}
// 2^k for -1022 <= k <= 1023
PAM_HD double pam_pow2(int k) { return pam_bits_to_double((uint64_t)(k + 1023) << 52); }

// exp: x = k ln2 + r, |r| <= ln2/2, degree-13 Taylor (Horner, fma).  Results
// below 2^-1022 are flushed to +0 (pinned, keeps both sides identical).
PAM_HD double exp_p(double x) {
  if (x != x) return x;
  if (x > 709.782712893383973096) return HUGE_VAL;
  if (x < -708.3964185322641) return 0.0;
  const double INV_LN2 = 0x1.71547652b82fep+0;
  const double LN2_HI = 0x1.62e42fefa3800p-1;
  const double LN2_LO = 0x1.ef35793c76730p-45;
  const double k = rint(x * INV_LN2);
  double r = fma(-k, LN2_HI, x);
  r = fma(-k, LN2_LO, r);
  double p = 0x1.6124613a86d09p-33;           // 1/13!
  p = fma(p, r, 0x1.1eed8eff8d898p-29);       // 1/12!
  p = fma(p, r, 0x1.ae64567f544e4p-26);       // 1/11!
  p = fma(p, r, 0x1.27e4fb7789f5cp-22);       // 1/10!
  p = fma(p, r, 0x1.71de3a556c734p-19);       // 1/9!
  p = fma(p, r, 0x1.a01a01a01a01ap-16);       // 1/8!
  p = fma(p, r, 0x1.a01a01a01a01ap-13);       // 1/7!
  p = fma(p, r, 0x1.6c16c16c16c17p-10);       // 1/6!
  p = fma(p, r, 0x1.1111111111111p-7);        // 1/5!
  p = fma(p, r, 0x1.5555555555555p-5);        // 1/4!
  p = fma(p, r, 0x1.5555555555555p-3);        // 1/3!
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const int ki = (int)k;
  if (ki < -1021) {                       // result may be subnormal: flush
    const double t = ldexp(p, ki + 60);
    return (t < 0x1p-962) ? 0.0 : ldexp(t, -60);
  }
  if (ki > 1023) return (p * pam_pow2(ki - 1)) * 2.0;  // ki = 1024 (x near the overflow bound)
  return p * pam_pow2(ki);                             // == ldexp(p, ki): exact scaling
}

// log: x = 2^e m, m in [sqrt(1/2), sqrt(2)), f = (m-1)/(m+1),
// log m = 2 atanh f = 2f (1 + f^2/3 + f^4/5 + ... + f^22/23).
PAM_HD double log_p(double x) {
  if (x != x) return x;
  if (x < 0.0) return (double)NAN;
  if (x == 0.0) return -HUGE_VAL;
  if (x > 1.79769313486231570815e308) return x;  // +inf
  int e;
  double m;
  const uint64_t xb = pam_double_to_bits(x);
  if ((xb >> 52) != 0) {  // normal: == frexp(x, &e), m in [1/2, 1)
    e = (int)(xb >> 52) - 1022;
    m = pam_bits_to_double((xb & 0x000fffffffffffffULL) | 0x3fe0000000000000ULL);
  } else {
    m = frexp(x, &e);
  }
  if (m < 0x1.6a09e667f3bcdp-1) { m = m + m; e = e - 1; }
  const double f = (m - 1.0) / (m + 1.0);
  const double s = f * f;
  double q = 0x1.642c8590b2164p-5;            // 1/23
  q = fma(q, s, 0x1.8618618618618p-5);        // 1/21
  q = fma(q, s, 0x1.af286bca1af28p-5);        // 1/19
  q = fma(q, s, 0x1.e1e1e1e1e1e1ep-5);        // 1/17
  q = fma(q, s, 0x1.1111111111111p-4);        // 1/15
  q = fma(q, s, 0x1.3b13b13b13b14p-4);        // 1/13
  q = fma(q, s, 0x1.745d1745d1746p-4);        // 1/11
  q = fma(q, s, 0x1.c71c71c71c71cp-4);        // 1/9
  q = fma(q, s, 0x1.2492492492492p-3);        // 1/7
  q = fma(q, s, 0x1.999999999999ap-3);        // 1/5
  q = fma(q, s, 0x1.5555555555555p-2);        // 1/3
  const double t = f + f;
  const double logm = fma(t * s, q, t);
  const double ed = (double)e;
  const double LN2_HI = 0x1.62e42fefa3800p-1;
  const double LN2_LO = 0x1.ef35793c76730p-45;
  return fma(ed, LN2_HI, fma(ed, LN2_LO, logm));
}

// ------------------------------------------- table-driven log / exp -------
// The sampler evaluates a log and an exp per element for its noise and an exp
// per element for the nucleus test, so those use table-driven forms (~12 fp64
// operations each instead of ~25): tables from tools/gen_logexp_tables.py
// (pam_logexp_tables.h), identical on host and device, mirrored bit for bit
// by the oracle (orc_log_t / orc_exp_t).  Accuracy <= 2 ulp (tests/test_oracle.py).
//
// log_t_core: positive normal x.  x = 2^e m, m in [1, 2); i = top 7 mantissa
// bits; m/2 and e + 1 for i >= 53, so m in [0.707, 1.414); r = m * invc[i] - 1
// (|r| < 2^-7, one rounding), log1p(r) to degree 8; invc = 1 on the two
// intervals next to 1, so results near x = 1 keep their relative accuracy.
PAM_HD double log_t_core(double x, const double* invc, const double* logc) {
  const uint64_t xb = pam_double_to_bits(x);
  const uint64_t mb = xb & 0x000fffffffffffffULL;
  const int i = (int)(mb >> 45);
  const bool half = i >= 53;
  const int e = (int)(xb >> 52) - 1023 + (half ? 1 : 0);
  double m = pam_bits_to_double(mb | 0x3ff0000000000000ULL);
  m = half ? m * 0.5 : m;
  const double r = fma(m, invc[i], -1.0);
  double a = fma(r, -0.125, 0x1.2492492492492p-3);  // -1/8, 1/7
  a = fma(a, r, -0x1.5555555555555p-3);             // -1/6
  a = fma(a, r, 0x1.999999999999ap-3);              // 1/5
  a = fma(a, r, -0.25);
  a = fma(a, r, 0x1.5555555555555p-2);              // 1/3
  a = fma(a, r, -0.5);
  const double lp = fma(r * r, a, r);
  const double t = logc[i] + lp;
  const double ed = (double)e;
  return fma(ed, 0x1.62e42fefa3800p-1, fma(ed, 0x1.ef35793c76730p-45, t));
}
// exp_t_parts: x = (128 q + j) ln2/128 + r (two-step Cody-Waite), |r| <= ln2/256,
// exp(r) - 1 to degree 5; returns 2^(j/128) (1 + (exp(r) - 1)) with one rounding
// and the binary exponent q.
PAM_HD double exp_t_parts(double x, const double* e2, int* q) {
  const double k = rint(x * 0x1.71547652b82fep+7);  // 128 / ln2
  double r = fma(-k, PAM_EXPT_LN2N_HI, x);
  r = fma(-k, PAM_EXPT_LN2N_LO, r);
  double p = fma(r, 0x1.1111111111111p-7, 0x1.5555555555555p-5);  // 1/120, 1/24
  p = fma(p, r, 0x1.5555555555555p-3);                              // 1/6
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  const double em1 = r * p;
  const int ki = (int)k;
  const double t = e2[ki & 127];
  *q = ki >> 7;  // arithmetic shift: floor(ki / 128)
  return fma(t, em1, t);
}
// for -708 <= x <= 709 (q in [-1022, 1023]: no subnormal result, no overflow)
PAM_HD double exp_t_core(double x, const double* e2) {
  int q;
  const double y = exp_t_parts(x, e2, &q);
  return y * pam_pow2(q);
}

#ifdef __CUDACC__
__device__ static const double pam_d_logt_invc[128] = {PAM_LOGT_INVC_VALUES};
__device__ static const double pam_d_logt_logc[128] = {PAM_LOGT_LOGC_VALUES};
__device__ static const double pam_d_expt_e2[128] = {PAM_EXPT_E2_VALUES};
#endif
static const double pam_h_logt_invc[128] = {PAM_LOGT_INVC_VALUES};
static const double pam_h_logt_logc[128] = {PAM_LOGT_LOGC_VALUES};
static const double pam_h_expt_e2[128] = {PAM_EXPT_E2_VALUES};
#ifdef __CUDA_ARCH__
#define PAM_LOGT_INVC pam_d_logt_invc
#define PAM_LOGT_LOGC pam_d_logt_logc
#define PAM_EXPT_E2 pam_d_expt_e2
#else
#define PAM_LOGT_INVC pam_h_logt_invc
#define PAM_LOGT_LOGC pam_h_logt_logc
#define PAM_EXPT_E2 pam_h_expt_e2
#endif

// Portable forms with exp_p / log_p's special cases (NaN, range, zero, inf;
// subnormal log arguments take log_p, which the sampler never produces).
PAM_HD double exp_t(double x) {
  if (x != x) return x;
  if (x > 709.782712893383973096) return HUGE_VAL;
  if (x < -708.3964185322641) return 0.0;
  int q;
  const double y = exp_t_parts(x, PAM_EXPT_E2, &q);
  if (q < -1021) {  // result may be subnormal: flush (as exp_p)
    const double t = ldexp(y, q + 60);
    return (t < 0x1p-962) ? 0.0 : ldexp(t, -60);
  }
  if (q > 1023) return (y * pam_pow2(q - 1)) * 2.0;
  return y * pam_pow2(q);
}
PAM_HD double log_t(double x) {
  if (x != x) return x;
  if (x < 0.0) return (double)NAN;
  if (x == 0.0) return -HUGE_VAL;
  if (x > 1.79769313486231570815e308) return x;  // +inf
  if ((pam_double_to_bits(x) >> 52) == 0) return log_p(x);  // subnormal
  return log_t_core(x, PAM_LOGT_INVC, PAM_LOGT_LOGC);
}

// ------------------------------------------------------- sampling --------
// Beta(alpha,1) inverse CDF u^(1/alpha), given inv_alpha.
PAM_HD double beta_icdf(double u, double inv_alpha) {
  if (!(u > 0.0)) return 0.0;
  if (u >= 1.0) return 1.0;
  if (inv_alpha == 1.0) return u;
  return exp_t(log_t(u) * inv_alpha);
}

// Gumbel from uniform -log(-log u), u in (0,1).
PAM_HD double gumbel_from_u(double u) { return -log_t(-log_t(u)); }

#ifdef __CUDACC__
// ---- branch-free device forms of the above, bit-identical on their domain ----
// The portable functions branch per element on special cases (NaN, 0, inf,
// subnormal, overflow); on the inputs the sampler feeds them none can occur, so
// these run the same arithmetic without branches (and with the tables in
// shared memory).  tools/fastmath_check.cu compares them bit for bit with the
// portable forms.

// Table-driven noise with the tables in shared memory (t = invc[128],
// logc[128], e2[128]; the sampler copies them there once per CTA): the same
// arithmetic as beta_icdf / gumbel_from_u on the sampler's domain, u in
// [2^-53, 1 - 2^-53] and inv_alpha <= 19 (log(u) * inv_alpha >= -700, checked
// once per launch), so bit-identical to them and to the oracle.
__device__ __forceinline__ double beta_icdf_tab(double u, double inv_alpha, const double* t) {
  return inv_alpha == 1.0 ? u : exp_t_core(log_t_core(u, t, t + 128) * inv_alpha, t + 256);
}
__device__ __forceinline__ double gumbel_tab(double u, const double* t) {
  return -log_t_core(-log_t_core(u, t, t + 128), t, t + 128);
}

#endif

}  // namespace pam

#endif  // PAM_SCALAR_H
