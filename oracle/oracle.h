/*
 * oracle.h — CPU ORACLE for the CutMax decoding core.  TEST INFRASTRUCTURE ONLY.
 *
 * This is a deliberately simple, plain-loop C restatement of the reference's
 * algorithm (arXiv 2509.08383 as specified in /root/reference/SPEC.md and
 * PAPER.md).  It is the checker for the CUDA product and the "reference" CPU
 * arm of bench.py; it is never linked into, imported by, or called from the
 * product library (paper_2509_08383_b200/).  Only tests/, __graft_entry__.smoke()
 * and bench.py (cpu_baseline / --impl reference) may load it.
 *
 * PARITY PINNING.  The reference ships no implementation, no tests and no
 * fixtures: only SPEC.md, PAPER.md, an empty CMake project
 * and errors.hpp.  This oracle is therefore pinned to the SPEC's known answers
 * (SPEC.md:67,77,78,79,84-88,97,163-165,173-175,403-404,421-425,433-435 — see
 * tests/golden/spec_known_answers.json and tests/test_oracle_*.py) and to the
 * SPEC invariants, and cross-checked against an
 * independent numpy/math.fsum restatement (tests/golden/make_golden.py).
 * No reference-produced outputs exist to pin against.
 *
 * Numerical pins — identical choices to the product:
 *   A2  population variance, two-pass (mean first, then sum of squared deviations)
 *   A3  poly mode: Newton invsqrt from y0 = 1.5 - x/2, Goldschmidt inverse, AUTO rescale
 *   A4  rescale identity invsqrt(x/b)/sqrt(b)
 *   A5  per-row key seed ^ row driving a Philox4x32-10 per-element stream
 *   A6  portable exp/log (restated here independently of the product header)
 *   A7  argmax of the final iterate Y^(T+1) (= argmax Z, the normaliser being
 *       required positive: sum Y <= 0 is a RangeError), ties -> lowest index;
 *       TieWarning when the input top-2 gap < 1e-9
 *   A9  nucleus: inside(tok) <=> sum_{x_k > x_tok} softmax(x)_k < p
 *   final normalisation uses the state after the T-th update (PAPER.md:69
 *   writes Y^(T); with Y^(1)=X that is read as the last iterate) and is
 *   applied as Z_i = Y_i * inv(sum Y) (Alg. 2 line 8).
 */
#ifndef PAM_ORACLE_H
#define PAM_ORACLE_H

#include <stdint.h>
#include "../include/pam_c_api.h"

#ifdef __cplusplus
extern "C" {
#endif

/* scalar pins */
double orc_ipow(double z, int p);
float  orc_ipowf(float z, int p);
double orc_invsqrt_newton(double x, int iters);
double orc_goldschmidt_inv(double x, int d);
int    orc_invsqrt_cfg(double x, const pam_approx_config* cfg, double* out);
int    orc_inv_cfg(double x, const pam_approx_config* cfg, double* out);
double orc_exp(double x);
double orc_log(double x);
void   orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double orc_uniform(uint64_t seed, uint64_t row, uint64_t draw, uint64_t i);
double orc_log_t(double x);   /* table-driven log / exp of the sampler (pam_scalar.h log_t / exp_t) */
double orc_exp_t(double x);
double orc_beta_icdf(double u, double alpha);
double orc_gumbel(double u);
double orc_nucleus_alpha(double p, double q);

/* core */
int orc_cutmax(const double* x, int64_t n, const pam_cutmax_params* prm,
               double* z, int32_t* argmax, double* stats, int32_t* iters_run);
int orc_cutmax_f32(const float* x, int64_t n, const pam_cutmax_params* prm,
                   float* z, int32_t* argmax, double* stats);
/* batch over rows with OpenMP (nthreads <= 0: all cores); returns the number
 * of rows with non-zero status. */
int64_t orc_cutmax_batch(const double* x, int64_t ld, int64_t B, int64_t n,
                         const pam_cutmax_params* prm, double* z, int64_t ldz,
                         int32_t* argmax, int32_t* status, int nthreads);
int64_t orc_cutmax_batch_f32(const float* x, int64_t ld, int64_t B, int64_t n,
                             const pam_cutmax_params* prm, float* z, int64_t ldz,
                             int32_t* argmax, int32_t* status, int nthreads);
/* cutmaxStep: next_i = (1 + r_i/c)^p, stats {mu, s2, dispersion}
 * and residuals r (nullable).  top = argmax(y) (lowest index). */
int orc_cutmax_step(const double* y, int64_t n, int p, double c, double eps_var,
                    double* next, double* residuals, double* mu, double* s2, double* dispersion);
/* Appendix E closed forms */
int orc_fixed_point_target(int64_t n, int p, double c, double* out /* n */, double* s_star);
int orc_contraction_factor(int64_t n, int p, double c, double* kappa);
/* convergenceTrace: per iteration {mu, s2, dispersion, frac_below_mean} */
int orc_convergence_trace(const double* x, int64_t n, const pam_cutmax_params* prm, double* out /* T x 4 */);
/* cutmaxJvp: forward-mode directional derivative (and Z) */
int orc_cutmax_jvp(const double* x, const double* v, int64_t n, const pam_cutmax_params* prm, double* z, double* dz);

/* TieWarning flag: PAM_ROW_FLAG_TIE if the input top-2 gap < 1e-9, else 0 */
int orc_tie_warning(const double* x, int64_t n);

/* sampling */
int orc_nucleus_inside(const double* x, int64_t n, double p, int64_t tok);
int orc_nucleus_set(const double* x, int64_t n, double p, double* cutoff, int32_t* size, double* mass);
int64_t orc_nucleus_set_batch(const double* x, int64_t ld, int64_t B, int64_t n, double p, double* cutoff,
                              int32_t* size, double* mass, int32_t* status);
int orc_sample(const double* x, int64_t n, const pam_sampler_cfg* cfg, const pam_cutmax_params* prm,
               uint64_t row, int gumbel, int32_t* token, uint8_t* inside, double* onehot);
int64_t orc_sample_batch(const double* x, int64_t ld, int64_t B, int64_t n, const pam_sampler_cfg* cfg,
                         const pam_cutmax_params* prm, int gumbel, int32_t* token, uint8_t* inside,
                         int32_t* status, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
