/*
 * pam_c_api.h — C ABI of the B200 CutMax decoding core ("pam" = polyargmax).
 *
 * This is the drop-in boundary.  The reference (arXiv 2509.08383, specified in
 * /root/reference/SPEC.md) is a pure C++ host library in namespace `polyargmax`
 * with exception-based errors (proj/include/polyargmax/errors.hpp:9-87).  The
 * C++ API in include/polyargmax/polyargmax.hpp keeps the reference's entry
 * points and sits on top of the plain-C functions declared here; a foreign
 * host (ctypes, cgo, JNI) binds this header directly.
 *
 * Entry points and the reference interface each one replaces:
 *
 *   pam_cutmax_batch_f64 / _f32      core.cutmax            SPEC.md:60-69   (Alg. 1)
 *                                     core.cutmaxStep        SPEC.md:71-79   (T=1, PAM_F_NO_NORMALIZE, stats)
 *   pam_cutmax_batch_host_f64/_f32   core.cutmax on host vectors — H2D, kernel, D2H inside
 *   pam_nucleus_sample_batch_f64     sampling.nucleusOneShotSample SPEC.md:437-445 (Alg. 3)
 *                                     + the nucleus-membership ground truth SPEC.md:440,464
 *   pam_gumbel_sample_batch_f64      sampling.gumbelMaxSample SPEC.md:407-415 (Lemma 1)
 *   pam_goldschmidt_inv              polyapprox.goldschmidtInv
 *   pam_goldschmidt_invsqrt          polyapprox.goldschmidtInvSqrt
 *   pam_nucleus_alpha                sampling.nucleusAlpha
 *   pam_beta_inverse_cdf             sampling.betaInverseCdf
 *   pam_gumbel_from_uniform          sampling.gumbelFromUniform
 *   pam_validate_cutmax_params       CutMaxParams invariants
 *
 * Conventions
 *   - Device-pointer entry points are stream-ordered and asynchronous: they
 *     validate parameters, launch, and return.  Data-dependent failures land in
 *     the per-row status array (int32, one per row, values pam_status).
 *   - The library allocates nothing in the device-pointer hot calls.
 *   - Layout: row-major B x n, leading dimension ld (elements), rows contiguous.
 *   - Status codes mirror the errors.hpp classes (SPEC.md error clauses).
 */
#ifndef PAM_C_API_H
#define PAM_C_API_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PAM_ABI_VERSION 1
#define PAM_MAX_T 16

/* Status codes (call-level return values and per-row status entries).
 * errors.hpp:16 DegenerateInputError, :21 InvalidParamsError, :27 RangeError,
 * :32 DomainError, :77 NonFiniteError. */
typedef enum pam_status {
  PAM_OK = 0,
  PAM_ERR_INVALID_PARAMS = 1,   /* InvalidParamsError */
  PAM_ERR_DEGENERATE_INPUT = 2, /* DegenerateInputError: s^2 < eps_var */
  PAM_ERR_RANGE = 3,            /* RangeError: approx domain / normaliser */
  PAM_ERR_DOMAIN = 4,           /* DomainError */
  PAM_ERR_NON_FINITE = 5,       /* NonFiniteError: non-finite input row */
  PAM_ERR_CUDA = 6,             /* CUDA runtime error (launch / copy) */
  PAM_ERR_BAD_ARGUMENT = 7,     /* null pointer, bad shape or leading dimension */
  PAM_ERR_UNSUPPORTED = 8,      /* a parameter combination this build does not implement */
  PAM_ERR_FORMAT = 9,           /* FormatError          (errors.hpp:65): malformed logit file */
  PAM_ERR_SINGULAR = 10         /* SingularityError     (errors.hpp:55): JVP through s^2 < eps_var */
} pam_status;

/* Row flag bits OR-ed into the per-row status value's high byte (never an error;
 * test errors with (status & 0xff) != PAM_OK).  Set only on PAM_OK rows. */
#define PAM_ROW_FLAG_TIE 0x100      /* TieWarning: input top-2 gap < 1e-9; the
                                       sampler tests x + G, the vector CutMax sees */

/* ApproxConfig.  `rescale` selects how the caller-side
 * rescaling of SPEC.md:205 / PAPER.md:139 is done:
 *   PAM_RESCALE_AUTO   x -> x / 4^k (invsqrt) or x / 2^k (inv), k from the exponent bits,
 *                      so the approximation always runs on [1/4,1) resp. [1/2,1);
 *   PAM_RESCALE_STATIC x -> x / 2^scale_log2 (invsqrt: scale_log2 even, so sqrt(b) is exact),
 *                      then RangeError unless lo <= x/b <= hi;
 *   PAM_RESCALE_NONE   no rescale, RangeError unless lo <= x <= hi.
 * The result is post-multiplied by 1/sqrt(b) (invsqrt) or 1/b (inv): the
 * SPEC/PAPER text "invsqrt(x/b)/b" is corrected to "/sqrt(b)". */
enum { PAM_RESCALE_AUTO = 0, PAM_RESCALE_STATIC = 1, PAM_RESCALE_NONE = 2 };

typedef struct pam_approx_config {
  int32_t iterations;  /* d */
  int32_t alpha_bits;  /* target error exponent; informational */
  int32_t rescale;     /* PAM_RESCALE_* */
  int32_t scale_log2;  /* PAM_RESCALE_STATIC: b = 2^scale_log2 */
  double lo, hi;       /* guaranteed domain after rescaling */
} pam_approx_config;

enum { PAM_MODE_EXACT = 0, PAM_MODE_POLY = 1 };

/* CutMaxParams flags */
#define PAM_F_UNCHECKED    0x1  /* allow even p */
#define PAM_F_GUARANTEE    0x2  /* require every c[t] > sqrt(n-1) */
#define PAM_F_NO_NORMALIZE 0x4  /* return Y^(T+1) un-normalised (cutmaxStep) */

/* CutMaxParams with the decisions of SPEC.md:121-127:
 * per-iteration schedules p[t], c[t] for t < T (scalars are broadcast by the
 * C++/Python front ends), eps_var (default 1e-24), eps_stop (0 = off; > 0 stops
 * after iteration t < T-1 once max Y / sum Y >= 1 - eps_stop, SPEC.md:126 —
 * CutMax f64/f32 and both samplers; the analysis entry points reject it). */
typedef struct pam_cutmax_params {
  int32_t T;
  int32_t flags;
  int32_t invsqrt_mode;           /* PAM_MODE_EXACT: 1/sqrt(s2); PAM_MODE_POLY: Newton invsqrt */
  int32_t inv_mode;               /* PAM_MODE_EXACT: 1/S;        PAM_MODE_POLY: Goldschmidt inverse */
  int32_t p[PAM_MAX_T];
  double c[PAM_MAX_T];
  double eps_var;
  double eps_stop;
  pam_approx_config invsqrt[PAM_MAX_T];
  pam_approx_config inv;
} pam_cutmax_params;

/* SamplerConfig. alpha <= 0 means "derive from (p, q)". */
typedef struct pam_sampler_cfg {
  double p;        /* nucleus mass p in (0,1) */
  double q;        /* tail mass q in (0,1); q = p gives Lemma 2 */
  double alpha;    /* Beta(alpha,1) shape; derived as ln(1-q)/ln(p) when <= 0 */
  uint64_t seed;   /* 64-bit seed; row key = seed ^ row_index */
  uint64_t draw;   /* draw index (Philox counter high word), for repeated draws */
} pam_sampler_cfg;

/* ---- parameter helpers --------------------------------------------------- */
int  pam_abi_version(void);
const char* pam_status_string(int status);
/* Fill defaults: T, p, c broadcast; eps_var=1e-24; exact modes; invsqrt preset
 * alpha_bits=7 (5 Newton iterations), inv d=5, AUTO rescale. */
void pam_default_params(pam_cutmax_params* prm, int32_t T, int32_t p, double c);
/* Validate params for vector length n (InvalidParams / Unsupported). */
int  pam_validate_cutmax_params(const pam_cutmax_params* prm, int64_t n);

/* ---- scalar API (host) --------------------------------------------------- */
int    pam_goldschmidt_inv(double x, const pam_approx_config* cfg, double* out);
int    pam_goldschmidt_invsqrt(double x, const pam_approx_config* cfg, double* out);
int    pam_nucleus_alpha(double p, double q, double* out);
double pam_beta_inverse_cdf(double u, double alpha);
int    pam_gumbel_from_uniform(double u, double* out);
/* Philox4x32-10 uniform in (0,1) for (seed, row, draw, element index). */
double pam_uniform(uint64_t seed, uint64_t row, uint64_t draw, uint64_t index);

/* ---- batched CutMax, device pointers (hot path) -------------------------- */
int pam_cutmax_batch_f64(const double* d_x, int64_t ld_x, int64_t B, int64_t n,
                         const pam_cutmax_params* prm,
                         double* d_z, int64_t ld_z,
                         int32_t* d_argmax,      /* nullable */
                         int32_t* d_row_status,  /* nullable */
                         double* d_stats,        /* nullable: B x T x 2 {mu_t, s2_t} */
                         void* stream);
int pam_cutmax_batch_f32(const float* d_x, int64_t ld_x, int64_t B, int64_t n,
                         const pam_cutmax_params* prm,
                         float* d_z, int64_t ld_z,
                         int32_t* d_argmax, int32_t* d_row_status, double* d_stats,
                         void* stream);

/* ---- batched CutMax, host pointers (end-to-end entry) ---------------------
 * Copies X to the device, runs the kernel and copies Z / argmax / status back,
 * chunked over rows and overlapped over streams.  Synchronous.  Host buffers
 * should be pinned (cudaHostAlloc) for full PCIe bandwidth. */
int pam_cutmax_batch_host_f64(const double* h_x, int64_t B, int64_t n,
                              const pam_cutmax_params* prm,
                              double* h_z, int32_t* h_argmax, int32_t* h_row_status);
int pam_cutmax_batch_host_f32(const float* h_x, int64_t B, int64_t n,
                              const pam_cutmax_params* prm,
                              float* h_z, int32_t* h_argmax, int32_t* h_row_status);

/* ---- fused Beta-cut nucleus sampler (Alg. 3) + nucleus membership ---------
 * token[r]  = argmax(cutmax(x_r + G_r)), G_ri = u_ri^(1/alpha)
 * inside[r] = 1 iff token is in the top-p nucleus of softmax(x_r) (ties included):
 *             sum_{k: x_k > x_tok} softmax(x)_k < p
 * d_onehot (nullable) receives the CutMax output of the perturbed logits. */
int pam_nucleus_sample_batch_f64(const double* d_x, int64_t ld_x, int64_t B, int64_t n,
                                 const pam_sampler_cfg* cfg, const pam_cutmax_params* prm,
                                 int32_t* d_token, uint8_t* d_inside,
                                 double* d_onehot, int64_t ld_onehot,
                                 int32_t* d_row_status, void* stream);
/* Gumbel-max variant (G = -log(-log u)); inside[] uses nucleus mass cfg->p. */
int pam_gumbel_sample_batch_f64(const double* d_x, int64_t ld_x, int64_t B, int64_t n,
                                const pam_sampler_cfg* cfg, const pam_cutmax_params* prm,
                                int32_t* d_token, uint8_t* d_inside,
                                double* d_onehot, int64_t ld_onehot,
                                int32_t* d_row_status, void* stream);

/* ---- the top-p nucleus itself (csrc/nucleus_set.cu) ---
 * Per row: cutoff[r] = the smallest logit inside the top-p nucleus of
 * softmax(x_r) (ties included), size[r] = number of entries >= cutoff, mass[r] =
 * their softmax mass; x_k is inside <=> x_k >= cutoff[r].  The cumulative-mass
 * step is a cluster-wide histogram scan (radix select) over 40-bit fixed-point
 * masses floor(exp(x - max) 2^40 + 1/2), which makes the result independent of
 * the summation order (bit-exact against the oracle).  n <= 180224.  Outputs
 * are nullable.  Replaces the nucleus ground truth of sampling.violationExperiment
 * (SPEC.md:447-455, 464).  Row status: PAM_OK or PAM_ERR_NON_FINITE. */
int pam_nucleus_set_batch_f64(const double* d_x, int64_t ld_x, int64_t B, int64_t n, double p,
                              double* d_cutoff, int32_t* d_size, double* d_mass,
                              int32_t* d_row_status, void* stream);

/* ---- analysis outputs (csrc/analysis_kernel.cuh) -------------------
 * convergenceTrace: d_out[B][T][4] = {mu, s2, U, fraction of
 * entries below the mean} per iteration, U = sum_{j != top} (r_j - rbar)^2 the
 * non-top dispersion.  Entries after a failing iteration are
 * not written; the row status says why.  Replaces core::convergenceTrace. */
int pam_convergence_trace_batch_f64(const double* d_x, int64_t ld_x, int64_t B, int64_t n,
                                    const pam_cutmax_params* prm, double* d_out, int32_t* d_row_status,
                                    void* stream);
/* cutmaxJvp: d_dz = d cutmax(x; params) / dx . v, forward mode
 * through mean, variance, 1/sqrt, odd power and normalisation; d_z (nullable) =
 * cutmax(x).  x and v share ld_x.  s2 < eps_var -> PAM_ERR_SINGULAR per row.
 * Replaces grad::cutmaxJvp (cutmaxJacobian = n JVPs, one batched call). */
int pam_cutmax_jvp_batch_f64(const double* d_x, const double* d_v, int64_t ld_x, int64_t B, int64_t n,
                             const pam_cutmax_params* prm, double* d_z, double* d_dz, int64_t ld_z,
                             int32_t* d_row_status, void* stream);

/* ---- logit files (csrc/ingest.cpp) -------------------------
 * LGT1:  "LGT1" | u16 version (1) | u32 count | u32 n | count*n little-endian float32.
 * JSONL: one JSON array of numbers per line, all of one length.
 * Readers fill a caller buffer (pinned host memory feeds the batch API with one
 * copy).  PAM_ERR_FORMAT sets info->err_offset (byte offset); PAM_ERR_NON_FINITE
 * sets info->bad_vector (first vector with NaN/Inf; the data is still written).
 * Replaces cli::ingest and the LogitFile writer. */
typedef struct pam_ingest_info {
  int64_t count, n;    /* vectors, length */
  int64_t err_offset;  /* PAM_ERR_FORMAT: byte offset of the problem, else -1 */
  int64_t bad_vector;  /* PAM_ERR_NON_FINITE: first non-finite vector, else -1 */
} pam_ingest_info;
int pam_lgt1_probe(const char* path, pam_ingest_info* info);
int pam_lgt1_read(const char* path, float* dst, int64_t capacity, pam_ingest_info* info);
int pam_lgt1_write(const char* path, const float* src, int64_t count, int64_t n);
int pam_jsonl_probe(const char* path, pam_ingest_info* info);
int pam_jsonl_read(const char* path, double* dst, int64_t capacity, pam_ingest_info* info);

/* ---- introspection (bench / tests) --------------------------------------- */
typedef struct pam_launch_info {
  int32_t threads, elems_per_thread, cluster, clusters, ctas, smem_bytes, tma, kernel_id, groups;
} pam_launch_info;
/* Launch geometry the library would use for (dtype_bytes, B, n). */
int pam_query_launch(int dtype_bytes, int64_t B, int64_t n, const pam_cutmax_params* prm,
                     pam_launch_info* info);
/* Number of kernels this library launched since load (tests / bench evidence). */
int64_t pam_kernel_launch_count(void);
/* Tuning / test hooks (explicit calls; the library reads no environment variables).
 * pam_set_geometry_override: force the CutMax geometry for one dtype (threads x
 *   elems_per_thread per CTA from the compiled variant table, cluster size 1..16,
 *   launch-bounds min_blocks); threads = 0 clears it.  PAM_ERR_UNSUPPORTED if no
 *   such variant is compiled.  A forced geometry that cannot hold a row makes the
 *   batch call return PAM_ERR_UNSUPPORTED.
 * pam_set_host_chunk_bytes: pipeline chunk of the host-pointer entry points
 *   (default 128 MiB of input per chunk; <= 0 restores the default).
 * pam_set_lean_p3: 1 (default) runs p = 3, T >= 2, aligned fp64 rows on the lean
 *   kernel (cutmax_p3_kernel.cuh); 0 runs them on the general kernel (A/B tests:
 *   both give bit-identical results). */
int pam_set_geometry_override(int dtype_bytes, int threads, int elems_per_thread, int cluster, int min_blocks);
int pam_set_host_chunk_bytes(int64_t bytes);
int pam_set_lean_p3(int on);
/* Debug: device buffer (grid x 8 rows x 32 events of int64 clock64 stamps) that
 * the CutMax kernel fills with per-CTA phase timestamps; NULL disables. */
void pam_set_trace_buffer(long long* d_buf, int64_t entries);
/* Last CUDA error string seen by the library (thread-unsafe diagnostic). */
const char* pam_last_cuda_error(void);

#ifdef __cplusplus
}
#endif
#endif /* PAM_C_API_H */
