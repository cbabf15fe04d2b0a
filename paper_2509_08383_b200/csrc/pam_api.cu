// pam_api.cu — the C ABI (include/pam_c_api.h): parameter validation, launch
// geometry selection, kernel launches, the host-buffer end-to-end path and the
// host scalar API.  No CPU compute path exists for the batched entry points:
// if a kernel cannot be launched the call fails with PAM_ERR_CUDA.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/pam_c_api.h"
#include "analysis_kernel.cuh"
#include "cutmax_ahead_kernel.cuh"
#include "cutmax_kernel.cuh"
#include "nucleus_kernel.cuh"
#include "pam_variants.h"
#include "pam_scalar.h"

using namespace pam;

namespace {

std::atomic<int64_t> g_launches{0};
long long* g_trace = nullptr;  // debug phase-trace buffer (pam_set_trace_buffer)
int64_t g_trace_entries = 0;
thread_local char g_last_err[256] = "";

int cuda_fail(cudaError_t e, const char* what) {
  snprintf(g_last_err, sizeof g_last_err, "%s: %s", what, cudaGetErrorString(e));
  return PAM_ERR_CUDA;
}

// Kernel tables: pam_variants.h (defined in cutmax_variants.cu / sampler_variants.cu).

struct Geometry {
  const Variant* var = nullptr;
  int C = 0;
  int L = 0;
};

// Dev override: PAM_FORCE_CFG_F64 / PAM_FORCE_CFG_F32 = "NTG,E,C[,MINB]".
bool parse_force(int elem_bytes, int* ntg, int* e, int* c, int* minb) {
  const char* s = getenv(elem_bytes == 8 ? "PAM_FORCE_CFG_F64" : "PAM_FORCE_CFG_F32");
  if (!s || !*s) return false;
  *minb = 0;
  return sscanf(s, "%d,%d,%d,%d", ntg, e, c, minb) >= 3;
}

int buffer_bytes(const Variant& v) { return ((v.ntg * v.e * v.elem_bytes + 127) / 128) * 128; }
int smem_bytes(const Variant& v) { return buffer_bytes(v) + (int)sizeof(ControlBlock); }

int64_t slice_len(int64_t n, int C, int vec) { return ((n + C - 1) / C + vec - 1) / vec * vec; }

int max_active_clusters(const void* fn, int nt, int C, int smem);

// Launch geometry.  Candidates are every (variant, cluster size C = 1..16)
// whose per-CTA capacity covers the slice ceil(n/C) with < 30% phantom waste.
// They are ranked by rows per microsecond, clusters / t_row, with the row
// period fitted to B200 measurements (tools/tune.py, tools/trace.py):
//   t_row ~= a + b * cap * k
// a = latency per row (T exchanges + scalar chains: fp64 4.8 us, fp32 2.5 us),
// b = element cost per CTA-slot (fp64 0.33 ns, fp32 0.35 ns), cap = NTG*E, and
// k = CTAs sharing an SM (clusters*C / #SMs, rounded up) from the occupancy
// query.  Non power-of-two clusters matter: 9-CTA clusters pack 135 SMs vs 120
// for 8.
Geometry choose_geometry(int elem_bytes, int64_t B, int64_t n) {
  Geometry g;
  const int vec = 16 / elem_bytes;
  int fntg, fe, fc, fmb;
  if (parse_force(elem_bytes, &fntg, &fe, &fc, &fmb)) {
    for (int i = 0; i < kNumCutmaxVariants; ++i) {
      const Variant& v = kCutmaxVariants[i];
      if (v.elem_bytes == elem_bytes && v.ntg == fntg && v.e == fe && v.minb == fmb) {
        const int64_t L = slice_len(n, fc, vec);
        if ((int64_t)v.ntg * v.e >= L) { g.var = &v; g.C = fc; g.L = (int)L; return g; }
      }
    }
  }
  int dev = 0;
  const bool have_gpu = cudaGetDevice(&dev) == cudaSuccess;
  int nsm = 148;
  if (have_gpu && cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) nsm = 148;
  const double a_us = elem_bytes == 8 ? 4.8 : 2.5, b_ns = elem_bytes == 8 ? 0.33 : 0.35;
  double best_score = -1.0;
  for (int C = 1; C <= 16; ++C) {
    const int64_t L = slice_len(n, C, vec);
    for (int i = 0; i < kNumCutmaxVariants; ++i) {
      const Variant& v = kCutmaxVariants[i];
      if (v.elem_bytes != elem_bytes) continue;
      const int64_t cap = (int64_t)v.ntg * v.e;
      if (cap < L || (C > 1 && cap > L + L * 3 / 10)) continue;
      if (C > 1 && L < 2048) continue;  // tiny slices: exchanges would dominate
      const int smem = smem_bytes(v);
      if (smem > 227 * 1024) continue;
      const int active = have_gpu ? max_active_clusters(v.fn[1], v.ntg, C, smem) : nsm / C;
      if (active <= 0) continue;
      const int64_t clusters = (B < active) ? B : active;
      const int64_t k = (clusters * C + nsm - 1) / nsm;
      const double t_us = a_us + 1e-3 * b_ns * (double)cap * (double)(k < 1 ? 1 : k);
      const double score = (double)clusters / t_us - 1e-9 * (double)C;  // tie-break: smaller clusters
      if (score > best_score) { best_score = score; g.var = &v; g.C = C; g.L = (int)L; }
    }
  }
  cudaGetLastError();
  return g;
}

struct OccKey {
  const void* fn;
  int C, smem;
};
std::mutex g_occ_mu;
std::vector<std::pair<OccKey, int>> g_occ_cache;

std::vector<std::pair<const void*, int>> g_smem_attr;  // per kernel: largest dynamic smem opted in

// Raise the kernel's dynamic-smem opt-in to at least `smem` (never lower it:
// an earlier, larger cached configuration must stay launchable).
void ensure_smem_attr(const void* fn, int smem, int C) {
  std::lock_guard<std::mutex> lk(g_occ_mu);
  for (auto& kv : g_smem_attr)
    if (kv.first == fn) {
      if (kv.second >= smem) return;
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kv.second = smem;
      return;
    }
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  g_smem_attr.push_back({fn, smem});
  (void)C;
}

int max_active_clusters(const void* fn, int nt, int C, int smem) {
  ensure_smem_attr(fn, smem, C);
  {
    std::lock_guard<std::mutex> lk(g_occ_mu);
    for (auto& kv : g_occ_cache)
      if (kv.first.fn == fn && kv.first.C == C && kv.first.smem == smem) return kv.second;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3(C * 16);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    ncl = 0;
  }
  std::lock_guard<std::mutex> lk(g_occ_mu);
  g_occ_cache.push_back({OccKey{fn, C, smem}, ncl});
  return ncl;
}

int launch_cluster_kernel(const void* fn, int nt, int C, int clusters, int smem, cudaStream_t stream, void* kargs) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3((unsigned)(clusters * C));
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {kargs};
  cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernelExC");
  g_launches.fetch_add(1);
  return PAM_OK;
}

int binom2(int p) { return p * (p - 1) / 2; }

int fill_row_params(const pam_cutmax_params* prm, RowParams* rp) {
  memset(rp, 0, sizeof *rp);
  rp->T = prm->T;
  rp->flags = prm->flags;
  rp->invsqrt_mode = prm->invsqrt_mode;
  rp->inv_mode = prm->inv_mode;
  rp->eps_var = prm->eps_var;
  for (int t = 0; t < prm->T; ++t) {
    rp->p[t] = prm->p[t];
    rp->inv_c[t] = 1.0 / prm->c[t];
    rp->invsqrt[t] = prm->invsqrt[t];
    // second-order prediction of mean((1 + r/c)^p) with mean(r)=0, mean(r^2)=1
    rp->kshift[t + 1] = (t + 1 == prm->T) ? 0.0 : 1.0 + (double)binom2(prm->p[t]) / (prm->c[t] * prm->c[t]);
  }
  rp->inv = prm->inv;
  return PAM_OK;
}

// Geometry of the two-iterations-per-exchange kernel (cutmax_ahead_kernel.cuh).
// Same scoring as choose_geometry: rows per microsecond = clusters / t_row with
// t_row ~= a + b * cap * k; a (two exchanges + chains per row) = 2.6 us,
// b ~= 36 fp64 instructions per element slot at 64/clk/SM = 0.33 ns.
// Dev override: PAM_FORCE_AHEAD = "NTG,E,C".
struct AheadGeometry {
  const AheadVariant* var = nullptr;
  int C = 0, L = 0;
};
int ahead_smem_bytes(const AheadVariant& v) { return ((v.ntg * v.e * 8 + 127) / 128) * 128 + v.ctl_bytes; }

AheadGeometry choose_ahead_geometry(int64_t B, int64_t n) {
  AheadGeometry g;
  if (const char* fs = getenv("PAM_FORCE_AHEAD")) {
    int ntg = 0, e = 0, c = 0;
    if (sscanf(fs, "%d,%d,%d", &ntg, &e, &c) == 3) {
      for (int i = 0; i < kNumAheadVariants; ++i) {
        const AheadVariant& v = kAheadVariants[i];
        const int64_t L = slice_len(n, c, 2);
        if (v.ntg == ntg && v.e == e && (int64_t)v.ntg * v.e >= L) {
          g.var = &v;
          g.C = c;
          g.L = (int)L;
          return g;
        }
      }
    }
  }
  int dev = 0;
  const bool have_gpu = cudaGetDevice(&dev) == cudaSuccess;
  int nsm = 148;
  if (have_gpu && cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) nsm = 148;
  const double a_us = 2.6, b_ns = 0.33;
  double best_score = -1.0;
  for (int C = 1; C <= 16; ++C) {
    const int64_t L = slice_len(n, C, 2);
    for (int i = 0; i < kNumAheadVariants; ++i) {
      const AheadVariant& v = kAheadVariants[i];
      const int64_t cap = (int64_t)v.ntg * v.e;
      if (cap < L || (C > 1 && cap > L + L * 3 / 10)) continue;
      if (C > 1 && L < 2048) continue;
      const int smem = ahead_smem_bytes(v);
      if (smem > 227 * 1024) continue;
      const int active = have_gpu ? max_active_clusters(v.fn, v.ntg, C, smem) : nsm / C;
      if (active <= 0) continue;
      const int64_t clusters = (B < active) ? B : active;
      const int64_t k = (clusters * C + nsm - 1) / nsm;
      const double t_us = a_us + 1e-3 * b_ns * (double)cap * (double)(k < 1 ? 1 : k);
      const double score = (double)clusters / t_us - 1e-9 * (double)C;
      if (score > best_score) {
        best_score = score;
        g.var = &v;
        g.C = C;
        g.L = (int)L;
      }
    }
  }
  cudaGetLastError();
  return g;
}

// The ahead kernel serves fp64, p = 3 everywhere, exact scalars, normalised
// output without the stats side output, on TMA-aligned rows.
bool ahead_eligible(const pam_cutmax_params* prm, bool tma, const double* d_stats) {
  // Opt-in until it beats cutmax_rows_kernel on the headline shape:
  // PAM_ENABLE_AHEAD=1 (or PAM_FORCE_AHEAD=NTG,E,C) selects it.
  if (!getenv("PAM_ENABLE_AHEAD") && !getenv("PAM_FORCE_AHEAD")) return false;
  if (!tma || d_stats || getenv("PAM_DISABLE_AHEAD") || getenv("PAM_FORCE_CFG_F64") || getenv("PAM_FORCE_GENERIC_P"))
    return false;
  if (prm->flags & PAM_F_NO_NORMALIZE) return false;
  if (prm->invsqrt_mode != PAM_MODE_EXACT || prm->inv_mode != PAM_MODE_EXACT) return false;
  for (int t = 0; t < prm->T; ++t)
    if (prm->p[t] != 3) return false;
  return true;
}

template <typename Elem>
int cutmax_batch_impl(const Elem* d_x, int64_t ld_x, int64_t B, int64_t n, const pam_cutmax_params* prm, Elem* d_z,
                      int64_t ld_z, int32_t* d_argmax, int32_t* d_status, double* d_stats, cudaStream_t stream) {
  if (!prm) return PAM_ERR_BAD_ARGUMENT;
  int st = pam_validate_cutmax_params(prm, n);
  if (st) return st;
  if (B < 0 || ld_x < n || ld_z < n || (B > 0 && (!d_x || !d_z))) return PAM_ERR_BAD_ARGUMENT;
  if (prm->eps_stop > 0.0) return PAM_ERR_UNSUPPORTED;
  if (B == 0) return PAM_OK;
  if (n > (int64_t)1 << 30) return PAM_ERR_UNSUPPORTED;
  const int vec = 16 / (int)sizeof(Elem);
  const bool tma = ((uintptr_t)d_x % 16 == 0) && ((uintptr_t)d_z % 16 == 0) && (ld_x % vec == 0) &&
                   (ld_z % vec == 0) && (n % vec == 0) && getenv("PAM_DISABLE_TMA") == nullptr;
  if (sizeof(Elem) == 8 && ahead_eligible(prm, tma, d_stats)) {
    const AheadGeometry ag = choose_ahead_geometry(B, n);
    if (ag.var) {
      const int smem = ahead_smem_bytes(*ag.var);
      const int maxcl = max_active_clusters(ag.var->fn, ag.var->ntg, ag.C, smem);
      if (maxcl <= 0) return cuda_fail(cudaErrorInvalidConfiguration, "no cluster fits (occupancy 0)");
      const int clusters = (int)(B < maxcl ? B : maxcl);
      CutmaxArgs ka;
      memset(&ka, 0, sizeof ka);
      ka.x = d_x;
      ka.z = d_z;
      ka.argmax = d_argmax;
      ka.status = d_status;
      ka.ldx = ld_x;
      ka.ldz = ld_z;
      ka.B = B;
      ka.n = n;
      ka.L = ag.L;
      ka.ctrl_offset = ((ag.var->ntg * ag.var->e * 8 + 127) / 128) * 128;
      ka.tma = 1;
      ka.inv_n = 1.0 / (double)n;
      const char* df = getenv("PAM_DEBUG_FLAGS");
      ka.debug_flags = df ? atoi(df) : 0;
      fill_row_params(prm, &ka.rp);
      if (g_trace && (int64_t)clusters * ag.C * kTraceRows * kTraceEvents <= g_trace_entries) ka.trace = g_trace;
      return launch_cluster_kernel(ag.var->fn, ag.var->ntg, ag.C, clusters, smem, stream, &ka);
    }
  }
  const Geometry g = choose_geometry((int)sizeof(Elem), B, n);
  if (!g.var) return PAM_ERR_UNSUPPORTED;
  bool p3 = getenv("PAM_FORCE_GENERIC_P") == nullptr;  // dev knob: A/B the generic-p kernel
  for (int t = 0; t < prm->T; ++t) p3 = p3 && (prm->p[t] == 3);
  const void* fn = g.var->fn[p3 ? 1 : 0];
  // the row buffer is sized for the full capacity even without TMA so the
  // occupancy (and the chooser's estimate) does not depend on alignment
  const int smem = smem_bytes(*g.var);
  const int nt = g.var->ntg;
  const int maxcl = max_active_clusters(fn, nt, g.C, smem);
  if (maxcl <= 0) return cuda_fail(cudaErrorInvalidConfiguration, "no cluster fits (occupancy 0)");
  const int clusters = (int)(B < maxcl ? B : maxcl);
  CutmaxArgs ka;
  memset(&ka, 0, sizeof ka);
  ka.x = d_x;
  ka.z = d_z;
  ka.argmax = d_argmax;
  ka.status = d_status;
  ka.stats = d_stats;
  ka.ldx = ld_x;
  ka.ldz = ld_z;
  ka.B = B;
  ka.n = n;
  ka.L = g.L;
  ka.ctrl_offset = buffer_bytes(*g.var);
  ka.tma = tma ? 1 : 0;
  ka.inv_n = 1.0 / (double)n;
  {
    const char* df = getenv("PAM_DEBUG_FLAGS");
    ka.debug_flags = df ? atoi(df) : 0;
  }
  if (g_trace && (int64_t)clusters * g.C * kTraceRows * kTraceEvents <= g_trace_entries) ka.trace = g_trace;
  fill_row_params(prm, &ka.rp);
  return launch_cluster_kernel(fn, nt, g.C, clusters, smem, stream, &ka);
}

int sampler_batch_impl(const double* d_x, int64_t ld_x, int64_t B, int64_t n, const pam_sampler_cfg* cfg,
                       const pam_cutmax_params* prm, int32_t* d_token, uint8_t* d_inside, double* d_onehot,
                       int64_t ld_onehot, int32_t* d_status, cudaStream_t stream, bool gumbel) {
  if (!prm || !cfg) return PAM_ERR_BAD_ARGUMENT;
  int st = pam_validate_cutmax_params(prm, n);
  if (st) return st;
  if (B < 0 || ld_x < n || (B > 0 && !d_x) || (d_onehot && ld_onehot < n)) return PAM_ERR_BAD_ARGUMENT;
  if (prm->eps_stop > 0.0) return PAM_ERR_UNSUPPORTED;
  if (!(cfg->p > 0.0 && cfg->p < 1.0)) return PAM_ERR_DOMAIN;
  double alpha = cfg->alpha;
  if (!gumbel && !(alpha > 0.0)) {
    st = pam_nucleus_alpha(cfg->p, cfg->q, &alpha);  // Alg. 3 line 1 / Observation 1
    if (st) return st;
  }
  if (B == 0) return PAM_OK;
  // geometry: smallest cluster whose CTAs can hold the slice
  const SamplerVariant* var = nullptr;
  int C = 0;
  int64_t L = 0;
  for (int c = 1; c <= 16 && !var; c *= 2) {
    L = ((n + c - 1) / c + 1) / 2 * 2;
    for (int i = 0; i < kNumSamplerVariants; ++i) {
      const SamplerVariant& v = kSamplerVariants[i];
      if ((int64_t)v.nt * v.e >= L && (!var || v.nt * v.e < var->nt * var->e)) var = &v;
    }
    if (var) C = c;
  }
  if (!var) return PAM_ERR_UNSUPPORTED;
  bool p3 = true;
  for (int t = 0; t < prm->T; ++t) p3 = p3 && (prm->p[t] == 3);
  const void* fn = var->fn[p3 ? 1 : 0][gumbel ? 1 : 0];
  const int buf_bytes = (int)(((L * 8) + 127) / 128 * 128);
  const int smem = buf_bytes + (int)sizeof(ControlBlock);
  const int maxcl = max_active_clusters(fn, var->nt, C, smem);
  if (maxcl <= 0) return cuda_fail(cudaErrorInvalidConfiguration, "no cluster fits (occupancy 0)");
  const int clusters = (int)(B < maxcl ? B : maxcl);
  SamplerArgs sa;
  memset(&sa, 0, sizeof sa);
  sa.x = d_x;
  sa.onehot = d_onehot;
  sa.token = d_token;
  sa.inside = d_inside;
  sa.status = d_status;
  sa.ldx = ld_x;
  sa.ld_onehot = ld_onehot;
  sa.B = B;
  sa.n = n;
  sa.L = (int32_t)L;
  sa.ctrl_offset = buf_bytes;
  sa.inv_alpha = gumbel ? 1.0 : 1.0 / alpha;
  sa.p_nucleus = cfg->p;
  sa.seed = cfg->seed;
  sa.draw = cfg->draw;
  sa.inv_n = 1.0 / (double)n;
  sa.tma = ((uintptr_t)d_x % 16 == 0) && (ld_x % 2 == 0) && (n % 2 == 0) && getenv("PAM_DISABLE_TMA") == nullptr;
  fill_row_params(prm, &sa.rp);
  if (g_trace && (int64_t)clusters * C * kTraceRows * kTraceEvents <= g_trace_entries) sa.trace = g_trace;
  return launch_cluster_kernel(fn, var->nt, C, clusters, smem, stream, &sa);
}

// ---------------------------------------------------- analysis kernels (§8f)
// Smallest cluster whose CTAs hold ceil(n/C) in registers with one of the
// analysis variants; rows stream over min(B, active clusters) clusters.
int analysis_impl(bool jvp, const double* d_x, const double* d_v, int64_t ld_x, int64_t B, int64_t n,
                  const pam_cutmax_params* prm, double* d_z, double* d_dz, int64_t ld_z, double* d_out,
                  int32_t* d_status, cudaStream_t stream) {
  if (!prm) return PAM_ERR_BAD_ARGUMENT;
  int st = pam_validate_cutmax_params(prm, n);
  if (st) return st;
  if (prm->eps_stop > 0.0) return PAM_ERR_UNSUPPORTED;
  if (B < 0 || ld_x < n || (B > 0 && !d_x)) return PAM_ERR_BAD_ARGUMENT;
  if (jvp && B > 0 && (!d_v || !d_dz || ld_z < n)) return PAM_ERR_BAD_ARGUMENT;
  if (B == 0) return PAM_OK;
  const AnalysisVariant* var = nullptr;
  int C = 0;
  int64_t L = 0;
  for (int c = 1; c <= 16 && !var; ++c) {
    L = (n + c - 1) / c;
    for (int i = 0; i < kNumAnalysisVariants; ++i) {
      const AnalysisVariant& v = kAnalysisVariants[i];
      if ((int64_t)v.nt * v.e >= L && (!var || v.nt * v.e < var->nt * var->e)) var = &v;
    }
    if (var) C = c;
  }
  if (!var) return PAM_ERR_UNSUPPORTED;
  const void* fn = jvp ? var->jvp : var->trace;
  const int smem = (int)sizeof(ControlBlock);
  const int maxcl = max_active_clusters(fn, var->nt, C, smem);
  if (maxcl <= 0) return cuda_fail(cudaErrorInvalidConfiguration, "no cluster fits (occupancy 0)");
  const int clusters = (int)(B < maxcl ? B : maxcl);
  AnalysisArgs aa;
  memset(&aa, 0, sizeof aa);
  aa.x = d_x;
  aa.v = d_v;
  aa.z = d_z;
  aa.dz = d_dz;
  aa.out = d_out;
  aa.status = d_status;
  aa.ldx = ld_x;
  aa.ldz = ld_z;
  aa.B = B;
  aa.n = n;
  aa.L = (int32_t)L;
  aa.ctrl_offset = 0;
  aa.inv_n = 1.0 / (double)n;
  fill_row_params(prm, &aa.rp);
  return launch_cluster_kernel(fn, var->nt, C, clusters, smem, stream, &aa);
}

// ---------------------------------------------------- host-buffer e2e path
struct HostWorkspace {
  std::mutex mu;
  void* dbuf = nullptr;
  size_t cap = 0;
  cudaStream_t streams[3] = {nullptr, nullptr, nullptr};
  int dev = -1;
};
HostWorkspace g_ws;

template <typename Elem>
int cutmax_host_impl(const Elem* h_x, int64_t B, int64_t n, const pam_cutmax_params* prm, Elem* h_z,
                     int32_t* h_argmax, int32_t* h_status) {
  if (!prm || (B > 0 && (!h_x || !h_z))) return PAM_ERR_BAD_ARGUMENT;
  int st = pam_validate_cutmax_params(prm, n);
  if (st) return st;
  if (B == 0) return PAM_OK;
  std::lock_guard<std::mutex> lk(g_ws.mu);
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_ws.dev != dev) {
    for (auto& s : g_ws.streams) s = nullptr;
    g_ws.dbuf = nullptr;
    g_ws.cap = 0;
    g_ws.dev = dev;
  }
  for (auto& s : g_ws.streams)
    if (!s) {
      cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
    }
  const size_t row_bytes = (size_t)n * sizeof(Elem);
  // chunk: ~128 MiB of input per chunk, 3 chunks in flight (PCIe-bound either way: 32 MiB gave
  // 35.5k rows/s, 128 MiB 37.8k at 4096 x 151936 fp64; dev knob PAM_HOST_CHUNK_MB)
  size_t chunk_mb = 128;
  if (const char* e = getenv("PAM_HOST_CHUNK_MB")) chunk_mb = (size_t)atoi(e) > 0 ? (size_t)atoi(e) : 128;
  int64_t rows_per_chunk = (int64_t)((chunk_mb << 20) / row_bytes);
  if (rows_per_chunk < 1) rows_per_chunk = 1;
  if (rows_per_chunk > B) rows_per_chunk = B;
  const size_t per_slot = rows_per_chunk * (2 * row_bytes + 2 * sizeof(int32_t)) + 256;
  const size_t need = 3 * per_slot;
  if (g_ws.cap < need) {
    if (g_ws.dbuf) cudaFree(g_ws.dbuf);
    g_ws.dbuf = nullptr;
    cudaError_t e = cudaMalloc(&g_ws.dbuf, need);
    if (e != cudaSuccess) { g_ws.cap = 0; return cuda_fail(e, "cudaMalloc workspace"); }
    g_ws.cap = need;
  }
  int rc = PAM_OK;
  int64_t chunk = 0;
  for (int64_t r0 = 0; r0 < B; r0 += rows_per_chunk, ++chunk) {
    const int64_t rows = (B - r0) < rows_per_chunk ? (B - r0) : rows_per_chunk;
    const int slot = (int)(chunk % 3);
    cudaStream_t s = g_ws.streams[slot];
    char* base = (char*)g_ws.dbuf + slot * per_slot;
    Elem* dx = (Elem*)base;
    Elem* dz = (Elem*)(base + rows_per_chunk * row_bytes);
    int32_t* dam = (int32_t*)(base + 2 * rows_per_chunk * row_bytes);
    int32_t* dst = dam + rows_per_chunk;
    cudaError_t e = cudaMemcpyAsync(dx, h_x + r0 * n, rows * row_bytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) { rc = cuda_fail(e, "H2D"); break; }
    rc = cutmax_batch_impl<Elem>(dx, n, rows, n, prm, dz, n, dam, dst, nullptr, s);
    if (rc) break;
    e = cudaMemcpyAsync(h_z + r0 * n, dz, rows * row_bytes, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && h_argmax)
      e = cudaMemcpyAsync(h_argmax + r0, dam, rows * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && h_status)
      e = cudaMemcpyAsync(h_status + r0, dst, rows * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) { rc = cuda_fail(e, "D2H"); break; }
  }
  for (auto& s : g_ws.streams) {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess && rc == PAM_OK) rc = cuda_fail(e, "cudaStreamSynchronize");
  }
  return rc;
}

}  // namespace

// ======================================================================= C ABI
extern "C" {

int pam_abi_version(void) { return PAM_ABI_VERSION; }

const char* pam_status_string(int status) {
  switch (status & 0xff) {
    case PAM_OK: return "ok";
    case PAM_ERR_INVALID_PARAMS: return "invalid params";
    case PAM_ERR_DEGENERATE_INPUT: return "degenerate input (variance below eps_var)";
    case PAM_ERR_RANGE: return "range error (approximation domain or normaliser)";
    case PAM_ERR_DOMAIN: return "domain error";
    case PAM_ERR_NON_FINITE: return "non-finite input";
    case PAM_ERR_CUDA: return "CUDA error";
    case PAM_ERR_BAD_ARGUMENT: return "bad argument";
    case PAM_ERR_UNSUPPORTED: return "unsupported";
    case PAM_ERR_FORMAT: return "malformed logit file";
    case PAM_ERR_SINGULAR: return "singular (variance below eps_var on the JVP path)";
    default: return "unknown status";
  }
}

void pam_default_params(pam_cutmax_params* prm, int32_t T, int32_t p, double c) {
  memset(prm, 0, sizeof *prm);
  prm->T = T;
  prm->eps_var = 1e-24;
  prm->invsqrt_mode = PAM_MODE_EXACT;
  prm->inv_mode = PAM_MODE_EXACT;
  for (int t = 0; t < PAM_MAX_T; ++t) {
    prm->p[t] = p;
    prm->c[t] = c;
    prm->invsqrt[t].iterations = 5;  // Table 3: alpha=7 -> 5 iterations
    prm->invsqrt[t].alpha_bits = 7;
    prm->invsqrt[t].rescale = PAM_RESCALE_AUTO;
    prm->invsqrt[t].lo = 0.25;
    prm->invsqrt[t].hi = 1.0;
  }
  prm->inv.iterations = 5;
  prm->inv.alpha_bits = 7;
  prm->inv.rescale = PAM_RESCALE_AUTO;
  prm->inv.lo = 0.5;
  prm->inv.hi = 1.0;
}

int pam_validate_cutmax_params(const pam_cutmax_params* prm, int64_t n) {
  if (!prm) return PAM_ERR_BAD_ARGUMENT;
  if (n < 2) return PAM_ERR_INVALID_PARAMS;
  if (prm->T < 1 || prm->T > PAM_MAX_T) return PAM_ERR_INVALID_PARAMS;      // SPEC.md:67 (T=0 invalid)
  if (!(prm->eps_var >= 0.0) || !(prm->eps_stop >= 0.0)) return PAM_ERR_INVALID_PARAMS;
  if (prm->invsqrt_mode != PAM_MODE_EXACT && prm->invsqrt_mode != PAM_MODE_POLY) return PAM_ERR_INVALID_PARAMS;
  if (prm->inv_mode != PAM_MODE_EXACT && prm->inv_mode != PAM_MODE_POLY) return PAM_ERR_INVALID_PARAMS;
  for (int t = 0; t < prm->T; ++t) {
    const int p = prm->p[t];
    const double c = prm->c[t];
    if (p < 1 || p > 63) return PAM_ERR_INVALID_PARAMS;
    if (!(prm->flags & PAM_F_UNCHECKED) && (p < 3 || p % 2 == 0)) return PAM_ERR_INVALID_PARAMS;
    if (!(c > 0.0) || !std::isfinite(c)) return PAM_ERR_INVALID_PARAMS;
    if ((prm->flags & PAM_F_GUARANTEE) && !(c > std::sqrt((double)(n - 1)))) return PAM_ERR_INVALID_PARAMS;  // :41
    if (prm->invsqrt_mode == PAM_MODE_POLY) {
      const pam_approx_config& a = prm->invsqrt[t];
      if (a.iterations < 0 || a.iterations > 64) return PAM_ERR_INVALID_PARAMS;
      if (a.rescale < 0 || a.rescale > 2) return PAM_ERR_INVALID_PARAMS;
      if (a.rescale == PAM_RESCALE_STATIC && (a.scale_log2 % 2 != 0)) return PAM_ERR_INVALID_PARAMS;
    }
  }
  if (prm->inv_mode == PAM_MODE_POLY) {
    const pam_approx_config& a = prm->inv;
    if (a.iterations < 0 || a.iterations > 64 || a.rescale < 0 || a.rescale > 2) return PAM_ERR_INVALID_PARAMS;
  }
  return PAM_OK;
}

int pam_goldschmidt_inv(double x, const pam_approx_config* cfg, double* out) {
  if (!cfg || !out) return PAM_ERR_BAD_ARGUMENT;
  if (cfg->rescale == PAM_RESCALE_NONE && !(x > 0.0 && x < 2.0)) { *out = 0.0; return PAM_ERR_RANGE; }
  return inv_rescaled(x, cfg->iterations, cfg->rescale, cfg->scale_log2, cfg->lo, cfg->hi, out);
}

int pam_goldschmidt_invsqrt(double x, const pam_approx_config* cfg, double* out) {
  if (!cfg || !out) return PAM_ERR_BAD_ARGUMENT;
  return invsqrt_rescaled(x, cfg->iterations, cfg->rescale, cfg->scale_log2, cfg->lo, cfg->hi, out);
}

int pam_nucleus_alpha(double p, double q, double* out) {
  if (!out) return PAM_ERR_BAD_ARGUMENT;
  if (!(p > 0.0 && p < 1.0 && q > 0.0 && q < 1.0)) { *out = NAN; return PAM_ERR_DOMAIN; }
  *out = log_p(1.0 - q) / log_p(p);
  return PAM_OK;
}

double pam_beta_inverse_cdf(double u, double alpha) { return beta_icdf(u, 1.0 / alpha); }

int pam_gumbel_from_uniform(double u, double* out) {
  if (!out) return PAM_ERR_BAD_ARGUMENT;
  if (!(u > 0.0 && u < 1.0)) { *out = NAN; return PAM_ERR_DOMAIN; }
  *out = gumbel_from_u(u);
  return PAM_OK;
}

double pam_uniform(uint64_t seed, uint64_t row, uint64_t draw, uint64_t index) {
  return uniform_at(seed, row, draw, index);
}

int pam_cutmax_batch_f64(const double* d_x, int64_t ld_x, int64_t B, int64_t n, const pam_cutmax_params* prm,
                         double* d_z, int64_t ld_z, int32_t* d_argmax, int32_t* d_row_status, double* d_stats,
                         void* stream) {
  return cutmax_batch_impl<double>(d_x, ld_x, B, n, prm, d_z, ld_z, d_argmax, d_row_status, d_stats,
                                   (cudaStream_t)stream);
}

int pam_cutmax_batch_f32(const float* d_x, int64_t ld_x, int64_t B, int64_t n, const pam_cutmax_params* prm,
                         float* d_z, int64_t ld_z, int32_t* d_argmax, int32_t* d_row_status, double* d_stats,
                         void* stream) {
  return cutmax_batch_impl<float>(d_x, ld_x, B, n, prm, d_z, ld_z, d_argmax, d_row_status, d_stats,
                                  (cudaStream_t)stream);
}

int pam_cutmax_batch_host_f64(const double* h_x, int64_t B, int64_t n, const pam_cutmax_params* prm, double* h_z,
                              int32_t* h_argmax, int32_t* h_row_status) {
  return cutmax_host_impl<double>(h_x, B, n, prm, h_z, h_argmax, h_row_status);
}

int pam_cutmax_batch_host_f32(const float* h_x, int64_t B, int64_t n, const pam_cutmax_params* prm, float* h_z,
                              int32_t* h_argmax, int32_t* h_row_status) {
  return cutmax_host_impl<float>(h_x, B, n, prm, h_z, h_argmax, h_row_status);
}

int pam_nucleus_sample_batch_f64(const double* d_x, int64_t ld_x, int64_t B, int64_t n, const pam_sampler_cfg* cfg,
                                 const pam_cutmax_params* prm, int32_t* d_token, uint8_t* d_inside, double* d_onehot,
                                 int64_t ld_onehot, int32_t* d_row_status, void* stream) {
  return sampler_batch_impl(d_x, ld_x, B, n, cfg, prm, d_token, d_inside, d_onehot, ld_onehot, d_row_status,
                            (cudaStream_t)stream, false);
}

int pam_gumbel_sample_batch_f64(const double* d_x, int64_t ld_x, int64_t B, int64_t n, const pam_sampler_cfg* cfg,
                                const pam_cutmax_params* prm, int32_t* d_token, uint8_t* d_inside, double* d_onehot,
                                int64_t ld_onehot, int32_t* d_row_status, void* stream) {
  return sampler_batch_impl(d_x, ld_x, B, n, cfg, prm, d_token, d_inside, d_onehot, ld_onehot, d_row_status,
                            (cudaStream_t)stream, true);
}

int pam_convergence_trace_batch_f64(const double* d_x, int64_t ld_x, int64_t B, int64_t n,
                                    const pam_cutmax_params* prm, double* d_out, int32_t* d_row_status,
                                    void* stream) {
  if (B > 0 && !d_out) return PAM_ERR_BAD_ARGUMENT;
  return analysis_impl(false, d_x, nullptr, ld_x, B, n, prm, nullptr, nullptr, n, d_out, d_row_status,
                       (cudaStream_t)stream);
}

int pam_cutmax_jvp_batch_f64(const double* d_x, const double* d_v, int64_t ld_x, int64_t B, int64_t n,
                             const pam_cutmax_params* prm, double* d_z, double* d_dz, int64_t ld_z,
                             int32_t* d_row_status, void* stream) {
  return analysis_impl(true, d_x, d_v, ld_x, B, n, prm, d_z, d_dz, ld_z, nullptr, d_row_status,
                       (cudaStream_t)stream);
}

int pam_query_launch(int dtype_bytes, int64_t B, int64_t n, const pam_cutmax_params* prm, pam_launch_info* info) {
  if (!info || (dtype_bytes != 4 && dtype_bytes != 8)) return PAM_ERR_BAD_ARGUMENT;
  memset(info, 0, sizeof *info);
  if (dtype_bytes == 8 && prm && n % 2 == 0 && ahead_eligible(prm, true, nullptr)) {
    const AheadGeometry ag = choose_ahead_geometry(B, n);
    if (ag.var) {
      const int smem = ahead_smem_bytes(*ag.var);
      info->threads = ag.var->ntg;
      info->elems_per_thread = ag.var->e;
      info->cluster = ag.C;
      info->smem_bytes = smem;
      info->tma = 1;
      const int maxcl = max_active_clusters(ag.var->fn, ag.var->ntg, ag.C, smem);
      info->clusters = (int)(B < maxcl ? B : maxcl);
      info->ctas = info->clusters * ag.C;
      info->groups = 1;
      info->kernel_id = 1000 + (int)(ag.var - kAheadVariants);  // 1000+: the two-iterations-per-exchange kernel
      return PAM_OK;
    }
  }
  const Geometry g = choose_geometry(dtype_bytes, B, n);
  if (!g.var) return PAM_ERR_UNSUPPORTED;
  bool p3 = true;
  if (prm)
    for (int t = 0; t < prm->T; ++t) p3 = p3 && (prm->p[t] == 3);
  const void* fn = g.var->fn[p3 ? 1 : 0];
  const int smem = smem_bytes(*g.var);
  info->threads = g.var->ntg;
  info->elems_per_thread = g.var->e;
  info->cluster = g.C;
  info->smem_bytes = smem;
  info->tma = 1;
  const int maxcl = max_active_clusters(fn, info->threads, g.C, smem);
  info->clusters = (int)(B < maxcl ? B : maxcl);
  info->ctas = info->clusters * g.C;
  info->groups = 1;
  info->kernel_id = (int)(g.var - kCutmaxVariants);
  return PAM_OK;
}

int64_t pam_kernel_launch_count(void) { return g_launches.load(); }

void pam_set_trace_buffer(long long* d_buf, int64_t entries) {
  g_trace = d_buf;
  g_trace_entries = d_buf ? entries : 0;
}

const char* pam_last_cuda_error(void) { return g_last_err; }

}  // extern "C"
