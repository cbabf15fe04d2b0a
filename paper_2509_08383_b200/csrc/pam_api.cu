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
#include <unordered_map>
#include <vector>

#include "../../include/pam_c_api.h"
#include "analysis_kernel.cuh"
#include "cutmax_kernel.cuh"
#include "cutmax_warp_kernel.cuh"
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

// Tuning/test overrides (pam_set_geometry_override, pam_set_host_chunk_bytes).
// Explicit API calls only: the library reads no environment variables.
struct Overrides {
  std::atomic<int> ntg[2]{{0}, {0}}, e[2]{{0}, {0}}, c[2]{{0}, {0}}, minb[2]{{0}, {0}};  // [fp32, fp64]
  std::atomic<int64_t> host_chunk_bytes{128ll << 20};
  std::atomic<int> generation{0};  // bumped on every override change: invalidates the geometry cache
  std::atomic<int> lean{1};        // 0: p = 3 rows always run the general kernel (pam_set_lean_p3, A/B tests)
};
Overrides g_ovr;

// Kernel tables: pam_variants.h (cutmax_variants_f64.cu / _f32.cu, sampler_variants.cu).
const VariantTable kCutmaxTables[2] = {{kCutmaxVariantsF32, kNumCutmaxVariantsF32},
                                       {kCutmaxVariantsF64, kNumCutmaxVariantsF64}};

// Kernel flavour of a CutMax launch: 0 generic p, 1 p = 3 everywhere, 2 generic with early stop.
int flavour_of(const pam_cutmax_params* prm) {
  if (prm->eps_stop > 0.0) return 2;
  for (int t = 0; t < prm->T; ++t)
    if (prm->p[t] != 3) return 0;
  return 1;
}

struct Geometry {
  const Variant* var = nullptr;
  int C = 0;
  int L = 0;
};

int buffer_bytes(const Variant& v) { return ((v.ntg * v.e * v.elem_bytes + 127) / 128) * 128; }
int smem_bytes(const Variant& v) { return buffer_bytes(v) + (int)sizeof(ControlBlock); }

int64_t slice_len(int64_t n, int C, int vec) { return ((n + C - 1) / C + vec - 1) / vec * vec; }

// ---- per-device kernel attributes and occupancy -------------------------------
// cudaFuncSetAttribute applies per device context, so both caches are keyed by
// the device ordinal as well as the kernel.
std::mutex g_occ_mu;
struct FnKey {
  int dev;
  const void* fn;
  int C, smem;
  bool operator==(const FnKey& o) const { return dev == o.dev && fn == o.fn && C == o.C && smem == o.smem; }
};
std::vector<std::pair<FnKey, int>> g_occ_cache;      // (dev, fn, C, smem) -> max active clusters
std::vector<std::pair<FnKey, int>> g_smem_attr;      // (dev, fn) -> largest dynamic smem opted in

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return dev;
}

// Raise the kernel's dynamic-smem opt-in on this device to at least `smem`
// (never lower it: an earlier, larger configuration must stay launchable).
void ensure_smem_attr(int dev, const void* fn, int smem) {
  std::lock_guard<std::mutex> lk(g_occ_mu);
  for (auto& kv : g_smem_attr)
    if (kv.first.dev == dev && kv.first.fn == fn) {
      if (kv.second >= smem) return;
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kv.second = smem;
      return;
    }
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  g_smem_attr.push_back({FnKey{dev, fn, 0, 0}, smem});
}

int max_active_clusters(const void* fn, int nt, int C, int smem) {
  const int dev = current_device();
  ensure_smem_attr(dev, fn, smem);
  const FnKey key{dev, fn, C, smem};
  {
    std::lock_guard<std::mutex> lk(g_occ_mu);
    for (auto& kv : g_occ_cache)
      if (kv.first == key) return kv.second;
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
  g_occ_cache.push_back({key, ncl});
  return ncl;
}

// Launch geometry.  Candidates are every (variant, cluster size C = 1..16)
// whose per-CTA capacity covers the slice ceil(n/C) with < 30% phantom waste.
// They are ranked by rows per microsecond, clusters / t_row, with the row
// period fitted to B200 measurements (tools/tune.py, tools/trace.py):
//   t_row ~= a + b * cap * k
// a = latency per row (T exchanges + scalar chains: fp64 4.8 us, fp32 2.5 us),
// b = element cost per CTA-slot (fp64 0.33 ns, fp32 0.35 ns), cap = NTG*E, and
// k = CTAs sharing an SM (clusters*C / #SMs, rounded up) from the occupancy
// query.  Non power-of-two clusters matter: 9-CTA clusters pack 135 SMs vs 120
// for 8.  Results are cached per (device, dtype, B, n, flavour).
Geometry score_geometry(int elem_bytes, int64_t B, int64_t n, int flavour) {
  Geometry g;
  const int vec = 16 / elem_bytes;
  const VariantTable& tab = kCutmaxTables[elem_bytes == 8 ? 1 : 0];
  const int oi = elem_bytes == 8 ? 1 : 0;
  const int fntg = g_ovr.ntg[oi].load(), fe = g_ovr.e[oi].load(), fc = g_ovr.c[oi].load(), fmb = g_ovr.minb[oi].load();
  if (fntg > 0) {  // pam_set_geometry_override
    for (int i = 0; i < tab.count; ++i) {
      const Variant& v = tab.v[i];
      if (v.ntg == fntg && v.e == fe && v.minb == fmb && v.fn[flavour]) {
        const int64_t L = slice_len(n, fc, vec);
        if ((int64_t)v.ntg * v.e >= L) {
          g.var = &v;
          g.C = fc;
          g.L = (int)L;
        }
        return g;
      }
    }
    return g;
  }
  const int dev = current_device();
  int nsm = 148;
  if (dev >= 0 && cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) nsm = 148;
  const double a_us = elem_bytes == 8 ? 4.8 : 2.5, b_ns = elem_bytes == 8 ? 0.33 : 0.35;
  double best_score = -1.0;
  for (int C = 1; C <= 16; ++C) {
    const int64_t L = slice_len(n, C, vec);
    for (int i = 0; i < tab.count; ++i) {
      const Variant& v = tab.v[i];
      if (!v.fn[flavour]) continue;
      const int64_t cap = (int64_t)v.ntg * v.e;
      if (cap < L || (C > 1 && cap > L + L * 3 / 10 && flavour != 2)) continue;
      if (C > 1 && L < 2048) continue;  // tiny slices: exchanges would dominate
      const int smem = smem_bytes(v);
      if (smem > 227 * 1024) continue;
      const int active = dev >= 0 ? max_active_clusters(v.fn[flavour], v.ntg, C, smem) : nsm / C;
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

struct GeoKey {
  int dev, elem_bytes, flavour, gen;
  int64_t B, n;
  bool operator==(const GeoKey& o) const {
    return dev == o.dev && elem_bytes == o.elem_bytes && flavour == o.flavour && gen == o.gen && B == o.B && n == o.n;
  }
};
struct GeoKeyHash {
  size_t operator()(const GeoKey& k) const {
    return std::hash<int64_t>()(k.B * 1000003 + k.n) ^ ((size_t)k.dev << 40) ^ ((size_t)k.elem_bytes << 48) ^
           ((size_t)k.flavour << 52) ^ ((size_t)k.gen << 56);
  }
};
std::mutex g_geo_mu;
std::unordered_map<GeoKey, Geometry, GeoKeyHash> g_geo_cache;

Geometry choose_geometry(int elem_bytes, int64_t B, int64_t n, int flavour) {
  const GeoKey key{current_device(), elem_bytes, flavour, g_ovr.generation.load(), B, n};
  {
    std::lock_guard<std::mutex> lk(g_geo_mu);
    auto it = g_geo_cache.find(key);
    if (it != g_geo_cache.end()) return it->second;
  }
  const Geometry g = score_geometry(elem_bytes, B, n, flavour);
  std::lock_guard<std::mutex> lk(g_geo_mu);
  if (g_geo_cache.size() > 4096) g_geo_cache.clear();  // bounded
  g_geo_cache.emplace(key, g);
  return g;
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
  rp->eps_stop = prm->eps_stop;
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

// The odd power used at every iteration, or 0 for a mixed schedule.
int uniform_p(const pam_cutmax_params* prm) {
  for (int t = 1; t < prm->T; ++t)
    if (prm->p[t] != prm->p[0]) return 0;
  return prm->p[0];
}

// Lean kernel (cutmax_p3_kernel.cuh) of a general-kernel geometry for one fixed
// power p at every iteration (nullptr: none compiled).  Used for T >= 2,
// aligned rows, no early stopping, unless switched off (pam_set_lean_p3(0)).
const LeanVariant* find_lean(int elem_bytes, const Variant& v, int p) {
  if (!g_ovr.lean.load() || p < 0) return nullptr;  // p = 0: a mixed schedule (the P = 0 kernels)
  const LeanVariant* tabs[3] = {elem_bytes == 8 ? kCutmaxP3F64 : kCutmaxP3F32,
                                elem_bytes == 8 ? kCutmaxPGenF64 : nullptr, elem_bytes == 8 ? kCutmaxPMixF64 : nullptr};
  const int cnts[3] = {elem_bytes == 8 ? kNumCutmaxP3F64 : kNumCutmaxP3F32, elem_bytes == 8 ? kNumCutmaxPGenF64 : 0,
                       elem_bytes == 8 ? kNumCutmaxPMixF64 : 0};
  for (int k = 0; k < 3; ++k)
    for (int i = 0; i < cnts[k]; ++i) {
      const LeanVariant& l = tabs[k][i];
      if (l.p == p && l.ntg == v.ntg && l.e == v.e && l.minb == v.minb) return &l;
    }
  return nullptr;
}

// The fixed-power kernel of the schedule if one is compiled, else the
// mixed-schedule kernel (P = 0: any powers, e.g. the HE schedule p = [16, 4, 4, 6]).
const LeanVariant* find_lean_any(int elem_bytes, const Variant& v, const pam_cutmax_params* prm) {
  const int up = uniform_p(prm);
  const LeanVariant* lv = up > 0 ? find_lean(elem_bytes, v, up) : nullptr;
  return lv ? lv : find_lean(elem_bytes, v, 0);
}

// ---- warp-per-row kernels ------------------------------------------------------
constexpr int kWarpBlock = 256;  // 8 rows in flight per CTA
// smallest compiled E that holds the row; none for early stopping (general kernel)
// or when the specialised kernels are switched off (pam_set_lean_p3(0), A/B tests)
const WarpVariant* pick_warp_variant(int elem_bytes, int64_t n, int flavour) {
  if (flavour == 2 || !g_ovr.lean.load() || g_ovr.ntg[elem_bytes == 8 ? 1 : 0].load() > 0) return nullptr;
  const WarpVariant* best = nullptr;
  for (int i = 0; i < kNumWarpVariants; ++i) {
    const WarpVariant& w = kWarpVariants[i];
    if (w.elem_bytes == elem_bytes && 32 * (int64_t)w.e >= n && (!best || w.e < best->e)) best = &w;
  }
  return best;
}
int warp_kernel_blocks(const void* fn, int64_t B) {
  const int dev = current_device();
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, const void*>, int>> cache;  // (dev, fn) -> resident blocks
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& kv : cache)
      if (kv.first.first == dev && kv.first.second == fn) per_sm = kv.second;
  }
  if (per_sm == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kWarpBlock, 0) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    std::lock_guard<std::mutex> lk(mu);
    cache.push_back({{dev, fn}, per_sm});
  }
  int nsm = 148;
  if (dev >= 0 && cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) nsm = 148;
  const int64_t want = (B + kWarpBlock / 32 - 1) / (kWarpBlock / 32);
  const int64_t cap = (int64_t)per_sm * nsm;
  return (int)(want < cap ? want : cap);
}

template <typename Elem>
int cutmax_batch_impl(const Elem* d_x, int64_t ld_x, int64_t B, int64_t n, const pam_cutmax_params* prm, Elem* d_z,
                      int64_t ld_z, int32_t* d_argmax, int32_t* d_status, double* d_stats, cudaStream_t stream) {
  if (!prm) return PAM_ERR_BAD_ARGUMENT;
  int st = pam_validate_cutmax_params(prm, n);
  if (st) return st;
  if (B < 0 || ld_x < n || ld_z < n || (B > 0 && (!d_x || !d_z))) return PAM_ERR_BAD_ARGUMENT;
  if (B == 0) return PAM_OK;
  if (n > (int64_t)1 << 30) return PAM_ERR_UNSUPPORTED;
  const int vec = 16 / (int)sizeof(Elem);
  const bool tma = ((uintptr_t)d_x % 16 == 0) && ((uintptr_t)d_z % 16 == 0) && (ld_x % vec == 0) &&
                   (ld_z % vec == 0) && (n % vec == 0);
  const int flavour = flavour_of(prm);
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
  ka.tma = tma ? 1 : 0;
  ka.inv_n = 1.0 / (double)n;
  fill_row_params(prm, &ka.rp);
  // short rows: one warp per row (cutmax_warp_kernel.cuh), no cluster
  const WarpVariant* wv = tma ? pick_warp_variant((int)sizeof(Elem), n, flavour) : nullptr;
  if (wv) {
    const void* wfn = wv->fn[n == 32 * (int64_t)wv->e ? 1 : 0][flavour == 1 ? 1 : 0];
    const int blocks = warp_kernel_blocks(wfn, B);
    if (blocks <= 0) return cuda_fail(cudaErrorInvalidConfiguration, "warp kernel occupancy 0");
    const void* args[] = {&ka};
    cudaError_t e = cudaLaunchKernel(wfn, dim3((unsigned)blocks), dim3(kWarpBlock), (void**)args, 0, stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernel(warp rows)");
    g_launches.fetch_add(1);
    return PAM_OK;
  }
  const Geometry g = choose_geometry((int)sizeof(Elem), B, n, flavour);
  if (!g.var) return PAM_ERR_UNSUPPORTED;
  const void* fn = g.var->fn[flavour];
  // p = 3 everywhere, T >= 2, aligned rows: the lean kernel of the same geometry
  if (flavour != 2 && tma && prm->T >= 2)
    if (const LeanVariant* lv = find_lean_any((int)sizeof(Elem), *g.var, prm)) fn = lv->fn;
  // the row buffer is sized for the full capacity even without TMA so the
  // occupancy (and the chooser's estimate) does not depend on alignment
  const int smem = smem_bytes(*g.var);
  const int nt = g.var->ntg;
  const int maxcl = max_active_clusters(fn, nt, g.C, smem);
  if (maxcl <= 0) return cuda_fail(cudaErrorInvalidConfiguration, "no cluster fits (occupancy 0)");
  const int clusters = (int)(B < maxcl ? B : maxcl);
  ka.L = g.L;
  ka.ctrl_offset = buffer_bytes(*g.var);
  if (g_trace && (int64_t)clusters * g.C * kTraceRows * kTraceEvents <= g_trace_entries) ka.trace = g_trace;
  return launch_cluster_kernel(fn, nt, g.C, clusters, smem, stream, &ka);
}

int sampler_batch_impl(const double* d_x, int64_t ld_x, int64_t B, int64_t n, const pam_sampler_cfg* cfg,
                       const pam_cutmax_params* prm, int32_t* d_token, uint8_t* d_inside, double* d_onehot,
                       int64_t ld_onehot, int32_t* d_status, cudaStream_t stream, bool gumbel) {
  if (!prm || !cfg) return PAM_ERR_BAD_ARGUMENT;
  int st = pam_validate_cutmax_params(prm, n);
  if (st) return st;
  if (B < 0 || ld_x < n || (B > 0 && !d_x) || (d_onehot && ld_onehot < n)) return PAM_ERR_BAD_ARGUMENT;
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
  const int flavour = flavour_of(prm);
  const void* fn = flavour == 2 ? var->stop[gumbel ? 1 : 0] : var->fn[flavour][gumbel ? 1 : 0];
  const int buf_bytes = (int)(((L * 8) + 127) / 128 * 128);
  const int smem = buf_bytes + kSamplerTabOffset + kSamplerTabBytes;  // + log/exp tables
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
  sa.tma = ((uintptr_t)d_x % 16 == 0) && (ld_x % 2 == 0) && (n % 2 == 0);
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
// Device staging for the host-pointer entry points: three pipeline slots
// (H2D -> kernel -> D2H, one stream each).  Workspaces are pooled per device:
// a call takes a free one (or creates one) and returns it, so concurrent host
// calls do not serialise on a global lock, and switching devices never drops a
// live allocation.  Workspaces live for the process.
struct HostWorkspace {
  int dev = -1;
  void* dbuf = nullptr;
  size_t cap = 0;
  cudaStream_t streams[3] = {nullptr, nullptr, nullptr};
};
std::mutex g_ws_mu;
std::vector<HostWorkspace*> g_ws_free;  // idle workspaces of every device

HostWorkspace* ws_acquire(int dev) {
  {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (size_t i = 0; i < g_ws_free.size(); ++i)
      if (g_ws_free[i]->dev == dev) {
        HostWorkspace* w = g_ws_free[i];
        g_ws_free.erase(g_ws_free.begin() + (long)i);
        return w;
      }
  }
  HostWorkspace* w = new HostWorkspace();
  w->dev = dev;
  return w;
}
void ws_release(HostWorkspace* w) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  g_ws_free.push_back(w);
}

template <typename Elem>
int cutmax_host_impl(const Elem* h_x, int64_t B, int64_t n, const pam_cutmax_params* prm, Elem* h_z,
                     int32_t* h_argmax, int32_t* h_status) {
  if (!prm || (B > 0 && (!h_x || !h_z))) return PAM_ERR_BAD_ARGUMENT;
  int st = pam_validate_cutmax_params(prm, n);
  if (st) return st;
  if (B == 0) return PAM_OK;
  const int dev = current_device();
  if (dev < 0) return cuda_fail(cudaErrorNoDevice, "cudaGetDevice");
  HostWorkspace* ws = ws_acquire(dev);
  struct Release {
    HostWorkspace* w;
    ~Release() { ws_release(w); }
  } release{ws};
  for (auto& s : ws->streams)
    if (!s) {
      cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
    }
  const size_t row_bytes = (size_t)n * sizeof(Elem);
  // chunk: ~128 MiB of input per chunk, 3 chunks in flight (PCIe-bound either way: 32 MiB gave
  // 35.5k rows/s, 128 MiB 37.8k at 4096 x 151936 fp64; pam_set_host_chunk_bytes overrides)
  const int64_t chunk_bytes = g_ovr.host_chunk_bytes.load();
  int64_t rows_per_chunk = (int64_t)((size_t)chunk_bytes / row_bytes);
  if (rows_per_chunk < 1) rows_per_chunk = 1;
  if (rows_per_chunk > B) rows_per_chunk = B;
  // every sub-buffer starts on a 256-byte boundary, so the kernel keeps its TMA path
  auto up256 = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t xz_bytes = up256(rows_per_chunk * row_bytes);
  const size_t i32_bytes = up256(rows_per_chunk * sizeof(int32_t));
  const size_t per_slot = 2 * xz_bytes + 2 * i32_bytes;
  const size_t need = 3 * per_slot;
  if (ws->cap < need) {
    if (ws->dbuf) {
      for (auto& s : ws->streams) cudaStreamSynchronize(s);
      cudaFree(ws->dbuf);
    }
    ws->dbuf = nullptr;
    ws->cap = 0;
    cudaError_t e = cudaMalloc(&ws->dbuf, need);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc workspace");
    ws->cap = need;
  }
  int rc = PAM_OK;
  int64_t chunk = 0;
  for (int64_t r0 = 0; r0 < B; r0 += rows_per_chunk, ++chunk) {
    const int64_t rows = (B - r0) < rows_per_chunk ? (B - r0) : rows_per_chunk;
    const int slot = (int)(chunk % 3);
    cudaStream_t s = ws->streams[slot];
    char* base = (char*)ws->dbuf + slot * per_slot;
    Elem* dx = (Elem*)base;
    Elem* dz = (Elem*)(base + xz_bytes);
    int32_t* dam = (int32_t*)(base + 2 * xz_bytes);
    int32_t* dst = (int32_t*)(base + 2 * xz_bytes + i32_bytes);
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
  for (auto& s : ws->streams) {
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
  const int flavour = prm ? flavour_of(prm) : 1;
  if (const WarpVariant* wv = pick_warp_variant(dtype_bytes, n, flavour)) {  // warp per row
    const int blocks = warp_kernel_blocks(wv->fn[n == 32 * (int64_t)wv->e ? 1 : 0][flavour == 1 ? 1 : 0], B);
    info->threads = 32;
    info->elems_per_thread = wv->e;
    info->cluster = 1;
    info->clusters = (int)(B < (int64_t)blocks * (kWarpBlock / 32) ? B : (int64_t)blocks * (kWarpBlock / 32));
    info->ctas = blocks;
    info->tma = 0;
    info->groups = 1;
    info->kernel_id = 2000 + (int)(wv - kWarpVariants) + 100 * flavour;
    return PAM_OK;
  }
  const Geometry g = choose_geometry(dtype_bytes, B, n, flavour);
  if (!g.var) return PAM_ERR_UNSUPPORTED;
  const void* fn = g.var->fn[flavour];
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
  const VariantTable& tab = kCutmaxTables[dtype_bytes == 8 ? 1 : 0];
  info->kernel_id = (int)(g.var - tab.v) + 100 * flavour;
  if (flavour != 2 && prm && prm->T >= 2 && find_lean_any(dtype_bytes, *g.var, prm))
    info->kernel_id += 1000;  // lean kernel (aligned rows)
  return PAM_OK;
}

int pam_set_geometry_override(int dtype_bytes, int threads, int elems_per_thread, int cluster, int min_blocks) {
  if (dtype_bytes != 4 && dtype_bytes != 8) return PAM_ERR_BAD_ARGUMENT;
  const int oi = dtype_bytes == 8 ? 1 : 0;
  if (threads > 0) {
    if (cluster < 1 || cluster > 16 || elems_per_thread < 1) return PAM_ERR_BAD_ARGUMENT;
    bool found = false;
    const VariantTable& tab = kCutmaxTables[oi];
    for (int i = 0; i < tab.count; ++i)
      found = found || (tab.v[i].ntg == threads && tab.v[i].e == elems_per_thread && tab.v[i].minb == min_blocks);
    if (!found) return PAM_ERR_UNSUPPORTED;
  }
  g_ovr.ntg[oi] = threads > 0 ? threads : 0;
  g_ovr.e[oi] = elems_per_thread;
  g_ovr.c[oi] = cluster;
  g_ovr.minb[oi] = min_blocks;
  g_ovr.generation.fetch_add(1);
  return PAM_OK;
}

int pam_set_lean_p3(int on) {
  g_ovr.lean = on ? 1 : 0;
  return PAM_OK;
}

int pam_set_host_chunk_bytes(int64_t bytes) {
  g_ovr.host_chunk_bytes = bytes > 0 ? bytes : (128ll << 20);
  return PAM_OK;
}

int64_t pam_kernel_launch_count(void) { return g_launches.load(); }

// for the entry points that live in their own translation unit (nucleus_set.cu)
extern "C" __attribute__((visibility("hidden"))) void pam_internal_count_launch(void) { g_launches.fetch_add(1); }
extern "C" __attribute__((visibility("hidden"))) int pam_internal_cuda_fail(int e, const char* what) {
  return cuda_fail((cudaError_t)e, what);
}

void pam_set_trace_buffer(long long* d_buf, int64_t entries) {
  g_trace = d_buf;
  g_trace_entries = d_buf ? entries : 0;
}

const char* pam_last_cuda_error(void) { return g_last_err; }

}  // extern "C"
