// cutmax_kernel.cuh — fused, row-resident batched CutMax for sm_100a.
//
// Replaces core.cutmax / core.cutmaxStep (Alg. 1).
//
// Geometry.  One logit row is owned by one thread-block cluster of C CTAs
// (C = 1..16).  CTA `rank` owns the contiguous slice [rank*L, min(n,(rank+1)*L))
// and each thread keeps E elements of it in registers for all T iterations:
// HBM is read once (1-D TMA bulk copy into a shared-memory landing buffer,
// prefetched one row ahead) and written once (128-bit streaming stores).
// Clusters are persistent and stride over rows.
//
// Reductions.  Every iteration needs the row mean and variance.  Values are
// stored shifted, v = y - K, with a shift K shared by every CTA (K = x[0] for
// the input, K = 1 + C(p,2)/c^2 — the second-order prediction of the mean of
// (1+r/c)^p — afterwards).  One pass then yields both sum(v) and sum(v^2), so
// one cluster exchange per iteration suffices:
//     dm = S/n,  s2 = Q/n - dm^2,  mu = K + dm.
// If the shift was poor (Q/n > 16 s2, i.e. more than ~1 digit of cancellation)
// the kernel does an exact second pass sum((v-dm)^2) and a second exchange;
// the decision is cluster-uniform because every CTA holds identical sums.
//
// Exchange.  warp shuffle tree -> CTA partial -> each CTA pushes its (S,Q)
// partial into every CTA's slot array with st.async (DSMEM) completing on the
// destination's mbarrier; every warp then sums the C partials in a fixed tree
// order, so all CTAs compute bit-identical mu and s2.  The argmax candidate is
// gathered to rank 0 the same way.
//
// Element update (z = (y-mu)/(c sigma) + 1, y' = z^p):
//     z = fma(v, k, b)  with k = inv_sigma/c, b = 1 - dm*k
//     v' = z^p - K'     (p = 3: fma(z*z, z, -K'))
// which is 5 fp64 instructions per element per iteration including the two
// accumulations (the oracle evaluates the same algebra in textbook order; the
// difference is rounding only and is covered by the 1e-12 normwise tolerance).
#pragma once

#include <stdint.h>
#include <cuda_runtime.h>

#include "../../include/pam_c_api.h"
#include "pam_ptx.cuh"
#include "pam_scalar.h"

namespace pam {

struct RowParams {
  int32_t T, flags, invsqrt_mode, inv_mode;
  int32_t p[PAM_MAX_T];
  double inv_c[PAM_MAX_T];
  double kshift[PAM_MAX_T + 1];  // shift of the stored Y^(t+1) values; kshift[T] = 0
  double eps_var;
  pam_approx_config invsqrt[PAM_MAX_T];
  pam_approx_config inv;
};

struct CutmaxArgs {
  const void* x;
  void* z;
  int32_t* argmax;
  int32_t* status;
  double* stats;
  int64_t ldx, ldz, B, n;
  int32_t L;            // slice length per CTA (elements)
  int32_t ctrl_offset;  // byte offset of the control block in dynamic smem
  RowParams rp;
};

struct __align__(16) ControlBlock {
  double2 xch[2][16];  // exchange slots, double-buffered by round parity
  double2 cand[16];    // argmax candidates (rank 0 only)
  double2 wred[32];    // per-warp partials
  double2 gat[16][2];  // all-gather records (sampler: token candidate + max x)
  unsigned long long mb_load;
  unsigned long long mb_x[2];
  unsigned long long mb_a;
  unsigned long long mb_g;
};

template <typename T>
struct ElemTraits;
template <>
struct ElemTraits<double> {
  using V = double2;
  static constexpr int VEC = 2;
};
template <>
struct ElemTraits<float> {
  using V = float4;
  static constexpr int VEC = 4;
};

__device__ __forceinline__ double fma_e(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float fma_e(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double ipow_e(double z, int p) { return ipow(z, p); }
__device__ __forceinline__ float ipow_e(float z, int p) { return ipowf(z, p); }

// ---------------------------------------------------------------------------
// Cluster-wide sum of two doubles.  All threads of the CTA must call it.
template <int NT>
__device__ __forceinline__ double2 cluster_sum2(double a, double b, ControlBlock* cb, uint32_t& round,
                                                uint32_t rank, uint32_t C) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, off);
    b += __shfl_down_sync(0xffffffffu, b, off);
  }
  if (lane == 0) cb->wred[warp] = make_double2(a, b);
  __syncthreads();
  const uint32_t par = round & 1u, ph = (round >> 1) & 1u;
  if (warp == 0) {
    double2 w = (lane < NW) ? cb->wred[lane] : make_double2(0.0, 0.0);
    a = w.x;
    b = w.y;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      a += __shfl_down_sync(0xffffffffu, a, off);
      b += __shfl_down_sync(0xffffffffu, b, off);
    }
    a = __shfl_sync(0xffffffffu, a, 0);
    b = __shfl_sync(0xffffffffu, b, 0);
    if (lane < (int)C) {
      const uint32_t dst = ptx::mapa(ptx::smem_addr(&cb->xch[par][rank]), (uint32_t)lane);
      const uint32_t bar = ptx::mapa(ptx::smem_addr(&cb->mb_x[par]), (uint32_t)lane);
      ptx::st_async_f64x2(dst, a, b, bar);
    }
  }
  ptx::mbar_wait_cluster(ptx::smem_addr(&cb->mb_x[par]), ph);
  if (threadIdx.x == 0) ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[par]), C * 16u);  // arm round+2
  double2 c = (lane < (int)C) ? cb->xch[par][lane] : make_double2(0.0, 0.0);
  a = c.x;
  b = c.y;
#pragma unroll
  for (int off = 8; off > 0; off >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, off);
    b += __shfl_down_sync(0xffffffffu, b, off);
  }
  a = __shfl_sync(0xffffffffu, a, 0);
  b = __shfl_sync(0xffffffffu, b, 0);
  ++round;
  return make_double2(a, b);
}

__device__ __forceinline__ bool cand_better(double v, long long i, double bv, long long bi) {
  return (v > bv) || (v == bv && i < bi);
}

// ---------------------------------------------------------------------------
// One element update z = fma(v, k, b), v' = z^p - K'.  Used for the register
// slice and for the scalar phantom trajectory, so both round identically.
template <typename Elem, int P>
__device__ __forceinline__ Elem cutmax_update(Elem v, Elem k, Elem b, Elem kn, int p) {
  const Elem zz = fma_e(v, k, b);
  if (P == 3) {
    const Elem z2 = zz * zz;
    return fma_e(z2, zz, kn);
  } else {
    return ipow_e(zz, P > 0 ? P : p) + kn;
  }
}

// Per-iteration scalars from the cluster sums.  Returns false if the shift
// left more than ~1 digit of cancellation (caller then does an exact pass).
__device__ __forceinline__ void moments_from_sums(double S, double Q, double nd, double& dm, double& s2) {
  dm = S / nd;
  s2 = Q / nd - dm * dm;
}

// ---------------------------------------------------------------------------
// CutMax on a register-resident row slice.
//
// On entry v[] holds the CTA's slice: `len` real elements followed by phantom
// elements (slots beyond the slice) that the caller filled with K0.  Phantoms
// keep every pass free of per-element predicates: all phantoms of the row
// carry one common value w_t (a copy of element 0's trajectory in spirit — they
// start at K0 and get the same updates), tracked here as a scalar, and their
// total contribution m*w (m = number of phantoms in the cluster) is subtracted
// from the cluster sums.
//
// On exit v holds Y^(T+1) (shift 0) and rnorm the normaliser inv(sum Y) (1
// when PAM_F_NO_NORMALIZE).  Returns the row status, identical in every CTA.
template <typename Elem, int NT, int E, int P>
__device__ __forceinline__ int cutmax_core(Elem (&v)[E], const double K0, const double mphantom,
                                           const RowParams& rp, const double nd, ControlBlock* cb,
                                           uint32_t& xround, const uint32_t rank, const uint32_t C,
                                           double* stats_row, double& rnorm) {
  constexpr double kGuard = sizeof(Elem) == 8 ? 16.0 : 2.0;  // cancellation guard (see header)
  const int T = rp.T;
  const bool normalize = !(rp.flags & PAM_F_NO_NORMALIZE);
  int st = PAM_OK;
  rnorm = 1.0;

  // exact second pass about dm when the shifted one-pass moments cancelled
  auto guard = [&](double S, double Q, double w, double& dm, double& s2) {
    moments_from_sums(S, Q, nd, dm, s2);
    if (st == PAM_OK && isfinite(Q) && Q / nd > kGuard * s2) {
      const Elem dme = (Elem)dm;
      Elem q2 = 0;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const Elem d = v[i] - dme;
        q2 = fma_e(d, d, q2);
      }
      const double2 r2 = cluster_sum2<NT>((double)q2, 0.0, cb, xround, rank, C);
      const Elem dw = (Elem)w - dme;
      s2 = (r2.x - mphantom * (double)dw * (double)dw) / nd;
    }
  };

  // ---- input pass: shift by K0 (phantoms hold K0 -> contribute exactly 0) ---
  double dm, s2;
  {
    const Elem k0 = (Elem)K0;
    Elem s = 0, q = 0;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const Elem d = v[i] - k0;
      v[i] = d;
      s += d;
      q = fma_e(d, d, q);
    }
    const double2 r = cluster_sum2<NT>((double)s, (double)q, cb, xround, rank, C);
    if (!isfinite(r.x) || !isfinite(r.y)) st = PAM_ERR_NON_FINITE;
    guard(r.x, r.y, 0.0, dm, s2);
  }
  double kcur = K0;
  Elem w = 0;  // phantom value (shifted representation)

  // ---- T iterations; the last one (no variance needed) is peeled ------------
  double total = 0.0;
  for (int t = 0; t < T; ++t) {
    const double mu = kcur + dm;
    if (st == PAM_OK && (!isfinite(mu) || !isfinite(s2))) st = PAM_ERR_RANGE;
    if (st == PAM_OK && s2 < rp.eps_var) st = PAM_ERR_DEGENERATE_INPUT;
    if (stats_row) {
      stats_row[t * 2 + 0] = mu;
      stats_row[t * 2 + 1] = s2;
    }
    double inv_sigma = 0.0;
    if (st == PAM_OK) {
      if (rp.invsqrt_mode == PAM_MODE_POLY) {
        const pam_approx_config& ac = rp.invsqrt[t];
        const int rs = invsqrt_rescaled(s2, ac.iterations, ac.rescale, ac.scale_log2, ac.lo, ac.hi, &inv_sigma);
        if (rs) st = rs;
      } else {
        inv_sigma = 1.0 / sqrt(s2);
      }
    }
    const double kd = (st == PAM_OK) ? inv_sigma * rp.inv_c[t] : 0.0;
    const double bd = fma(-dm, kd, 1.0);
    const double knext = rp.kshift[t + 1];
    const Elem ke = (Elem)kd, be = (Elem)bd, kn = (Elem)(-knext);
    const int p = rp.p[t];
    w = cutmax_update<Elem, P>(w, ke, be, kn, p);
    if (t + 1 < T) {
      Elem s = 0, q = 0;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const Elem d = cutmax_update<Elem, P>(v[i], ke, be, kn, p);
        v[i] = d;
        s += d;
        q = fma_e(d, d, q);
      }
      const double2 r = cluster_sum2<NT>((double)s, (double)q, cb, xround, rank, C);
      const double wd = (double)w;
      guard(r.x - mphantom * wd, r.y - mphantom * wd * wd, wd, dm, s2);
      kcur = knext;
    } else {
      Elem s = 0;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const Elem d = cutmax_update<Elem, P>(v[i], ke, be, kn, p);
        v[i] = d;
        s += d;
      }
      const double2 r = cluster_sum2<NT>((double)s, 0.0, cb, xround, rank, C);
      total = r.x - mphantom * (double)w;  // kshift[T] == 0: v holds Y^(T+1) itself
    }
  }

  if (st == PAM_OK && !isfinite(total)) st = PAM_ERR_RANGE;
  if (st == PAM_OK && normalize) {
    if (rp.inv_mode == PAM_MODE_POLY) {
      const pam_approx_config& ac = rp.inv;
      const int rs = inv_rescaled(total, ac.iterations, ac.rescale, ac.scale_log2, ac.lo, ac.hi, &rnorm);
      if (rs) st = rs;
    } else if (total == 0.0) {
      st = PAM_ERR_RANGE;
    } else {
      rnorm = 1.0 / total;
    }
  }
  return st;
}

// ---------------------------------------------------------------------------
template <typename Elem, int NT, int E, int P, bool TMA>
__global__ void __launch_bounds__(NT, 1) cutmax_rows_kernel(const CutmaxArgs a) {
  using Tr = ElemTraits<Elem>;
  using V = typename Tr::V;
  constexpr int VEC = Tr::VEC;
  constexpr int NV = E / VEC;
  constexpr int NW = NT / 32;
  static_assert(E % VEC == 0, "E must be a multiple of the vector width");
  static_assert(NT % 32 == 0 && NW <= 32, "bad block size");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  Elem* buf = reinterpret_cast<Elem*>(smem_raw);
  ControlBlock* cb = reinterpret_cast<ControlBlock*>(smem_raw + a.ctrl_offset);

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = ptx::cluster_ctarank();
  const uint32_t C = ptx::cluster_nctarank();
  const int64_t cid = ptx::cluster_id_x();
  const int64_t ncl = ptx::nclusters_x();
  const int64_t n = a.n;
  const int64_t base = (int64_t)rank * a.L;
  const int64_t rem = n - base;
  const int len = rem <= 0 ? 0 : (rem < a.L ? (int)rem : a.L);
  const double nd = (double)n;
  const double mphantom = (double)((int64_t)C * NT * E - n);  // phantom slots in the cluster
  const RowParams& rp = a.rp;
  const int T = rp.T;
  const Elem* __restrict__ X = reinterpret_cast<const Elem*>(a.x);
  Elem* __restrict__ Z = reinterpret_cast<Elem*>(a.z);

  const uint32_t bar_load = ptx::smem_addr(&cb->mb_load);
  const uint32_t load_bytes = (uint32_t)len * (uint32_t)sizeof(Elem);
  uint64_t policy = 0;
  if (TMA) policy = ptx::policy_evict_first();

  if (tid == 0) {
    ptx::mbar_init(bar_load, 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_x[0]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_x[1]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_a), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[0]), C * 16u);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[1]), C * 16u);
    if (rank == 0) ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_a), C * 16u);
  }
  ptx::cluster_sync();

  auto issue_load = [&](int64_t row) {
    // one elected thread: arm the load barrier and stream the slice in 32 KB pieces
    ptx::mbar_arrive_expect_tx(bar_load, load_bytes);
    const unsigned char* src = reinterpret_cast<const unsigned char*>(X + row * a.ldx + base);
    const uint32_t dst = ptx::smem_addr(buf);
    for (uint32_t off = 0; off < load_bytes; off += 32768u) {
      const uint32_t nb = (load_bytes - off) < 32768u ? (load_bytes - off) : 32768u;
      ptx::bulk_g2s(dst + off, src + off, nb, bar_load, policy);
    }
  };

  uint32_t xround = 0, load_par = 0, a_par = 0;
  if (TMA && tid == 0 && cid < a.B) issue_load(cid);

  Elem v[E];

  for (int64_t row = cid; row < a.B; row += ncl) {
    const Elem* xrow = X + row * a.ldx;
    const Elem k0e = __ldg(xrow);           // shift for the input pass (same in every CTA)
    const double K0 = (double)k0e;
    __syncthreads();                          // previous row fully retired (wred / cand reuse)

    // ---- load the slice into registers --------------------------------------
    if (TMA) {
      ptx::mbar_wait_cta(bar_load, load_par);
      load_par ^= 1u;
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const int li0 = (k * NT + tid) * VEC;
        if (li0 + VEC <= len) {
          const V t = *reinterpret_cast<const V*>(buf + li0);
          *reinterpret_cast<V*>(&v[k * VEC]) = t;
        } else {
#pragma unroll
          for (int j = 0; j < VEC; ++j) v[k * VEC + j] = (li0 + j < len) ? buf[li0 + j] : k0e;  // phantoms = K0
        }
      }
      __syncthreads();  // landing buffer free: prefetch the next row of this cluster
      if (tid == 0 && row + ncl < a.B) issue_load(row + ncl);
    } else {
      const Elem* src = xrow + base;
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const int li0 = (k * NT + tid) * VEC;
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[k * VEC + j] = (li0 + j < len) ? __ldcs(src + li0 + j) : k0e;
      }
    }

    // ---- input statistics + T CutMax iterations + normaliser -------------------
    double rnorm = 1.0;
    int st = cutmax_core<Elem, NT, E, P>(v, K0, mphantom, rp, nd, cb, xround, rank, C,
                                         (rank == 0 && tid == 0 && a.stats) ? a.stats + row * T * 2 : nullptr,
                                         rnorm);

    // ---- normalisation, argmax, store ----------------------------------------
    const Elem re = (Elem)rnorm;
    double best = -HUGE_VAL;
    long long besti = 0x7fffffffffffffffLL;
    Elem* zrow = Z + row * a.ldz + base;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int li0 = (k * NT + tid) * VEC;
      Elem o[VEC];
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        o[j] = v[k * VEC + j] * re;
        if (li0 + j < len && (double)o[j] > best) {
          best = (double)o[j];
          besti = base + li0 + j;
        }
      }
      if (TMA && li0 + VEC <= len) {
        __stcs(reinterpret_cast<V*>(zrow + li0), *reinterpret_cast<V*>(o));
      } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j)
          if (li0 + j < len) __stcs(zrow + li0 + j, o[j]);
      }
    }
    // argmax: warp tree -> CTA -> gather to rank 0 (lowest index wins ties)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, best, off);
      const long long oi = __shfl_down_sync(0xffffffffu, besti, off);
      if (cand_better(ov, oi, best, besti)) { best = ov; besti = oi; }
    }
    if (lane == 0) cb->wred[warp] = make_double2(best, __longlong_as_double(besti));
    __syncthreads();
    if (warp == 0) {
      double2 w = (lane < NW) ? cb->wred[lane] : make_double2(-HUGE_VAL, __longlong_as_double(0x7fffffffffffffffLL));
      best = w.x;
      besti = __double_as_longlong(w.y);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, best, off);
        const long long oi = __shfl_down_sync(0xffffffffu, besti, off);
        if (cand_better(ov, oi, best, besti)) { best = ov; besti = oi; }
      }
      if (lane == 0) {
        const uint32_t dst = ptx::mapa(ptx::smem_addr(&cb->cand[rank]), 0u);
        const uint32_t bar = ptx::mapa(ptx::smem_addr(&cb->mb_a), 0u);
        ptx::st_async_b64x2(dst, (uint64_t)__double_as_longlong(best), (uint64_t)besti, bar);
      }
      if (rank == 0) {
        ptx::mbar_wait_cluster(ptx::smem_addr(&cb->mb_a), a_par);
        a_par ^= 1u;
        double2 w2 = (lane < (int)C) ? cb->cand[lane]
                                     : make_double2(-HUGE_VAL, __longlong_as_double(0x7fffffffffffffffLL));
        best = w2.x;
        besti = __double_as_longlong(w2.y);
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) {
          const double ov = __shfl_down_sync(0xffffffffu, best, off);
          const long long oi = __shfl_down_sync(0xffffffffu, besti, off);
          if (cand_better(ov, oi, best, besti)) { best = ov; besti = oi; }
        }
        if (lane == 0) {
          ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_a), C * 16u);  // arm next row
          if (a.argmax) a.argmax[row] = (st == PAM_OK) ? (int32_t)besti : -1;
          if (a.status) a.status[row] = st;
        }
      }
    }
  }
  ptx::cluster_sync();  // no CTA leaves while a peer may still push into its shared memory
}

}  // namespace pam
