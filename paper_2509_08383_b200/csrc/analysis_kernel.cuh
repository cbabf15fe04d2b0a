// analysis_kernel.cuh — the CutMax analysis outputs of SURVEY §8f on the GPU:
//   trace_rows_kernel  convergenceTrace: per iteration mu, s2,
//                      the non-top dispersion U and the
//                      fraction of entries below the mean (Fig. 3)
//   jvp_rows_kernel    cutmaxJvp: forward-mode directional
//                      derivative through mean, variance, 1/sqrt, odd power and
//                      normalisation (the math of oracle.c orc_cutmax_jvp)
// Both are fp64, one row per thread-block cluster (rows strided over the
// persistent clusters), slices in registers, direct loads (no TMA pipeline:
// these are analysis paths, not the decode hot path).  Cluster sums use the
// exchange of cutmax_kernel.cuh, so every CTA holds bit-identical statistics.
// Slots past the slice are excluded from every sum by a predicate.
#pragma once

#include "cutmax_kernel.cuh"

namespace pam {

struct AnalysisArgs {
  const double* x;
  const double* v;  // JVP direction (nullable for the trace)
  double* z;        // JVP: Z (nullable)
  double* dz;       // JVP: directional derivative
  double* out;      // trace: [B][T][4] {mu, s2, dispersion, frac_below_mean}
  int32_t* status;
  int64_t ldx, ldz, B, n;
  int32_t L;
  int32_t ctrl_offset;
  double inv_n;
  RowParams rp;
};

// Common per-CTA setup; returns false for CTAs without rows.
struct AnalysisCtx {
  uint32_t rank, C;
  int64_t cid, ncl, base;
  int len;
};

__device__ __forceinline__ AnalysisCtx analysis_ctx(const AnalysisArgs& a) {
  AnalysisCtx c;
  c.rank = ptx::cluster_ctarank();
  c.C = ptx::cluster_nctarank();
  c.cid = ptx::cluster_id_x();
  c.ncl = ptx::nclusters_x();
  c.base = (int64_t)c.rank * a.L;
  const int64_t rem = a.n - c.base;
  c.len = rem <= 0 ? 0 : (rem < a.L ? (int)rem : a.L);
  return c;
}

__device__ __forceinline__ void analysis_init(ControlBlock* cb, uint32_t C) {
  if (threadIdx.x == 0) {
    ptx::mbar_init(ptx::smem_addr(&cb->mb_x[0]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_x[1]), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[0]), C * kXchBytes);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[1]), C * kXchBytes);
  }
  ptx::cluster_sync();
}

// ---------------------------------------------------------------------------
// convergenceTrace.  Per iteration t (oracle.c orc_convergence_trace):
//   exchange 1: S = sum d, Q = sum d^2 (d = y - K0), argmax(y)   -> mu, s2, top
//   exchange 2: count(y < mu), R = sum_{j != top} r_j            -> rbar = R/(n-1)
//   exchange 3: U = sum_{j != top} (r_j - rbar)^2, with the update y <- (k(y - mu) + 1)^p
// r_j = (y_j - mu) / sigma.  The first failing iteration's status is final;
// later iterations still run (in lockstep) but write nothing.
template <int NT, int E>
__global__ void __launch_bounds__(NT, 1) trace_rows_kernel(const AnalysisArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ControlBlock* cb = reinterpret_cast<ControlBlock*>(smem_raw + a.ctrl_offset);
  const int tid = (int)threadIdx.x;
  const AnalysisCtx c = analysis_ctx(a);
  analysis_init(cb, c.C);
  const RowParams& rp = a.rp;
  const int T = rp.T;
  const double nd = (double)a.n;
  auto real = [&](int i) { return i * NT + tid < c.len; };  // slot i = element base + i*NT + tid
  uint32_t xr = 0;
  double y[E];
  for (int64_t row = c.cid; row < a.B; row += c.ncl) {
    const double* xr_ = a.x + row * a.ldx + c.base;
    const double K0 = __ldg(a.x + row * a.ldx);
#pragma unroll
    for (int i = 0; i < E; ++i) y[i] = real(i) ? __ldg(xr_ + i * NT + tid) - K0 : 0.0;  // shifted by K0
    double K = K0;  // shift of the stored values
    int st = PAM_OK;
    bool fin = true;
#pragma unroll
    for (int i = 0; i < E; ++i) fin = fin && isfinite(y[i]);
    {
      double dummy = 0.0;
      long long di = 0;
      const double2 f = cluster_reduce<NT, false>(fin ? 0.0 : 1.0, 0.0, dummy, di, cb, xr, c.rank, c.C, tid);
      if (f.x != 0.0) st = PAM_ERR_NON_FINITE;
    }
    for (int t = 0; t < T; ++t) {
      // exchange 1: moments + argmax
      double s = 0.0, q = 0.0, best = -HUGE_VAL;
      long long besti = 0x7fffffffffffffffLL;
#pragma unroll
      for (int i = 0; i < E; ++i)
        if (real(i)) {
          s += y[i];
          q = fma(y[i], y[i], q);
          if (y[i] > best) {
            best = y[i];
            besti = c.base + i * NT + tid;
          }
        }
      const double2 m = cluster_reduce<NT, true>(s, q, best, besti, cb, xr, c.rank, c.C, tid);
      const double dm = m.x / nd;
      double s2 = fma(-dm, dm, m.y / nd);
      if (isfinite(m.y) && m.y / nd > 16.0 * s2) {  // cancellation: exact second pass (cluster-uniform)
        double q2 = 0.0;
#pragma unroll
        for (int i = 0; i < E; ++i)
          if (real(i)) q2 = fma(y[i] - dm, y[i] - dm, q2);
        s2 = cluster_sum2<NT>(q2, 0.0, cb, xr, c.rank, c.C, tid).x / nd;
      }
      const double mu = K + dm;
      if (st == PAM_OK && (!isfinite(mu) || !isfinite(s2))) st = PAM_ERR_RANGE;
      if (st == PAM_OK && !(s2 >= rp.eps_var)) st = PAM_ERR_DEGENERATE_INPUT;
      const double inv_s = (st == PAM_OK) ? 1.0 / sqrt(s2) : 0.0;
      // exchange 2: count below the mean, sum of non-top residuals
      double below = 0.0, rs = 0.0;
#pragma unroll
      for (int i = 0; i < E; ++i)
        if (real(i)) {
          if (y[i] < dm) below += 1.0;
          if (c.base + i * NT + tid != besti) rs += (y[i] - dm) * inv_s;
        }
      const double2 br = cluster_sum2<NT>(below, rs, cb, xr, c.rank, c.C, tid);
      const double rbar = br.y / (nd - 1.0);
      // exchange 3: dispersion, fused with the update
      const double k = inv_s * rp.inv_c[t];
      const double Kn = (t + 1 < T) ? rp.kshift[t + 1] : 0.0;
      const int p = rp.p[t];
      double disp = 0.0;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const double d = y[i] - dm;
        if (real(i) && c.base + i * NT + tid != besti) {
          const double r = d * inv_s - rbar;
          disp = fma(r, r, disp);
        }
        y[i] = ipow(d * k + 1.0, p) - Kn;
      }
      const double U = cluster_sum2<NT>(disp, 0.0, cb, xr, c.rank, c.C, tid).x;
      if (c.rank == 0 && tid == 0 && st == PAM_OK && a.out) {
        double* o = a.out + (row * T + t) * 4;
        o[0] = mu;
        o[1] = s2;
        o[2] = U;
        o[3] = br.x / nd;
      }
      K = Kn;
    }
    if (c.rank == 0 && tid == 0 && a.status) a.status[row] = st;
  }
  ptx::cluster_sync();
}

// ---------------------------------------------------------------------------
// cutmaxJvp.  Registers hold d = y - K and the tangent y'.  Per iteration one
// exchange of (sum d, sum d^2) and one of (sum y', sum d y'):
//   mu' = sum y'/n,  s2' = 2 (sum d y' - dm sum y')/n,  k' = -k s2'/(2 s2)
//   u = k (d - dm) + 1,  u' = k' (d - dm) + k (y' - mu'),  y = u^p,  y' = p u^(p-1) u'
// then Z = Y/S and Z' = Y'/S - Y S'/S^2 after one more exchange (S, S').
template <int NT, int E>
__global__ void __launch_bounds__(NT, 1) jvp_rows_kernel(const AnalysisArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ControlBlock* cb = reinterpret_cast<ControlBlock*>(smem_raw + a.ctrl_offset);
  const int tid = (int)threadIdx.x;
  const AnalysisCtx c = analysis_ctx(a);
  analysis_init(cb, c.C);
  const RowParams& rp = a.rp;
  const int T = rp.T;
  const double nd = (double)a.n;
  auto real = [&](int i) { return i * NT + tid < c.len; };
  uint32_t xr = 0;
  double y[E], dy[E];
  for (int64_t row = c.cid; row < a.B; row += c.ncl) {
    const double* xrw = a.x + row * a.ldx + c.base;
    const double* vrw = a.v + row * a.ldx + c.base;
    const double K0 = __ldg(a.x + row * a.ldx);
    bool fin = true;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      y[i] = real(i) ? __ldg(xrw + i * NT + tid) - K0 : 0.0;
      dy[i] = real(i) ? __ldg(vrw + i * NT + tid) : 0.0;
      fin = fin && isfinite(y[i]) && isfinite(dy[i]);
    }
    int st = PAM_OK;
    {
      double dummy = 0.0;
      long long di = 0;
      const double2 f = cluster_reduce<NT, false>(fin ? 0.0 : 1.0, 0.0, dummy, di, cb, xr, c.rank, c.C, tid);
      if (f.x != 0.0) st = PAM_ERR_NON_FINITE;
    }
    for (int t = 0; t < T; ++t) {
      double s = 0.0, q = 0.0, ds = 0.0, dq = 0.0;
#pragma unroll
      for (int i = 0; i < E; ++i)
        if (real(i)) {
          s += y[i];
          q = fma(y[i], y[i], q);
          ds += dy[i];
          dq = fma(y[i], dy[i], dq);
        }
      const double2 m = cluster_sum2<NT>(s, q, cb, xr, c.rank, c.C, tid);
      const double2 dmm = cluster_sum2<NT>(ds, dq, cb, xr, c.rank, c.C, tid);
      const double dm = m.x / nd, dmu = dmm.x / nd;
      double s2 = fma(-dm, dm, m.y / nd);
      double ds2 = 2.0 * (dmm.y - dm * dmm.x) / nd;
      if (isfinite(m.y) && m.y / nd > 16.0 * s2) {  // cancellation: exact moments about dm
        double q2 = 0.0, dq2 = 0.0;
#pragma unroll
        for (int i = 0; i < E; ++i)
          if (real(i)) {
            q2 = fma(y[i] - dm, y[i] - dm, q2);
            dq2 = fma(y[i] - dm, dy[i], dq2);
          }
        const double2 e = cluster_sum2<NT>(q2, dq2, cb, xr, c.rank, c.C, tid);
        s2 = e.x / nd;
        ds2 = 2.0 * e.y / nd;
      }
      if (st == PAM_OK && !(s2 >= rp.eps_var)) st = PAM_ERR_SINGULAR;
      if (st == PAM_OK && (!isfinite(s2) || !isfinite(ds2))) st = PAM_ERR_RANGE;
      const double k = (st == PAM_OK) ? (1.0 / sqrt(s2)) * rp.inv_c[t] : 0.0;
      const double dk = (st == PAM_OK) ? -k * ds2 / (2.0 * s2) : 0.0;
      const double Kn = (t + 1 < T) ? rp.kshift[t + 1] : 0.0;
      const int p = rp.p[t];
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const double d = y[i] - dm;
        const double u = d * k + 1.0;
        const double du = dk * d + k * (dy[i] - dmu);
        y[i] = ipow(u, p) - Kn;
        dy[i] = (double)p * ipow(u, p - 1) * du;
      }
    }
    double sy = 0.0, sdy = 0.0;
#pragma unroll
    for (int i = 0; i < E; ++i)
      if (real(i)) {
        sy += y[i];
        sdy += dy[i];
      }
    const double2 S = cluster_sum2<NT>(sy, sdy, cb, xr, c.rank, c.C, tid);
    if (st == PAM_OK && (!(S.x > 0.0) || !isfinite(S.x))) st = PAM_ERR_RANGE;
    const double r = (st == PAM_OK) ? 1.0 / S.x : 0.0;
    double* zrw = a.z ? a.z + row * a.ldz + c.base : nullptr;
    double* dzrw = a.dz + row * a.ldz + c.base;
#pragma unroll
    for (int i = 0; i < E; ++i)
      if (real(i)) {
        if (zrw) zrw[i * NT + tid] = y[i] * r;
        dzrw[i * NT + tid] = dy[i] * r - y[i] * S.y * r * r;
      }
    if (c.rank == 0 && tid == 0 && a.status) a.status[row] = st;
  }
  ptx::cluster_sync();
}

}  // namespace pam
