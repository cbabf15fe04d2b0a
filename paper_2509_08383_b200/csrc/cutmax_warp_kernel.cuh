// cutmax_warp_kernel.cuh — batched CutMax for short rows: one warp per row.
//
// Replaces core.cutmax (Alg. 1) for n <= 32*E
// (fp64 n <= 1536, fp32 n <= 3072 with the compiled E): the whole row lives in
// one warp's registers, so every mean / variance reduction is a 5-level
// shuffle butterfly -- no CTA barrier, no DSMEM, no control warp -- and each
// warp streams its own rows (rows w, w + W, ... for W warps in the grid).  HBM
// is read once (128-bit streaming loads) and written once (128-bit streaming
// stores).  Same algebra and numerics pins as the cluster kernels
// (cutmax_kernel.cuh header): shifted one-pass moments with the exact second
// pass when they cancel, the fp64-rounded input mean, z = fma(v, k, b),
// p = 3 as fma(z*z, z, -K'), the analytic normaliser for p = 3 everywhere,
// argmax of Y^(T+1) with the lowest index on ties, TieWarning from the
// 32-bit screen (tie_decide) with an exact re-scan of the row when undecided.
#pragma once

#include "cutmax_kernel.cuh"

namespace pam {

// Polynomial-mode scalars out of line: a warp runs each row's code once, so
// keeping cold paths out of the instruction stream matters more here than in
// the cluster kernels (whose passes amortise the fetch over 17k elements).
static __device__ __noinline__ int warp_invsqrt_poly(double x, int iters, int rescale, int scale_log2, double lo,
                                                     double hi, double* out) {
  return invsqrt_rescaled(x, iters, rescale, scale_log2, lo, hi, out);
}
static __device__ __noinline__ int warp_inv_poly(double x, int iters, int rescale, int scale_log2, double lo,
                                                 double hi, double* out) {
  return inv_rescaled(x, iters, rescale, scale_log2, lo, hi, out);
}

// Resident 256-thread CTAs per SM the slice registers allow (E*size/4 data
// registers plus ~50 of state): more warps = more rows in flight per SM.
template <typename Elem, int E>
constexpr int warp_kernel_minb() {
  constexpr int data = E * (int)sizeof(Elem) / 4;
  return data <= 16 ? 3 : (data <= 64 ? 2 : 1);
}

// P = 3: p = 3 at every iteration (analytic normaliser); P = 0: runtime schedule.
// FULLROW: n == 32 * E, every slot holds an element (no phantom predicates).
template <typename Elem, int E, int P, bool FULLROW>
__global__ void __launch_bounds__(256, (warp_kernel_minb<Elem, E>())) cutmax_warp_kernel(const CutmaxArgs a) {
  using Tr = ElemTraits<Elem>;
  using V = typename Tr::V;
  constexpr int VEC = Tr::VEC;
  constexpr int NV = E / VEC;
  constexpr double kGuard = sizeof(Elem) == 8 ? 16.0 : 2.0;
  static_assert(E % VEC == 0, "E must be a multiple of the vector width");
  constexpr unsigned FULL = 0xffffffffu;

  const int lane = (int)(threadIdx.x & 31);
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n = a.n;
  const int T = a.rp.T;
  const double inv_n = a.inv_n, nd = (double)n;
  // aligned rows only (16-byte rows, n % VEC == 0; the launcher sends the rest
  // to the cluster kernel): whole vector slots are real or phantom
  const Elem* __restrict__ X = reinterpret_cast<const Elem*>(a.x);
  Elem* __restrict__ Z = reinterpret_cast<Elem*>(a.z);
  // element index of slot i of this lane (slots in increasing element order);
  // the real slots of a lane are a prefix 0 .. nreal-1 (the rest are phantoms)
  auto eidx = [&](int i) { return ((i / VEC) * 32 + lane) * VEC + (i % VEC); };
  int nreal = 0;
#pragma unroll
  for (int i = 0; i < E; ++i) nreal += (int64_t)eidx(i) < n ? 1 : 0;
  auto real = [&](int i) { return FULLROW || i < nreal; };
  auto wsum2 = [&](double& s, double& q) {
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) {
      s += __shfl_xor_sync(FULL, s, m);
      q += __shfl_xor_sync(FULL, q, m);
    }
  };
  auto wsum1 = [&](double& s) {
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) s += __shfl_xor_sync(FULL, s, m);
  };

  Elem v[E];
  for (int64_t row = wid; row < a.B; row += nwarps) {
    const Elem* xr = X + row * a.ldx;
    Elem* zr = Z + row * a.ldz;
    const Elem k0 = __ldg(xr);
    if (row + nwarps < a.B) {  // this warp's next row -> L2 while this one iterates
      const char* nx = reinterpret_cast<const char*>(X + (row + nwarps) * a.ldx);
      for (int64_t off = (int64_t)lane * 128; off < n * (int64_t)sizeof(Elem); off += 32 * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(nx + off));
    }
    // ---- load (phantom slots hold K0: exact zeros once shifted) + screen ----
    float t1 = -INFINITY, t2 = -INFINITY;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int64_t e0 = (int64_t)(k * 32 + lane) * VEC;
      if (real(k * VEC)) {
        const V xv = __ldcs(reinterpret_cast<const V*>(xr + e0));
        const Elem* xe = reinterpret_cast<const Elem*>(&xv);
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[k * VEC + j] = xe[j];
      } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[k * VEC + j] = k0;
      }
#pragma unroll
      for (int j = 0; j < VEC; ++j)
        if (real(k * VEC + j)) top2f_add(t1, t2, hiword_f(v[k * VEC + j]));
    }
    // ---- input moments about K0 ---------------------------------------------
    double S, Q;
    {
      Elem sa = 0, qa = 0;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const Elem d = v[i] - k0;
        v[i] = d;
        sa += d;  // phantoms contribute exactly 0
        qa = fma_e(d, d, qa);
      }
      S = (double)sa;
      Q = (double)qa;
      wsum2(S, Q);
    }
    int st = (isfinite(S) && isfinite(Q)) ? PAM_OK : PAM_ERR_NON_FINITE;
    double R = 0.0, kcur = (double)k0, rnorm = 1.0;
    double* stats_row = (a.stats && lane == 0) ? a.stats + row * T * 2 : nullptr;

    // moments of the current iterate (shift kcur) -> (dm, s2), with the exact
    // second pass about dm when the one-pass form cancelled (warp-uniform)
    auto moments = [&](bool need3, double& dm, double& s2, double& e1, double& m3) {
      dm = S * inv_n;
      const double qn = Q * inv_n;
      s2 = fma(-dm, dm, qn);
      e1 = 0.0;
      m3 = 0.0;
      if (need3) {
        e1 = fma(-nd, dm, S);
        m3 = fma(dm, fma(2.0 * dm, dm, -3.0 * qn), R * inv_n);
      }
      if (st == PAM_OK && isfinite(Q) && qn > kGuard * s2) {
        const Elem dme = (Elem)dm;
        Elem q2 = 0, r3 = 0;
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const Elem d = v[i] - dme;
          const Elem f = d * d;
          if (real(i)) {
            q2 += f;
            r3 = fma_e(f, d, r3);
          }
        }
        double q2d = (double)q2, r3d = (double)r3;
        wsum2(q2d, r3d);
        s2 = q2d * inv_n;
        if (need3) m3 = r3d * inv_n;
      }
    };
    auto finish_total = [&](double total) {
      double rn = 1.0;
      if (st == PAM_OK && !isfinite(total)) st = PAM_ERR_RANGE;
      if (st == PAM_OK && !(a.rp.flags & PAM_F_NO_NORMALIZE)) {
        if (!(total > 0.0)) {
          st = PAM_ERR_RANGE;  // Z must be a distribution (pin A7)
        } else if (a.rp.inv_mode == PAM_MODE_POLY) {
          const pam_approx_config& ac = a.rp.inv;
          const int rs = warp_inv_poly(total, ac.iterations, ac.rescale, ac.scale_log2, ac.lo, ac.hi, &rn);
          if (rs) st = rs;
        } else {
          rn = 1.0 / total;
        }
      }
      return rn;
    };
    // status, stats, 1/sigma -> (k, b) of iteration t
    auto chain = [&](int t, double& dm, double s2, double& kd, double& bd) {
      const double mu = kcur + dm;
      if (t == 0) dm = mu - kcur;  // the reference's fp64-rounded input mean
      const bool bad_range = !isfinite(mu) || !isfinite(s2);
      st = (st != PAM_OK) ? st : (bad_range ? PAM_ERR_RANGE : (s2 < a.rp.eps_var ? PAM_ERR_DEGENERATE_INPUT : PAM_OK));
      if (stats_row) {
        stats_row[t * 2 + 0] = mu;
        stats_row[t * 2 + 1] = s2;
      }
      double inv_sigma = 0.0;
      if (a.rp.invsqrt_mode != PAM_MODE_POLY) {
        inv_sigma = rsqrt(s2);
      } else if (st == PAM_OK) {
        const pam_approx_config& ac = a.rp.invsqrt[t];
        const int rs = warp_invsqrt_poly(s2, ac.iterations, ac.rescale, ac.scale_log2, ac.lo, ac.hi, &inv_sigma);
        if (rs) st = rs;
      }
      kd = (st == PAM_OK) ? inv_sigma * a.rp.inv_c[t] : 0.0;
      bd = fma(-dm, kd, 1.0);
    };

    // ---- iterations 0 .. T-2: update + moments (+ third power sum before the last, p = 3)
    for (int t = 0; t + 1 < T; ++t) {
      double dm, s2, e1, m3, kd, bd;
      moments(false, dm, s2, e1, m3);
      chain(t, dm, s2, kd, bd);
      const Elem ke = (Elem)kd, be = affine_coef<Elem>(bd, dm), kn = (Elem)(-a.rp.kshift[t + 1]);
      const int p = a.rp.p[t];
      const bool need3 = (P == 3) && (t + 2 == T);
      Elem sa = 0, qa = 0, ra = 0;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const Elem d = cutmax_update<Elem, P>(v[i], ke, be, kn, p);
        v[i] = d;
        if (real(i)) {
          sa += d;
          if (need3) {
            const Elem f = d * d;
            qa += f;
            ra = fma_e(f, d, ra);
          } else {
            qa = fma_e(d, d, qa);
          }
        }
      }
      S = (double)sa;
      Q = (double)qa;
      wsum2(S, Q);
      if (need3) {
        R = (double)ra;
        wsum1(R);
      }
      kcur = a.rp.kshift[t + 1];
      if (!isfinite(S) || !isfinite(Q)) st = (st != PAM_OK) ? st : PAM_ERR_RANGE;
    }

    // ---- last iteration: Y^(T+1), argmax, Z ---------------------------------
    double dm, s2, e1, m3, kd, bd;
    moments(P == 3 && T >= 2, dm, s2, e1, m3);
    chain(T - 1, dm, s2, kd, bd);
    bool explicit_sum = !(P == 3 && T >= 2);
    if (!explicit_sum) {  // analytic normaliser sum (1 + k d)^3 (cutmax_kernel.cuh p = 3 flow)
      const double total = nd + kd * (3.0 * e1 + kd * (3.0 * nd * s2 + kd * nd * m3));
      if (st == PAM_OK && !isfinite(total))
        explicit_sum = true;
      else
        rnorm = finish_total(total);
    }
    const Elem ke = (Elem)kd, be = affine_coef<Elem>(bd, dm), kz = (Elem)0;
    const int p = a.rp.p[T - 1];
    Elem bestv = -INFINITY;
    long long besti = 0x7fffffffffffffffLL;
    Elem ta = 0;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const Elem y = cutmax_update<Elem, P>(v[i], ke, be, kz, p);
      v[i] = y;
      if (real(i)) {
        ta += y;
        if (y > bestv) {  // slots in increasing element order: strict > keeps the lowest index
          bestv = y;
          besti = i;  // slot; the element index is formed once below
        }
      }
    }
    double best = (double)bestv;
    if (besti != 0x7fffffffffffffffLL) besti = eidx((int)besti);
    warp_argmax(best, besti);
    if (explicit_sum) {
      double tot = (double)ta;
      wsum1(tot);
      rnorm = finish_total(tot);
    }
    const Elem re = (Elem)rnorm;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int64_t e0 = (int64_t)(k * 32 + lane) * VEC;
      Elem o[VEC];
#pragma unroll
      for (int j = 0; j < VEC; ++j) o[j] = v[k * VEC + j] * re;
      if (real(k * VEC)) __stcs(reinterpret_cast<V*>(zr + e0), *reinterpret_cast<const V*>(o));
    }

    // ---- TieWarning: screen keys, exact re-scan when undecided ---------------
    int k1 = fkey(t1), k2 = fkey(t2);
    top2k_warp(k1, k2);
    int td = tie_decide<Elem>(st, k1, k2);
    if (td == 2) {  // warp-uniform: exact fp64 top-2 of the row
      double m1 = -HUGE_VAL, m2 = -HUGE_VAL;
      for (int64_t i = lane; i < n; i += 32) top2_add(m1, m2, (double)xr[i]);
      bfly_top2<32>(m1, m2);
      td = (m1 - m2 < 1e-9) ? 1 : 0;
    }
    if (lane == 0) {
      if (a.argmax) a.argmax[row] = (st == PAM_OK) ? (int32_t)besti : -1;
      if (a.status) a.status[row] = st | (td == 1 ? PAM_ROW_FLAG_TIE : 0);
    }
  }
}

}  // namespace pam
