// cutmax_p3_kernel.cuh — lean batched CutMax for a fixed odd power at every
// iteration (p = 3, the headline schedule, and the Table-1 powers 5, 9, 13, 19;
// PAPER.md:277-280) or, as P = 0, a per-iteration schedule p[t] (the HE
// schedule of PAPER.md:291), T >= 2, 16-byte aligned rows (TMA path).
//
// Replaces core.cutmax for those parameters (Alg. 1
// PAPER.md:51-72); every other case runs cutmax_rows_kernel (cutmax_kernel.cuh),
// whose p = 3 flow this kernel restates with the same algebra, exchanges and
// rounding, so both produce bit-identical Z, argmax and status.
//
// Row pipeline (one row per cluster of C CTAs, slice in registers):
//   control 0 -> pass 0 -> xchg 0 -> ... -> control T-2 -> pass T-2 (+ third
//   power sum) -> xchg T-2 -> control T-1 (+ analytic normaliser inv(sum Y))
//   -> fused last pass: Y = z^3 (argmax), Z = Y * inv(sum Y) into the row
//   buffer, X(next) - K0(next) out of it into registers with its moments and
//   TieWarning screen -> closing exchange (argmax + next row's input sums),
//   the DMA lane streams Z out behind it and X(next+1) in during xchg 0 / 1.
// Register budget.  The 512 threads hold the slice (E fp64 = 2E registers)
// and the pass coefficients.  The control warp's scalar state (cluster sums,
// moments, phantom value, status) lives in ControlBlock; the per-iteration
// shift K_t and 1/c_t are read from the kernel parameters where they are used.
// Argmax, status and the TieWarning decision of a row are written by the
// control warp inside the next row's first exchange wait.
#pragma once

#include "cutmax_kernel.cuh"

namespace pam {

// Runtime power -> compile-time constant for the even powers of the paper's HE
// schedule (p = [16, 4, 4, 6]) and their neighbours, so that the
// unrolled passes of the mixed-schedule kernel (P = 0) get a fully unrolled
// square-and-multiply; any other power runs ipow's loop (same multiplications in
// the same order either way).  p = 3 is left to the loop: the fixed-power kernel's
// fused fma(z^2, z, -K') rounds once less than ipow(z, 3) - K'.
template <int PP>
struct PowC {
  static constexpr int value = PP;
};
template <typename F>
__device__ __forceinline__ void dispatch_power(const int p, F&& f) {
  switch (p) {
    case 2: f(PowC<2>()); break;
    case 4: f(PowC<4>()); break;
    case 6: f(PowC<6>()); break;
    case 8: f(PowC<8>()); break;
    case 16: f(PowC<16>()); break;
    default: f(PowC<0>()); break;
  }
}

// P: the odd power at every iteration (3: analytic normaliser; other P: an
// explicit sum of Y^(T+1) -- one more pass and exchange -- before the fused
// last pass).  P = 0: a per-iteration schedule p[t] (any powers; explicit sum).
template <typename Elem, int NTG, int E, int MINB = 0, int P = 3>
__global__ void __launch_bounds__(NTG, (MINB > 0 ? MINB : min_blocks_for<Elem, NTG, E>()))
    cutmax_lean_kernel(const CutmaxArgs a) {
  using Tr = ElemTraits<Elem>;
  using V = typename Tr::V;
  constexpr int VEC = Tr::VEC;
  constexpr int NV = E / VEC;
  constexpr int NW = NTG / 32;
  constexpr double kGuard = sizeof(Elem) == 8 ? 16.0 : 2.0;  // cancellation guard (cutmax_kernel.cuh header)
  static_assert(E % VEC == 0 && E % 2 == 0, "E must be a multiple of the vector width");
  static_assert(NTG % 32 == 0 && NW >= 2 && NW <= 16 && (NW & (NW - 1)) == 0, "bad CTA size");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int gtid = (int)threadIdx.x;
  const int warp = gtid >> 5;
  Elem* buf = reinterpret_cast<Elem*>(smem_raw);
  ControlBlock* cb = reinterpret_cast<ControlBlock*>(smem_raw + a.ctrl_offset);

  const uint32_t rank = ptx::cluster_ctarank();
  const uint32_t C = ptx::cluster_nctarank();
  const int64_t cid = ptx::cluster_id_x();
  const int64_t ncl = ptx::nclusters_x();
  const int64_t base = (int64_t)rank * a.L;
  const int64_t rem = a.n - base;
  const int len = rem <= 0 ? 0 : (rem < a.L ? (int)rem : a.L);
  const bool dma = gtid == NTG - 32;  // lane 0 of the last warp issues every bulk copy
  const int T = a.rp.T;
  const Elem* __restrict__ X = reinterpret_cast<const Elem*>(a.x);
  Elem* __restrict__ Z = reinterpret_cast<Elem*>(a.z);
  // slot i of this thread holds a real element (fp32 predicates its sums; fp64
  // subtracts the phantoms' common contribution mph * w instead)
  auto real = [&](int i) { return sizeof(Elem) == 8 || ((i / VEC) * NTG + gtid) * VEC + (i % VEC) < len; };
  auto mph = [&]() { return sizeof(Elem) == 8 ? (double)((int64_t)C * NTG * E - a.n) : 0.0; };

  const uint32_t bar_load = ptx::smem_addr(&cb->mb_load);
  const uint32_t slice_bytes = (uint32_t)len * (uint32_t)sizeof(Elem);
  const uint32_t chunk = ((slice_bytes + 63u) / 64u) * 16u;  // 4 bulk chunks per slice
  const int nch = chunk ? (int)((slice_bytes + chunk - 1) / chunk) : 0;
  const uint64_t policy = ptx::policy_evict_first();

  if (gtid == 0) {
    cb->unc_n = 0;
    cb->fin_pending = 0;
    ptx::mbar_init(bar_load, 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_x[0]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_x[1]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_t[0]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_t[1]), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (gtid == 0) {
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[0]), C * kXchBytes);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[1]), C * kXchBytes);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_t[0]), C * 16u);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_t[1]), C * 16u);
  }
  ptx::cluster_sync();
#ifdef PAM_CHECKED_BUILD
  PAM_CHECK(len <= NTG * E && len % VEC == 0 && a.L % VEC == 0 && a.L <= NTG * E);
  PAM_CHECK((uintptr_t)a.x % 16 == 0 && (uintptr_t)a.z % 16 == 0 && a.ldx % VEC == 0 && a.ldz % VEC == 0);
  for (int i = gtid; i < NTG * E; i += NTG) buf[i] = Elem(NAN);  // poison: reading an unlanded row gives NaN
  ptx::fence_proxy_async_smem();
  __syncthreads();
#endif

  auto load_chunk = [&](int64_t r, int i) {
    const unsigned char* src = reinterpret_cast<const unsigned char*>(X + r * a.ldx + base);
    const uint32_t off = (uint32_t)i * chunk;
    const uint32_t nb = (slice_bytes - off) < chunk ? (slice_bytes - off) : chunk;
    PAM_CHECK(r >= 0 && r < a.B && ((uintptr_t)(src + off) & 15) == 0 && nb % 16 == 0 && off + nb <= slice_bytes);
    ptx::bulk_g2s(ptx::smem_addr(buf) + off, src + off, nb, bar_load, policy);
  };
  auto store_all = [&](int64_t r) {  // buf -> Z(r), one bulk group per chunk
    unsigned char* dst = reinterpret_cast<unsigned char*>(Z + r * a.ldz + base);
    for (int i = 0; i < nch; ++i) {
      const uint32_t off = (uint32_t)i * chunk;
      const uint32_t nb = (slice_bytes - off) < chunk ? (slice_bytes - off) : chunk;
      PAM_CHECK(r >= 0 && r < a.B && ((uintptr_t)(dst + off) & 15) == 0 && nb % 16 == 0);
      ptx::bulk_s2g(dst + off, ptx::smem_addr(buf) + off, nb, policy);
      ptx::bulk_commit();
    }
  };

  int64_t row = cid;
  uint32_t xround = 0, load_par = 0;
  int64_t lrow = 0;
  Elem v[E];
  auto bar1 = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(NTG) : "memory"); };

  // control warp, once per row: input top-2 keys -> TieWarning decision; rank 0
  // writes argmax and status; undecided rows are queued (cluster-uniform)
  // (called by warp 1 for pipelined rows, warp 0 for a cluster's last row)
  auto finish_row = [&](int64_t r, int st, long long amax, int64_t lr) {
    const int2 kk = top2k_wait_row(cb, lr, C, gtid & 31);
    const int td = tie_decide_shifted<Elem>(st, kk.x, kk.y);
    const bool lead = (gtid & 31) == 0;
    if (rank == 0 && lead) {
      if (a.argmax) a.argmax[r] = (st == PAM_OK) ? (int32_t)amax : -1;
      if (a.status) a.status[r] = st | (td == 1 ? PAM_ROW_FLAG_TIE : 0);
    }
    if (td == 2 && lead) {
      const int q = cb->unc_n;
      if (q < 16) cb->unc_rows[q] = r;
      cb->unc_n = q + 1;
    }
  };

  // TieWarning screen of a row's input (cutmax_kernel.cuh: tie_decide_shifted):
  // the top-2 high words of the shifted input v = fl(x - K0) over this
  // thread's real slots, reduced per warp and stashed in wt2[warp]; exchange 0
  // combines and sends the CTA's record.  Runs where the warps are idle: right
  // after the closing exchange's push (warp 0 before its wait, the others
  // before the control barrier), when the registers hold the next row's input.
  auto screen_stash = [&]() {
    float m1 = -INFINITY, m2 = -INFINITY;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      if ((k * NTG + gtid) * VEC < len) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) top2f_add(m1, m2, hiword_f(v[k * VEC + j]));
      }
    }
    int k1 = fkey(m1), k2 = fkey(m2);
    top2k_warp(k1, k2);
    if ((gtid & 31) == 0) cb->wt2[warp] = make_double2(__longlong_as_double((long long)pack_keys(k1, k2)), 0.0);
  };

  if (row < a.B) {  // ---- prologue: the cluster's first row -> registers, input sums
    if (dma) {
      ptx::mbar_arrive_expect_tx(bar_load, slice_bytes);
      for (int i = 0; i < nch; ++i) load_chunk(row, i);
    }
    ptx::mbar_wait_cta(bar_load, load_par);
    load_par ^= 1u;
    const Elem k0 = __ldg(X + row * a.ldx);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int li0 = (k * NTG + gtid) * VEC;
      if (li0 < len) {  // whole vector slots are real or phantom (see the last pass)
        const V xn = *reinterpret_cast<const V*>(buf + li0);
        const Elem* xe = reinterpret_cast<const Elem*>(&xn);
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[k * VEC + j] = xe[j];
      } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[k * VEC + j] = k0;  // phantoms = K0
      }
    }
    __syncthreads();  // buf free
    // same rounding and order as the swap's input sums, so a row's result does
    // not depend on whether it is its cluster's first row (T >= 2: the input's
    // third power sum is not needed)
    Elem sa = 0, qa = 0;  // same order as the last pass's input sums
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const Elem d = v[i] - k0;
      v[i] = d;
      sa += d;
      qa = fma_e(d, d, qa);
    }
    const double2 part = make_double2((double)sa, (double)qa);
    const double2 r = cluster_sum2<NTG>(part.x, part.y, cb, xround, rank, C, gtid);
    if (gtid == 0) {
      cb->p3_S = r.x;
      cb->p3_Q = r.y;
    }
    screen_stash();
  }

  Elem k0_cur = row < a.B ? __ldg(X + row * a.ldx) : Elem(0);
  for (; row < a.B; row += ncl, ++lrow) {
    const int64_t next = row + ncl;
    const bool has_next = next < a.B;
#ifdef PAM_TRACE_BUILD
    long long* tr =
        (a.trace && lrow < kTraceRows) ? a.trace + ((int64_t)blockIdx.x * kTraceRows + lrow) * kTraceEvents : nullptr;
#else
    long long* tr = nullptr;
#endif
    PAM_TRACE(tr, 0);
    const double K0 = (double)k0_cur;
    const Elem k0next = has_next ? __ldg(X + next * a.ldx) : Elem(0);
    if (warp == 0) {  // new row: status from the input sums, phantom value 0 (= K0 shifted)
      if (gtid == 0) {
        cb->p3_st = (isfinite(cb->p3_S) && isfinite(cb->p3_Q)) ? PAM_OK : PAM_ERR_NON_FINITE;
        cb->p3_w = 0.0;
      }
      __syncwarp();
    }
    PAM_TRACE(tr, 2);

    // DMA lane: X(next) -> buffer, chunk by chunk behind the previous row's Z store
    int issued = 0;
    auto issue_upto = [&](int upto) {
      if (!has_next) return;
      if (issued == 0 && upto > 0) ptx::mbar_arrive_expect_tx(bar_load, slice_bytes);
      for (; issued < upto; ++issued) {
        ptx::bulk_wait_read_le(nch - 1 - issued);
        load_chunk(next, issued);
      }
    };

    // ---- scalar chain of iteration t (control warp; every lane identical) -----
    // status, stats, 1/sigma, (k, b) and for t = T-1 the analytic normaliser
    // sum (1 + k d)^3 = n + 3k e1 + 3k^2 n s2 + k^3 n m3 (NaN: explicit sum needed)
    auto finish_total = [&](double total, int& st) -> double {
      double rn = 1.0;
      if (st == PAM_OK && !isfinite(total)) st = PAM_ERR_RANGE;
      if (st == PAM_OK && !(a.rp.flags & PAM_F_NO_NORMALIZE)) {
        if (!(total > 0.0)) {
          st = PAM_ERR_RANGE;  // Z must be a distribution (pin A7)
        } else if (a.rp.inv_mode == PAM_MODE_POLY) {
          const pam_approx_config& ac = a.rp.inv;
          const int rs = inv_rescaled(total, ac.iterations, ac.rescale, ac.scale_log2, ac.lo, ac.hi, &rn);
          if (rs) st = rs;
        } else {
          rn = 1.0 / total;
        }
      }
      return rn;
    };
    auto scalar_chain = [&](int t, double kcur, double& dm, double s2, double e1, double m3, int& st, double& kd,
                            double& bd, double& rn) {
      const double mu = kcur + dm;
      // input iteration: center on the reference's fp64-rounded mean
      if (t == 0) dm = mu - kcur;
      const bool bad_range = !isfinite(mu) || !isfinite(s2);
      st = (st != PAM_OK) ? st : (bad_range ? PAM_ERR_RANGE : (s2 < a.rp.eps_var ? PAM_ERR_DEGENERATE_INPUT : PAM_OK));
      if (a.stats && rank == 0 && gtid == 0) {
        a.stats[row * T * 2 + t * 2 + 0] = mu;
        a.stats[row * T * 2 + t * 2 + 1] = s2;
      }
      double inv_sigma = 0.0;
      if (a.rp.invsqrt_mode != PAM_MODE_POLY) {
        inv_sigma = rsqrt(s2);  // ~1 ulp; identical in every CTA of the cluster
      } else if (st == PAM_OK) {
        const pam_approx_config& ac = a.rp.invsqrt[t];
        const int rs = invsqrt_rescaled(s2, ac.iterations, ac.rescale, ac.scale_log2, ac.lo, ac.hi, &inv_sigma);
        if (rs) st = rs;
      }
      kd = (st == PAM_OK) ? inv_sigma * a.rp.inv_c[t] : 0.0;
      bd = fma(-dm, kd, 1.0);
      rn = 1.0;
      if (t == T - 1) {
        if (P != 3) {  // no closed form: the CTA sums Y^(T+1) explicitly
          rn = NAN;
          return;
        }
        const double nd = (double)a.n;
        const double total = nd + kd * (3.0 * e1 + kd * (3.0 * nd * s2 + kd * nd * m3));
        if (st == PAM_OK && !isfinite(total)) {
          rn = NAN;  // explicit sum needed (rare): signalled to the CTA
          return;
        }
        rn = finish_total(total, st);
      }
    };

    // ---- control step t (warp 0 computes, everyone receives) ----------------
    // returns the affine coefficients (ke, be) and, for t = T-1, the normaliser re
    auto control = [&](int t, Elem& ke, Elem& be, Elem& re) {
      const bool last = (t == T - 1);
      const double inv_n = a.inv_n, nd = (double)a.n;
      if (warp == 0) {
        const double kcur = (t == 0) ? K0 : a.rp.kshift[t];
        int st = cb->p3_st;
        const double S = cb->p3_S, Q = cb->p3_Q;
        double dm = S * inv_n;
        const double qn = Q * inv_n;
        double s2 = fma(-dm, dm, qn);
        double e1 = 0.0, m3 = 0.0;
        if (last && P == 3) {
          e1 = fma(-nd, dm, S);
          m3 = fma(dm, fma(2.0 * dm, dm, -3.0 * qn), cb->p3_R * inv_n);
        }
        const bool exact2 = (st == PAM_OK && isfinite(Q) && qn > kGuard * s2);
        if (exact2) {  // one-pass moments cancelled: exact second pass about dm first
          if (lane_of(gtid) == 0) {
            cb->p3_dm = dm;
            cb->p3_e1 = e1;
            cb->bc.dm = dm;
            cb->bc.flag = 1;
          }
        } else {
          double kd, bd, rn;
          scalar_chain(t, kcur, dm, s2, e1, m3, st, kd, bd, rn);
          if (lane_of(gtid) == 0) {
            cb->p3_st = st;
            cb->bc.ke = kd;
            cb->bc.be = bd;
            cb->bc.dm = dm;
            cb->bc.re = rn;
            cb->bc.flag = 0;
          }
        }
      }
      bar1();
      Bcast b = cb->bc;
      if (b.flag) {  // exact second pass about dm (cluster-uniform, rare)
        const Elem dme = (Elem)b.dm;
        Elem q2a = 0, q2b = 0, r3a = 0, r3b = 0;
#pragma unroll
        for (int i = 0; i < E; i += 2) {
          const Elem d0 = v[i] - dme, d1 = v[i + 1] - dme;
          const Elem f0 = d0 * d0, f1 = d1 * d1;
          if (real(i)) {
            q2a += f0;
            r3a = fma_e(f0, d0, r3a);
          }
          if (real(i + 1)) {
            q2b += f1;
            r3b = fma_e(f1, d1, r3b);
          }
        }
        const double2 r2 =
            cluster_sum2<NTG>((double)q2a + (double)q2b, (double)r3a + (double)r3b, cb, xround, rank, C, gtid);
        if (warp == 0) {
          const double kcur = (t == 0) ? K0 : a.rp.kshift[t];
          int st = cb->p3_st;
          double dm = b.dm;
          const double dw = (double)((Elem)cb->p3_w - dme);
          const double s2 = (r2.x - mph() * dw * dw) * inv_n;
          const double m3 = last ? (r2.y - mph() * dw * dw * dw) * inv_n : 0.0;
          double kd, bd, rn;
          scalar_chain(t, kcur, dm, s2, cb->p3_e1, m3, st, kd, bd, rn);
          if (lane_of(gtid) == 0) {
            cb->p3_st = st;
            cb->bc.ke = kd;
            cb->bc.be = bd;
            cb->bc.dm = dm;
            cb->bc.re = rn;
            cb->bc.flag = 0;
          }
        }
        bar1();
        b = cb->bc;
      }
      ke = (Elem)b.ke;
      be = affine_coef<Elem>(b.be, b.dm);
      re = (Elem)b.re;
      // (bc is rewritten only after the next push's CTA barrier: no barrier here)
    };
    for (int t = 0; t + 1 < T; ++t) {
      Elem ke, be, re_unused;
      control(t, ke, be, re_unused);
      const Elem kn = (Elem)(-a.rp.kshift[t + 1]);
      PAM_TRACE(tr, 13 + t);
      const bool need3 = (P == 3) && (t + 2 == T);
      Elem sa = 0, sb = 0, qa = 0, qb = 0, ra = 0, rb = 0;
      const int pt = P > 0 ? P : a.rp.p[t];
      auto pass = [&](auto r3_c, auto pc) {
        constexpr bool R3 = decltype(r3_c)::value;
        constexpr int PP = P > 0 ? P : decltype(pc)::value;
#pragma unroll
        for (int i = 0; i < E; i += 2) {
          const Elem d0 = cutmax_update<Elem, PP>(v[i], ke, be, kn, pt);
          const Elem d1 = cutmax_update<Elem, PP>(v[i + 1], ke, be, kn, pt);
          v[i] = d0;
          v[i + 1] = d1;
          if (R3) {
            const Elem f0 = d0 * d0, f1 = d1 * d1;
            if (real(i)) {
              sa += d0;
              qa += f0;
              ra = fma_e(f0, d0, ra);
            }
            if (real(i + 1)) {
              sb += d1;
              qb += f1;
              rb = fma_e(f1, d1, rb);
            }
          } else {
            if (real(i)) {
              sa += d0;
              qa = fma_e(d0, d0, qa);
            }
            if (real(i + 1)) {
              sb += d1;
              qb = fma_e(d1, d1, qb);
            }
          }
        }
      };
      if (P == 0)
        dispatch_power(pt, [&](auto pc) { pass(BoolC<false>(), pc); });
      else if (need3)
        pass(BoolC<true>(), PowC<P>());
      else
        pass(BoolC<false>(), PowC<P>());
      PAM_TRACE(tr, 5 + 2 * t);
      auto side = [&]() {
        if (t == 0) issue_upto(nch / 2);
        if (t == 1) issue_upto(nch);
        if (t < 2) PAM_TRACE_DMA(tr, 25 + t);
      };
      const KeyPush kp{t == 0, 0, 0, (uint32_t)(lrow & 1), true};  // records stashed by screen_stash()
      if (need3)
        xch_push<NTG, kSum3>((double)sa + (double)sb, (double)qa + (double)qb, (double)ra + (double)rb, 0LL, cb,
                             xround, rank, C, gtid, side, true, kp);
      else
        xch_push<NTG, kSum2>((double)sa + (double)sb, (double)qa + (double)qb, 0.0, 0LL, cb, xround, rank, C, gtid,
                             side, true, kp);
      PAM_TRACE(tr, 16 + t);
      if (warp == 1 && t == 0 && cb->fin_pending) {
        // previous row's argmax / status / TieWarning: warp 1 would only wait at
        // the control barrier now, so this stays off the control warp's path
        finish_row(cb->fin_row, cb->fin_st, cb->fin_best, lrow - 1);
        __syncwarp();
        if (gtid == 32) cb->fin_pending = 0;
      }
      if (warp == 0) {
        double r3 = 0.0;
        long long ci = 0;
        const double2 r = need3 ? xch_wait<kSum3>(r3, ci, cb, xround, C, gtid)
                                : xch_wait<kSum2>(r3, ci, cb, xround, C, gtid);
        const double wd = (double)cutmax_update<Elem, P>((Elem)cb->p3_w, ke, be, kn, pt);
        const double m = mph();
        __syncwarp();
        if (gtid == 0) {
          cb->p3_w = wd;
          cb->p3_S = r.x - m * wd;
          cb->p3_Q = r.y - m * wd * wd;
          cb->p3_R = r3 - m * wd * wd * wd;
        }
        __syncwarp();
      } else {
        ++xround;  // keep the round counter in step with warp 0
      }
      PAM_TRACE(tr, 6 + 2 * t);
    }

    // ---- last iteration: normaliser first, then the fused pass ---------------
    Elem ke, be, re;
    control(T - 1, ke, be, re);
    const Elem kz = (Elem)0;  // kshift[T] = 0
    const int pl = P > 0 ? P : a.rp.p[T - 1];
    if (!(re == re)) {  // explicit sum of Y: P != 3, or the analytic total is not finite (rare); cluster-uniform
      Elem ta = 0, tb = 0;
      auto sumy = [&](auto pc) {
        constexpr int PP = P > 0 ? P : decltype(pc)::value;
#pragma unroll
        for (int i = 0; i < E; i += 2) {
          const Elem y0 = cutmax_update<Elem, PP>(v[i], ke, be, kz, pl);
          const Elem y1 = cutmax_update<Elem, PP>(v[i + 1], ke, be, kz, pl);
          if (real(i)) ta += y0;
          if (real(i + 1)) tb += y1;
        }
      };
      if (P == 0)
        dispatch_power(pl, sumy);
      else
        sumy(PowC<P>());
      const double tot = cluster_sum2<NTG>((double)ta + (double)tb, 0.0, cb, xround, rank, C, gtid).x;
      if (warp == 0) {
        const double total = tot - mph() * (double)cutmax_update<Elem, P>((Elem)cb->p3_w, ke, be, kz, pl);
        int st = cb->p3_st;
        const double rn = finish_total(total, st);
        __syncwarp();
        if (lane_of(gtid) == 0) {
          cb->p3_st = st;
          cb->bc.re = rn;
        }
      }
      bar1();
      re = (Elem)cb->bc.re;
    }
    PAM_TRACE(tr, 22);
    if (has_next) {
      if (dma) issue_upto(nch);  // T = 2: the second half was not issued by a hook
      ptx::mbar_wait_cta(bar_load, load_par);  // X(next) has landed
      load_par ^= 1u;
    } else {
      if (dma) ptx::bulk_wait_read_all();  // the previous Z store has read the buffer
      __syncthreads();
    }
    PAM_TRACE(tr, 23);

    // fused last pass: Y = z^3 (argmax), Z = Y * inv(sum Y) -> buffer, and
    // X(next) - K0(next) -> registers with its moments and TieWarning screen
    Elem bestv = -INFINITY;
    int besto = 0;  // register slot of the best element (compile-time immediates)
    Elem sa = 0, qa = 0;
    auto last_pass = [&](auto merged_c, auto pc) {
      constexpr bool MERGED = decltype(merged_c)::value;  // X(next) swapped in (compile-time: no per-slot branch)
      constexpr int PP = P > 0 ? P : decltype(pc)::value;
#pragma unroll
      for (int kk = 0; kk < NV; ++kk) {
        const int li0 = (kk * NTG + gtid) * VEC;
        Elem o[VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          const Elem y = cutmax_update<Elem, PP>(v[kk * VEC + j], ke, be, kz, pl);
          if (y > bestv) {  // slots in increasing element order: strict > keeps the lowest index
            bestv = y;
            besto = kk * VEC + j;
          }
          o[j] = y * re;
        }
        // TMA rows: n and the slice length are multiples of VEC, so a vector
        // slot is either all real or all phantom (phantom: K0(next) - K0(next) = 0)
        if (li0 < len) {
          V xn;
          if (MERGED) xn = *reinterpret_cast<const V*>(buf + li0);
          *reinterpret_cast<V*>(buf + li0) = *reinterpret_cast<const V*>(o);
          if (MERGED) {
            const Elem* xe = reinterpret_cast<const Elem*>(&xn);
#pragma unroll
            for (int j = 0; j < VEC; ++j) v[kk * VEC + j] = xe[j] - k0next;
          }
        } else if (MERGED) {
#pragma unroll
          for (int j = 0; j < VEC; ++j) v[kk * VEC + j] = Elem(0);
        }
        if (MERGED) {  // one (sum, sum of squares) pair: the last pass is the register peak
#pragma unroll
          for (int j = 0; j < VEC; ++j) {
            const Elem d = v[kk * VEC + j];
            sa += d;
            qa = fma_e(d, d, qa);
          }
        }
      }
    };
    if (P == 0) {
      if (has_next)
        dispatch_power(pl, [&](auto pc) { last_pass(BoolC<true>(), pc); });
      else
        last_pass(BoolC<false>(), PowC<0>());
    } else if (has_next) {
      last_pass(BoolC<true>(), PowC<P>());
    } else {
      last_pass(BoolC<false>(), PowC<P>());
    }
    ptx::fence_proxy_async_smem();  // Z writes -> visible to the TMA engine after the barrier
    PAM_TRACE(tr, 24);
    double best = (double)bestv;
    long long besti = base + (long long)(((besto / VEC) * NTG + gtid) * VEC + (besto % VEC));
    const int64_t zr = row;
    xch_push<NTG, kArgmax>((double)sa, (double)qa, best, besti, cb, xround, rank, C, gtid,
                           [&]() { store_all(zr); });
    if (has_next) screen_stash();  // the next row's input, in the exchange's idle time
    if (warp == 0) {
      const double2 rn = xch_wait<kArgmax>(best, besti, cb, xround, C, gtid);
      const int st = cb->p3_st;
      __syncwarp();
      if (has_next) {  // argmax / status: deferred to the next row's first exchange wait
        if (gtid == 0) {
          cb->p3_S = rn.x;
          cb->p3_Q = rn.y;
          cb->fin_row = row;
          cb->fin_st = st;
          cb->fin_best = besti;
          cb->fin_pending = 1;
        }
        __syncwarp();
      } else {
        finish_row(row, st, besti, lrow);
      }
    } else {
      ++xround;
    }
    PAM_TRACE(tr, 6 + 2 * (T - 1));
    k0_cur = k0next;
    PAM_TRACE(tr, 21);
  }

  // ---- TieWarning rows the screen left undecided: exact fp64 top-2 ----------
  __syncthreads();
  const int unc = cb->unc_n;
  if (unc > 0 && a.status) {
    const int64_t cnt = unc <= 16 ? unc : (a.B - cid + ncl - 1) / ncl;  // overflow: every row of the cluster
    for (int64_t j = 0; j < cnt; ++j) {
      const int64_t r = unc <= 16 ? cb->unc_rows[j] : cid + j * ncl;
      const Elem* xr = X + r * a.ldx + base;
      double m1 = -HUGE_VAL, m2 = -HUGE_VAL;
      for (int i = gtid; i < len; i += NTG) top2_add(m1, m2, (double)xr[i]);
      const double2 t = cluster_top2<NTG>(m1, m2, cb, xround, rank, C, gtid);
      if (rank == 0 && gtid == 0) {
        const int s0 = a.status[r];
        if ((s0 & 0xff) == PAM_OK) a.status[r] = (s0 & ~PAM_ROW_FLAG_TIE) | (t.x - t.y < 1e-9 ? PAM_ROW_FLAG_TIE : 0);
      }
    }
  }
  if (dma) ptx::bulk_wait_all();  // Z stores complete before the CTA retires
  ptx::cluster_sync();            // no CTA leaves while a peer may still push into its shared memory
}

}  // namespace pam
