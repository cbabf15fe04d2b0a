// nucleus_kernel.cuh — fused Beta-cut nucleus sampler (Alg. 3, PAPER.md:216-239;
// SPEC.md:437-445) and its Gumbel-max sibling, with the
// top-p membership test of SPEC.md:440,464 fused in.
//
// Per row, one cluster:
//   1. TMA-load the logit slice into shared memory (kept there: x is needed again).
//   2. Registers: xt_i = x_i + G_i, G_i = u_i^(1/alpha) (Beta) or -log(-log u_i)
//      (Gumbel), u_i from Philox4x32-10 keyed by seed ^ row.
//      Two consecutive elements share one Philox call.  Local max of x.
//   3. input_pass + cutmax_iterate on xt (identical code to the CutMax kernel).
//   4. token = argmax Z, all-gathered across the cluster together with x_tok
//      and max(x) (one 32-byte record per CTA pushed to every CTA).
//   5. One pass over x (shared memory): e = exp(x - max x), sums of e and of
//      e over {x_k > x_tok}; one exchange; inside = above < p * total.
// The noise and the nucleus exp use the table-driven log / exp of
// pam_scalar.h (tables copied to shared memory once per CTA).
// The noise is generated on chip and never stored; HBM traffic is 8n bytes
// read per row plus 5 bytes written (+ 8n if the one-hot output is requested).
#pragma once

#include "cutmax_kernel.cuh"

namespace pam {

// shared memory after the row buffer: ControlBlock, then the log / exp tables
constexpr int kSamplerTabOffset = ((int)sizeof(ControlBlock) + 15) / 16 * 16;
constexpr int kSamplerTabBytes = 384 * 8;

struct SamplerArgs {
  const double* x;
  double* onehot;  // nullable
  int32_t* token;
  uint8_t* inside;
  int32_t* status;
  int64_t ldx, ld_onehot, B, n;
  int32_t L;
  int32_t ctrl_offset;
  double inv_alpha;
  double p_nucleus;
  uint64_t seed, draw;
  int32_t tma;  // 1: TMA bulk load (16-byte aligned rows), 0: thread copy
  double inv_n;
  long long* trace;  // debug phase stamps (trace builds)
  RowParams rp;
};

template <int NT, int E, int P, bool GUMBEL, bool STOP = false>
__global__ void __launch_bounds__(NT, 1) sampler_rows_kernel(const SamplerArgs a) {
  static_assert(!STOP || P == 0, "early stopping runs on the generic flow");
  constexpr int VEC = 2;
  constexpr int NV = E / VEC;
  constexpr int NW = NT / 32;
  static_assert(E % VEC == 0, "E must be even");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* buf = reinterpret_cast<double*>(smem_raw);
  ControlBlock* cb = reinterpret_cast<ControlBlock*>(smem_raw + a.ctrl_offset);
  // log / exp tables (pam_scalar.h log_t_core / exp_t_core) in shared memory:
  // invc[128], logc[128], e2[128] right after the control block
  double* tabs = reinterpret_cast<double*>(smem_raw + a.ctrl_offset + kSamplerTabOffset);

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
  const uint32_t bar_load = ptx::smem_addr(&cb->mb_load);
  const uint32_t load_bytes = (uint32_t)len * 8u;
  const uint64_t policy = ptx::policy_evict_first();

  for (int i = tid; i < 128; i += NT) {
    tabs[i] = pam_d_logt_invc[i];
    tabs[128 + i] = pam_d_logt_logc[i];
    tabs[256 + i] = pam_d_expt_e2[i];
  }
  if (tid == 0) {
    cb->unc_n = 0;
    ptx::mbar_init(bar_load, 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_x[0]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_x[1]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_g), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_t[0]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_t[1]), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[0]), C * kXchBytes);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[1]), C * kXchBytes);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_g), C * 32u);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_t[0]), C * 16u);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_t[1]), C * 16u);
  }
  ptx::cluster_sync();

  uint32_t xround = 0, load_par = 0, g_par = 0, t2_ph = 0;
  double v[E];

  int64_t lrow = 0;
  for (int64_t row = cid; row < a.B; row += ncl, ++lrow) {
#ifdef PAM_TRACE_BUILD
    long long* tr =
        (a.trace && lrow < kTraceRows) ? a.trace + ((int64_t)blockIdx.x * kTraceRows + lrow) * kTraceEvents : nullptr;
#else
    long long* tr = nullptr;
#endif
    const int gtid = tid;
    PAM_TRACE(tr, 0);
    const double* xrow = a.x + row * a.ldx;
    const double K0 = __ldg(xrow);
    __syncthreads();  // landing buffer and wred of the previous row retired
    if (a.tma && tid == 0) {
      ptx::mbar_arrive_expect_tx(bar_load, load_bytes);
      const unsigned char* src = reinterpret_cast<const unsigned char*>(xrow + base);
      for (uint32_t off = 0; off < load_bytes; off += 32768u) {
        const uint32_t nb = (load_bytes - off) < 32768u ? (load_bytes - off) : 32768u;
        ptx::bulk_g2s(ptx::smem_addr(buf) + off, src + off, nb, bar_load, policy);
      }
    }
    // Noise first (independent of x), then wait for the data.
    const uint64_t key = a.seed ^ (uint64_t)row;
    if (GUMBEL || a.inv_alpha <= 19.0) {  // branch-free forms (bit-identical on this domain)
      // two vector slots (four elements) per step, their chains written side by
      // side so the scheduler keeps four independent log/exp chains in flight
#pragma unroll
      for (int k = 0; k < NV; k += 2) {
        const int k1 = k + 1 < NV ? k + 1 : k;
        const int li0 = (k * NT + tid) * VEC, li1 = (k1 * NT + tid) * VEC;
        double u[4];
        uniform_pair(key, a.draw, (uint64_t)(base + li0) >> 1, &u[0], &u[1]);
        uniform_pair(key, a.draw, (uint64_t)(base + li1) >> 1, &u[2], &u[3]);
        double g[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) g[q] = log_t_core(u[q], tabs, tabs + 128);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          g[q] = GUMBEL ? -log_t_core(-g[q], tabs, tabs + 128) : exp_t_core(g[q] * a.inv_alpha, tabs + 256);
        if (!GUMBEL && a.inv_alpha == 1.0) {
#pragma unroll
          for (int q = 0; q < 4; ++q) g[q] = u[q];
        }
        v[k * VEC + 0] = g[0];
        v[k * VEC + 1] = g[1];
        v[k1 * VEC + 0] = g[2];
        v[k1 * VEC + 1] = g[3];
      }
    } else {
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const int li0 = (k * NT + tid) * VEC;
        double u0, u1;
        uniform_pair(key, a.draw, (uint64_t)(base + li0) >> 1, &u0, &u1);
        v[k * VEC + 0] = GUMBEL ? gumbel_from_u(u0) : beta_icdf(u0, a.inv_alpha);
        v[k * VEC + 1] = GUMBEL ? gumbel_from_u(u1) : beta_icdf(u1, a.inv_alpha);
      }
    }
    PAM_TRACE(tr, 1);
    if (a.tma) {
      ptx::mbar_wait_cta(bar_load, load_par);
      load_par ^= 1u;
    } else {
      for (int i = tid; i < len; i += NT) buf[i] = __ldg(xrow + base + i);
      __syncthreads();
    }
    double xmax = -HUGE_VAL;
    // TieWarning screen of x~ = x + G (the vector CutMax sees): top-2 high
    // words on the FP32 pipe (cutmax_kernel.cuh: tie_decide), exact re-scan of
    // undecided rows at the end of the kernel
    float t1 = -INFINITY, t2 = -INFINITY;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int li0 = (k * NT + tid) * VEC;
      if (li0 + VEC <= len) {
        const double2 t = *reinterpret_cast<const double2*>(buf + li0);
        v[k * VEC + 0] = t.x + v[k * VEC + 0];  // Alg. 3 line 5: x~ = x + G
        v[k * VEC + 1] = t.y + v[k * VEC + 1];
        xmax = fmax(xmax, fmax(t.x, t.y));
        top2f_add(t1, t2, hiword_f(v[k * VEC + 0]));
        top2f_add(t1, t2, hiword_f(v[k * VEC + 1]));
      } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          if (li0 + j < len) {
            const double xv = buf[li0 + j];
            v[k * VEC + j] = xv + v[k * VEC + j];
            xmax = fmax(xmax, xv);
            top2f_add(t1, t2, hiword_f(v[k * VEC + j]));
          } else {
            v[k * VEC + j] = K0;  // phantom (see cutmax_iterate)
          }
        }
      }
    }

    PAM_TRACE(tr, 2);
    double rnorm = 1.0;
    long long unused_argmax;
    const double2 part = input_pass<double, E>(v, K0);
    const double2 rin = cluster_sum2<NT>(part.x, part.y, cb, xround, rank, C, tid,
                                         KeyPush{true, fkey(t1), fkey(t2), (uint32_t)(lrow & 1)});
    auto final_xch = [&](double sy, double& bv, long long& bi) -> double {
      return cluster_reduce<NT, false>(sy, 0.0, bv, bi, cb, xround, rank, C, tid).x;
    };
    auto hooks = make_hooks(false, [](int) {}, [](int) {}, final_xch);
    int st = cutmax_iterate<double, NT, E, P, false, decltype(hooks), STOP>(
        v, rin.x, rin.y, K0, len, (double)((int64_t)C * NT * E - n), a.rp, a.inv_n, (double)n, cb, xround, rank, C,
        tid, base, nullptr, rnorm, unused_argmax, hooks, nullptr);

    PAM_TRACE(tr, 3);
    // token = argmax of Y^(T+1) before the normalisation (pin A7, oracle.c
    // orc_cutmax: Y * inv(sum Y) could round a near-tie into an exact one);
    // the optional one-hot output is Z = Y * rnorm.  Each thread tracks its
    // best register slot (compile-time immediates), x_tok is read once from
    // the slot that wins; warps and the cluster combine with REDUX (warp_argmax).
    double best = -HUGE_VAL;
    int besto = -1;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int li0 = (k * NT + tid) * VEC;
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        const double y = v[k * VEC + j];
        if (li0 + j < len) {
          if (y > best) {  // slots in increasing element order: strict > keeps the lowest index
            best = y;
            besto = k * VEC + j;
          }
          if (a.onehot) a.onehot[row * a.ld_onehot + base + li0 + j] = y * rnorm;
        }
      }
    }
    long long besti = 0x7fffffffffffffffLL;
    double bestx = 0.0;
    if (besto >= 0) {
      const int li = ((besto / VEC) * NT + tid) * VEC + (besto % VEC);
      besti = base + li;
      bestx = buf[li];
    }
    // warp: winner (value desc, index asc), its x, and max x
    auto argmax_with_x = [&](double& bv, long long& bi, double& bx) {
      const long long mine = bi;
      warp_argmax(bv, bi);
      const unsigned who = __ballot_sync(0xffffffffu, mine == bi);
      bx = __shfl_sync(0xffffffffu, bx, who ? __ffs(who) - 1 : 0);
    };
    auto max_all = [&](double m) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
      return m;
    };
    argmax_with_x(best, besti, bestx);
    xmax = max_all(xmax);
    if (lane == 0) cb->wred[warp] = make_double2(best, __longlong_as_double(besti));
    __shared__ double2 wx[32];
    if (lane == 0) wx[warp] = make_double2(bestx, xmax);
    __syncthreads();
    if (warp == 0) {
      const double2 w = (lane < NW) ? cb->wred[lane] : make_double2(-HUGE_VAL, __longlong_as_double(0x7fffffffffffffffLL));
      const double2 wxx = (lane < NW) ? wx[lane] : make_double2(0.0, -HUGE_VAL);
      best = w.x;
      besti = __double_as_longlong(w.y);
      bestx = wxx.x;
      argmax_with_x(best, besti, bestx);
      xmax = max_all(wxx.y);
      if (lane < (int)C) {  // all-gather: 32-byte record to every CTA
        const uint32_t bar = ptx::mapa(ptx::smem_addr(&cb->mb_g), (uint32_t)lane);
        ptx::st_async_b64x2(ptx::mapa(ptx::smem_addr(&cb->gat[rank][0]), (uint32_t)lane),
                            (uint64_t)__double_as_longlong(best), (uint64_t)besti, bar);
        ptx::st_async_f64x2(ptx::mapa(ptx::smem_addr(&cb->gat[rank][1]), (uint32_t)lane), bestx, xmax, bar);
      }
    }
    ptx::mbar_wait_cluster(ptx::smem_addr(&cb->mb_g), g_par);
    g_par ^= 1u;
    if (tid == 0) ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_g), C * 32u);  // arm next row
    {
      const bool have = lane < (int)C;
      const double2 r0 = have ? cb->gat[lane][0] : make_double2(-HUGE_VAL, __longlong_as_double(0x7fffffffffffffffLL));
      const double2 r1 = have ? cb->gat[lane][1] : make_double2(0.0, -HUGE_VAL);
      best = r0.x;
      besti = __double_as_longlong(r0.y);
      bestx = r1.x;
      argmax_with_x(best, besti, bestx);
      xmax = max_all(r1.y);
    }

    PAM_TRACE(tr, 4);
    // nucleus membership: sum over x_k > x_tok of exp(x_k - max) vs p * total
    double tot = 0.0, above = 0.0;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int li0 = (k * NT + tid) * VEC;
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        if (li0 + j < len) {
          const double xv = buf[li0 + j];
          // exp(x - max) for x - max >= -700 (bit-identical branch-free form); below,
          // exp < 1e-304 cannot change the totals, which include exp(0) = 1
          const double d = xv - xmax;
          const double e = d >= -700.0 ? exp_t_core(d, tabs + 256) : (d == d ? 0.0 : d);
          tot += e;
          if (xv > bestx) above += e;
        }
      }
    }
    const double2 ta = cluster_sum2<NT>(tot, above, cb, xround, rank, C, tid);
    PAM_TRACE(tr, 5);
    if (warp == 0) {
      const int2 kk = top2k_wait(cb, (uint32_t)(lrow & 1), t2_ph, C, tid);
      const int td = tie_decide<double>(st, kk.x, kk.y);
      if (rank == 0 && tid == 0) {
        if (a.token) a.token[row] = (st == PAM_OK) ? (int32_t)besti : -1;
        if (a.inside) a.inside[row] = (st == PAM_OK && ta.y < a.p_nucleus * ta.x) ? 1 : 0;
        if (a.status) a.status[row] = st | (td == 1 ? PAM_ROW_FLAG_TIE : 0);
      }
      if (td == 2 && tid == 0) {  // undecided (cluster-uniform): settled below
        const int q = cb->unc_n;
        if (q < 16) cb->unc_rows[q] = row;
        cb->unc_n = q + 1;
      }
    }
  }

  // ---- TieWarning rows the screen left undecided: exact top-2 of x + G -------
  // (rare: the two largest perturbed logits share their high word).  The noise
  // is regenerated with the same functions as above, element pair by pair.
  __syncthreads();
  const int unc = cb->unc_n;
  if (unc > 0 && a.status) {
    const int64_t cnt = unc <= 16 ? unc : (a.B - cid + ncl - 1) / ncl;  // overflow: every row of the cluster
    for (int64_t j = 0; j < cnt; ++j) {
      const int64_t r = unc <= 16 ? cb->unc_rows[j] : cid + j * ncl;
      const double* xr = a.x + r * a.ldx + base;
      const uint64_t key = a.seed ^ (uint64_t)r;
      double m1 = -HUGE_VAL, m2 = -HUGE_VAL;
      for (int i = 2 * tid; i < len; i += 2 * NT) {
        double u0, u1;
        uniform_pair(key, a.draw, (uint64_t)(base + i) >> 1, &u0, &u1);
        const double us[2] = {u0, u1};
        for (int q = 0; q < 2 && i + q < len; ++q) {
          double g;
          g = GUMBEL ? gumbel_from_u(us[q]) : beta_icdf(us[q], a.inv_alpha);
          top2_add(m1, m2, xr[i + q] + g);
        }
      }
      const double2 t = cluster_top2<NT>(m1, m2, cb, xround, rank, C, tid);
      if (rank == 0 && tid == 0) {
        const int s0 = a.status[r];
        if ((s0 & 0xff) == PAM_OK) a.status[r] = (s0 & ~PAM_ROW_FLAG_TIE) | (t.x - t.y < 1e-9 ? PAM_ROW_FLAG_TIE : 0);
      }
    }
  }
  ptx::cluster_sync();
}

}  // namespace pam
