// cutmax_kernel.cuh — fused, row-resident batched CutMax for sm_100a.
//
// Replaces core.cutmax / core.cutmaxStep (Alg. 1).
//
// Geometry.  One logit row is owned by one thread-block cluster of C CTAs
// (C = 1..16).  CTA `rank` owns the contiguous slice [rank*L, min(n,(rank+1)*L)).
// A CTA runs G independent "row groups" of NTG threads each (named barriers
// 1..G, own mbarriers, own landing buffer): group g of cluster c processes rows
// c*G + g, c*G + g + ncl*G, ...  While one group sits in a cluster exchange or
// streams its Z out, the other group's fp64 passes keep the SM busy.
// Each thread of a group keeps E elements of its slice in registers for all T
// iterations: HBM is read once (1-D TMA bulk copy into the group's shared
// memory landing buffer, prefetched one row ahead) and written once (128-bit
// streaming stores).
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
// Exchange.  Each warp butterfly-reduces its lanes and pushes its partial into
// slot (rank, warp) of every CTA of the cluster with st.async (DSMEM),
// completing on the destination group's mbarrier; every warp then sums the
// same C*NW slots in the same order.  xor-butterflies leave bit-identical sums
// in every lane (IEEE addition is commutative), so all CTAs compute identical
// mu and s2 without a broadcast.  The argmax candidate is gathered to rank 0.
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
  int32_t L;             // slice length per CTA (elements)
  int32_t buf_bytes;     // landing-buffer bytes per group (0 without TMA)
  int32_t ctrl_offset;   // byte offset of the first group's control block
  int32_t tma;           // 1: TMA bulk loads + 128-bit stores (16-byte aligned rows), 0: scalar path
  double inv_n;          // 1/n
  long long* trace;      // debug: per-CTA phase timestamps (pam_set_trace_buffer), normally null
  int64_t stagger;       // start offset (SM cycles) spread over clusters / groups to de-phase them
  int32_t debug_flags;   // dev experiments: 1 = skip Z stores
  RowParams rp;
};

// One 32-byte exchange record per (cluster rank): partial sums (a, b) and an
// argmax candidate (value, index) used by the last exchange of a row.
struct __align__(16) XchRecord {
  double2 ab;
  double2 cand;  // (value, index bits)
};

struct __align__(16) ControlBlock {
  XchRecord xch[2][16];  // exchange slots per cluster rank, double-buffered by round parity
  double2 wred[32];      // per-warp partial sums (CTA pre-reduction; sampler token gather)
  double2 wcand[32];     // per-warp argmax candidates
  double2 gat[16][2];    // all-gather records (sampler: token candidate + max x)
  unsigned long long mb_load;
  unsigned long long mb_x[2];
  unsigned long long mb_g;
};

// Debug phase tracing: thread 0 of group 0 of each CTA stamps clock64() at
// phase boundaries of its first kTraceRows rows (tools/trace.py reads them).
constexpr int kTraceRows = 8, kTraceEvents = 32;
#define PAM_TRACE(tr, k)                                   \
  do {                                                     \
    if ((tr) != nullptr && gtid == 0) (tr)[k] = clock64(); \
  } while (0)

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

// Named barrier for the NTG threads of group g (barrier 0 is __syncthreads).
template <int NTG>
__device__ __forceinline__ void group_sync(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(NTG) : "memory");
}

// Strict alternation of the fp64 element passes of the G=2 row groups of a CTA.
// A group holds the token while it streams its slice through the fp64 pipe and
// hands it over before waiting in its cluster exchange, so one group's
// exchange latency overlaps the other group's pass.  Named barrier 3+g carries
// the token to group g (the giver arrives, the taker syncs: 2*NTG threads).
// Group 0 starts with the token; every group takes and gives exactly
// K*(T+1) times except that group 0 skips its first take and group 1 its last
// give, which keeps the barrier arrivals balanced.  G=1: no-ops.
template <int NTG, int G>
struct PassToken {
  int g;
  int64_t left;  // gives still to perform
  bool skip_take;
  __device__ __forceinline__ PassToken(int g_, int64_t total) : g(g_), left(total - (g_ == 1 ? 1 : 0)), skip_take(g_ == 0) {}
  __device__ __forceinline__ void take() {
    if (G == 2) {
      if (skip_take) {
        skip_take = false;
      } else {
        asm volatile("bar.sync %0, %1;" ::"r"(3 + g), "r"(2 * NTG) : "memory");
      }
    }
  }
  __device__ __forceinline__ void give() {
    if (G == 2 && left > 0) {
      --left;
      asm volatile("bar.arrive %0, %1;" ::"r"(3 + (g ^ 1)), "r"(2 * NTG) : "memory");
    }
  }
};

__device__ __forceinline__ void butterfly_sum2(double& a, double& b) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, m);
    b += __shfl_xor_sync(0xffffffffu, b, m);
  }
}

__device__ __forceinline__ bool cand_better(double v, long long i, double bv, long long bi) {
  return (v > bv) || (v == bv && i < bi);
}

// xor-butterfly over the low `width` lanes' groups (width a power of two <= 32):
// every lane ends with the combination of its aligned width-group, and because
// IEEE addition / the argmax rule are commutative, all lanes of a group hold
// bit-identical values.
template <int WIDTH>
__device__ __forceinline__ void bfly_sum2(double& a, double& b) {
#pragma unroll
  for (int m = WIDTH / 2; m > 0; m >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, m);
    b += __shfl_xor_sync(0xffffffffu, b, m);
  }
}

template <int WIDTH>
__device__ __forceinline__ void bfly_argmax(double& best, long long& besti) {
#pragma unroll
  for (int m = WIDTH / 2; m > 0; m >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, m);
    const long long oi = __shfl_xor_sync(0xffffffffu, besti, m);
    if (cand_better(ov, oi, best, besti)) {
      best = ov;
      besti = oi;
    }
  }
}

__device__ __forceinline__ void butterfly_argmax(double& best, long long& besti) { bfly_argmax<32>(best, besti); }

// ---------------------------------------------------------------------------
// Cluster-wide reduction over one row group: sums of (a, b) and, when ARGMAX,
// the lexicographic (value desc, index asc) maximum of (best, besti).  All NTG
// threads of group g must call it; every thread returns the cluster result,
// bit-identical in every CTA.
//   warp butterfly -> per-warp partial in smem -> named barrier -> warp 0
//   combines the NW partials and pushes one 32-byte record into slot [rank] of
//   every CTA (st.async, complete_tx on the destination's mbarrier) -> every
//   warp combines the C records in the same fixed butterfly order.
template <int NTG, bool ARGMAX>
__device__ __forceinline__ double2 cluster_reduce(double a, double b, double& best, long long& besti, ControlBlock* cb,
                                                  uint32_t& round, uint32_t rank, uint32_t C, int g, int gtid,
                                                  long long* tr = nullptr) {
  constexpr int NW = NTG / 32;
  const int lane = gtid & 31, warp = gtid >> 5;
  bfly_sum2<32>(a, b);
  if (ARGMAX) bfly_argmax<32>(best, besti);
  if (lane == 0) {
    cb->wred[warp] = make_double2(a, b);
    if (ARGMAX) cb->wcand[warp] = make_double2(best, __longlong_as_double(besti));
  }
  group_sync<NTG>(g);
  const uint32_t par = round & 1u, ph = (round >> 1) & 1u;
  if (warp == 0) {
    const double2 w = cb->wred[lane & (NW - 1)];
    double ca = w.x, cbv = w.y;
    bfly_sum2<NW>(ca, cbv);
    double cv = -HUGE_VAL;
    long long ci = 0x7fffffffffffffffLL;
    if (ARGMAX) {
      const double2 wc = cb->wcand[lane & (NW - 1)];
      cv = wc.x;
      ci = __double_as_longlong(wc.y);
      bfly_argmax<NW>(cv, ci);
    }
    if (lane < (int)C) {
      const uint32_t bar = ptx::mapa(ptx::smem_addr(&cb->mb_x[par]), (uint32_t)lane);
      ptx::st_async_f64x2(ptx::mapa(ptx::smem_addr(&cb->xch[par][rank].ab), (uint32_t)lane), ca, cbv, bar);
      ptx::st_async_b64x2(ptx::mapa(ptx::smem_addr(&cb->xch[par][rank].cand), (uint32_t)lane),
                          (uint64_t)__double_as_longlong(cv), (uint64_t)ci, bar);
    }
  }
  PAM_TRACE(tr, 24);
  ptx::mbar_wait_cta(ptx::smem_addr(&cb->mb_x[par]), ph);
  PAM_TRACE(tr, 25);
  if (gtid == 0) ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[par]), C * 32u);  // arm round+2
  const int src = lane & 15;
  const bool have = src < (int)C;
  const XchRecord rec = cb->xch[par][have ? src : 0];
  a = have ? rec.ab.x : 0.0;
  b = have ? rec.ab.y : 0.0;
  bfly_sum2<16>(a, b);
  if (ARGMAX) {
    best = have ? rec.cand.x : -HUGE_VAL;
    besti = have ? __double_as_longlong(rec.cand.y) : 0x7fffffffffffffffLL;
    bfly_argmax<16>(best, besti);
  }
  PAM_TRACE(tr, 26);
  ++round;
  return make_double2(a, b);
}

template <int NTG>
__device__ __forceinline__ double2 cluster_sum2(double a, double b, ControlBlock* cb, uint32_t& round, uint32_t rank,
                                                uint32_t C, int g, int gtid, long long* tr = nullptr) {
  double bv = 0.0;
  long long bi = 0;
  return cluster_reduce<NTG, false>(a, b, bv, bi, cb, round, rank, C, g, gtid, tr);
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

__device__ __forceinline__ void moments_from_sums(double S, double Q, double inv_n, double& dm, double& s2) {
  dm = S * inv_n;
  s2 = fma(-dm, dm, Q * inv_n);
}

// ---------------------------------------------------------------------------
// CutMax on a register-resident row slice (one row group).
//
// On entry v[] holds the group's slice: `len` real elements followed by
// phantom elements (slots beyond the slice) that the caller filled with K0.
// Phantoms keep every pass free of per-element predicates: all phantoms of the
// row carry one common value w_t (they start at K0 and get the same updates),
// tracked here as a scalar, and their total contribution m*w (m = number of
// phantoms in the cluster) is subtracted from the cluster sums.
//
// With ARGMAX, the last iteration's pass also tracks the argmax of Y^(T+1)
// (pin A7: equals argmax Z for the positive normaliser) and the last exchange
// carries it, so no separate gather is needed.  When the caller filled the
// phantoms with x[0] and K0 = x[0], phantoms are exact copies of element 0 and
// can never beat it (equal value, larger index), so no predicate is needed.
//
// On exit v holds Y^(T+1) (shift 0) and rnorm the normaliser inv(sum Y) (1
// when PAM_F_NO_NORMALIZE).  Returns the row status, identical in every CTA.
struct NoOp {
  __device__ __forceinline__ void operator()() const {}
};

template <typename Elem, int NTG, int G, int E, int P, bool ARGMAX, typename AfterFirstXchg = NoOp>
__device__ __forceinline__ int cutmax_core(Elem (&v)[E], PassToken<NTG, G>& tok, const double K0, const double mphantom,
                                           const RowParams& rp, const double inv_n, ControlBlock* cb,
                                           uint32_t& xround, const uint32_t rank, const uint32_t C, const int g,
                                           const int gtid, const int64_t gbase, double* stats_row, double& rnorm,
                                           long long& argmax_out, long long* tr = nullptr,
                                           const AfterFirstXchg& after_first_xchg = AfterFirstXchg()) {
  using Tr = ElemTraits<Elem>;
  constexpr int VEC = Tr::VEC;
  constexpr double kGuard = sizeof(Elem) == 8 ? 16.0 : 2.0;  // cancellation guard (see header)
  // kernel parameters the per-iteration scalar chain needs, held in registers
  // (the exchanges' memory clobbers would otherwise re-load them every round)
  const int T = rp.T;
  const bool normalize = !(rp.flags & PAM_F_NO_NORMALIZE);
  const bool poly_invsqrt = rp.invsqrt_mode == PAM_MODE_POLY;
  const double eps_var = rp.eps_var;
  int st = PAM_OK;
  rnorm = 1.0;
  argmax_out = -1;

  // exact second pass about dm when the shifted one-pass moments cancelled
  auto guard = [&](double S, double Q, double w, double& dm, double& s2) {
    moments_from_sums(S, Q, inv_n, dm, s2);
    if (st == PAM_OK && isfinite(Q) && Q * inv_n > kGuard * s2) {
      const Elem dme = (Elem)dm;
      Elem q2a = 0, q2b = 0;
#pragma unroll
      for (int i = 0; i < E; i += 2) {
        const Elem d0 = v[i] - dme, d1 = v[i + 1] - dme;
        q2a = fma_e(d0, d0, q2a);
        q2b = fma_e(d1, d1, q2b);
      }
      const double2 r2 = cluster_sum2<NTG>((double)q2a + (double)q2b, 0.0, cb, xround, rank, C, g, gtid);
      const Elem dw = (Elem)w - dme;
      s2 = (r2.x - mphantom * (double)dw * (double)dw) * inv_n;
    }
  };

  // per-iteration constants, loaded ahead of the exchange they follow
  double c_inv = rp.inv_c[0], knext = rp.kshift[1];
  int pcur = rp.p[0];

  // ---- input pass: shift by K0 (phantoms hold K0 -> contribute exactly 0) ---
  double dm, s2;
  {
    const Elem k0 = (Elem)K0;
    Elem sa = 0, sb = 0, qa = 0, qb = 0;
#pragma unroll
    for (int i = 0; i < E; i += 2) {
      const Elem d0 = v[i] - k0, d1 = v[i + 1] - k0;
      v[i] = d0;
      v[i + 1] = d1;
      sa += d0;
      sb += d1;
      qa = fma_e(d0, d0, qa);
      qb = fma_e(d1, d1, qb);
    }
    PAM_TRACE(tr, 3);
    tok.give();
    const double2 r =
        cluster_sum2<NTG>((double)sa + (double)sb, (double)qa + (double)qb, cb, xround, rank, C, g, gtid, tr);
    PAM_TRACE(tr, 4);
    if (T == 1) after_first_xchg();
    if (!isfinite(r.x) || !isfinite(r.y)) st = PAM_ERR_NON_FINITE;
    guard(r.x, r.y, 0.0, dm, s2);
    PAM_TRACE(tr, 28);
  }
  double kcur = K0;
  Elem w = 0;  // phantom value (shifted representation)

  // ---- T iterations; the last one (no variance; argmax) is peeled -----------
  double total = 0.0;
  for (int t = 0; t < T; ++t) {
    const double mu = kcur + dm;
    // status: first failure wins (branch-free on the common path)
    const bool bad_range = !isfinite(mu) || !isfinite(s2);
    st = (st != PAM_OK) ? st : (bad_range ? PAM_ERR_RANGE : (s2 < eps_var ? PAM_ERR_DEGENERATE_INPUT : PAM_OK));
    if (stats_row) {
      stats_row[t * 2 + 0] = mu;
      stats_row[t * 2 + 1] = s2;
    }
    if (t == 0) PAM_TRACE(tr, 29);
    double inv_sigma;
    if (!poly_invsqrt) {
      inv_sigma = rsqrt(s2);  // ~1 ulp; identical in every CTA of the cluster
    } else {
      const pam_approx_config& ac = rp.invsqrt[t];
      inv_sigma = 0.0;
      if (st == PAM_OK) {
        const int rs = invsqrt_rescaled(s2, ac.iterations, ac.rescale, ac.scale_log2, ac.lo, ac.hi, &inv_sigma);
        if (rs) st = rs;
      }
    }
    if (t == 0) PAM_TRACE(tr, 30);
    const double kd = (st == PAM_OK) ? inv_sigma * c_inv : 0.0;
    const double bd = fma(-dm, kd, 1.0);
    const Elem ke = (Elem)kd, be = (Elem)bd, kn = (Elem)(-knext);
    const int p = pcur;
    if (t == 0) PAM_TRACE(tr, 27);
    w = cutmax_update<Elem, P>(w, ke, be, kn, p);
    const double kthis = knext;
    tok.take();
    if (t + 1 < T) {
      Elem sa = 0, sb = 0, qa = 0, qb = 0;
#pragma unroll
      for (int i = 0; i < E; i += 2) {
        const Elem d0 = cutmax_update<Elem, P>(v[i], ke, be, kn, p);
        const Elem d1 = cutmax_update<Elem, P>(v[i + 1], ke, be, kn, p);
        v[i] = d0;
        v[i + 1] = d1;
        sa += d0;
        sb += d1;
        qa = fma_e(d0, d0, qa);
        qb = fma_e(d1, d1, qb);
      }
      c_inv = rp.inv_c[t + 1];  // prefetch next iteration's constants
      knext = rp.kshift[t + 2];
      pcur = rp.p[t + 1];
      PAM_TRACE(tr, 5 + 2 * t);
      tok.give();
      const double2 r =
          cluster_sum2<NTG>((double)sa + (double)sb, (double)qa + (double)qb, cb, xround, rank, C, g, gtid);
      PAM_TRACE(tr, 6 + 2 * t);
      // deferred work (the next-row prefetch into the landing buffer): the
      // previous row's Z bulk store drains at the HBM write rate and holds the
      // buffer for several exchanges, so wait until the third exchange
      if (t == 1 || (t == 0 && T == 2)) after_first_xchg();
      const double wd = (double)w;
      guard(r.x - mphantom * wd, r.y - mphantom * wd * wd, wd, dm, s2);
      kcur = kthis;
    } else {
      Elem sa = 0, sb = 0;
      Elem bestv = -INFINITY;
      int besto = 0;  // register slot of the best element (compile-time immediates)
#pragma unroll
      for (int i = 0; i < E; i += 2) {
        const Elem d0 = cutmax_update<Elem, P>(v[i], ke, be, kn, p);
        const Elem d1 = cutmax_update<Elem, P>(v[i + 1], ke, be, kn, p);
        v[i] = d0;
        v[i + 1] = d1;
        sa += d0;
        sb += d1;
        if (ARGMAX) {  // slots in increasing element order: strict > keeps the lowest index
          if (d0 > bestv) { bestv = d0; besto = i; }
          if (d1 > bestv) { bestv = d1; besto = i + 1; }
        }
      }
      double best = (double)bestv;
      long long besti = gbase + (long long)(((besto / VEC) * NTG + gtid) * VEC + (besto % VEC));
      PAM_TRACE(tr, 5 + 2 * t);
      tok.give();
      const double2 r = cluster_reduce<NTG, ARGMAX>((double)sa + (double)sb, 0.0, best, besti, cb, xround, rank, C,
                                                    g, gtid);
      PAM_TRACE(tr, 6 + 2 * t);
      total = r.x - mphantom * (double)w;  // kshift[T] == 0: v holds Y^(T+1) itself
      argmax_out = besti;
    }
  }

  if (st == PAM_OK && !isfinite(total)) st = PAM_ERR_RANGE;
  if (st == PAM_OK && normalize) {
    if (!(total > 0.0)) {
      st = PAM_ERR_RANGE;  // Z must be a distribution (pin A7)
    } else if (rp.inv_mode == PAM_MODE_POLY) {
      const pam_approx_config& ac = rp.inv;
      const int rs = inv_rescaled(total, ac.iterations, ac.rescale, ac.scale_log2, ac.lo, ac.hi, &rnorm);
      if (rs) st = rs;
    } else {
      rnorm = 1.0 / total;
    }
  }
  return st;
}

// Resident CTAs per SM the register budget should allow (launch-bounds hint).
template <typename Elem, int NT, int E>
constexpr int min_blocks_for() {
  constexpr int regs = E * (int)sizeof(Elem) / 4 + 48;
  constexpr int b = 65536 / (NT * regs);
  return b < 1 ? 1 : (b > 8 ? 8 : b);
}

// ---------------------------------------------------------------------------
template <typename Elem, int NTG, int G, int E, int P>
__global__ void __launch_bounds__(NTG* G, (min_blocks_for<Elem, NTG * G, E>())) cutmax_rows_kernel(const CutmaxArgs a) {
  using Tr = ElemTraits<Elem>;
  using V = typename Tr::V;
  constexpr int VEC = Tr::VEC;
  constexpr int NV = E / VEC;
  constexpr int NW = NTG / 32;
  static_assert(E % VEC == 0 && E % 2 == 0, "E must be a multiple of the vector width");
  static_assert(NTG % 32 == 0 && NW <= 16 && (NW & (NW - 1)) == 0, "bad group size");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int g = (G == 1) ? 0 : (int)(threadIdx.x / NTG);
  const int gtid = (G == 1) ? (int)threadIdx.x : (int)(threadIdx.x % NTG);
  Elem* buf = reinterpret_cast<Elem*>(smem_raw + g * a.buf_bytes);
  ControlBlock* cb = reinterpret_cast<ControlBlock*>(smem_raw + a.ctrl_offset) + g;

  const uint32_t rank = ptx::cluster_ctarank();
  const uint32_t C = ptx::cluster_nctarank();
  const int64_t cid = ptx::cluster_id_x();
  const int64_t ncl = ptx::nclusters_x();
  const int64_t n = a.n;
  const int64_t base = (int64_t)rank * a.L;
  const int64_t rem = n - base;
  const int len = rem <= 0 ? 0 : (rem < a.L ? (int)rem : a.L);
  const bool TMA = a.tma != 0;
  const double mphantom = (double)((int64_t)C * NTG * E - n);  // phantom slots in the cluster
  const RowParams& rp = a.rp;
  const int T = rp.T;
  const Elem* __restrict__ X = reinterpret_cast<const Elem*>(a.x);
  Elem* __restrict__ Z = reinterpret_cast<Elem*>(a.z);

  const uint32_t bar_load = ptx::smem_addr(&cb->mb_load);
  const uint32_t load_bytes = (uint32_t)len * (uint32_t)sizeof(Elem);
  uint64_t policy = 0;
  if (TMA) policy = ptx::policy_evict_first();

  if (gtid == 0) {
    ptx::mbar_init(bar_load, 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_x[0]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_x[1]), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (gtid == 0) {
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[0]), C * 32u);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[1]), C * 32u);
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

  const int64_t row0 = cid * G + g, rstride = ncl * G;
  uint32_t xround = 0, load_par = 0;
  // De-phase the row streams (dev knob, default off).
  if (a.stagger > 0) {
    const long long wait = a.stagger * (long long)(g * ncl + cid) / (long long)(G * ncl);
    const long long t0 = clock64();
    while (clock64() - t0 < wait) __nanosleep(256);
  }

  Elem v[E];
  // Register <- shared-memory slice copy (phantoms = k0).  Used for the first row.
  auto lds_slice = [&](Elem k0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int li0 = (k * NTG + gtid) * VEC;
      if (li0 + VEC <= len) {
        const V t = *reinterpret_cast<const V*>(buf + li0);
        *reinterpret_cast<V*>(&v[k * VEC]) = t;
      } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[k * VEC + j] = (li0 + j < len) ? buf[li0 + j] : k0;
      }
    }
  };

  // TMA pipeline per group (landing buffer `buf`):
  //   row r computes from registers while buf receives X(r+1);
  //   at the end of row r each thread swaps Z(r) into buf and X(r+1) into its
  //   registers, and one thread streams buf -> Z(r) with a bulk TMA store;
  //   once that store has read buf (checked after the next row's first
  //   exchange) the load of X(r+2) is issued into buf.
  if (TMA && gtid == 0 && row0 < a.B) issue_load(row0);
  if (TMA && row0 < a.B) {
    ptx::mbar_wait_cta(bar_load, load_par);
    load_par ^= 1u;
    lds_slice(__ldg(X + row0 * a.ldx));
    group_sync<NTG>(g);  // buf free
  }
  bool need_issue = TMA;  // deferred prefetch of the row after next

  // Row slots: both groups of a CTA walk the same number of slots so their pass
  // tokens stay balanced (a group without a row in its last slot idles).
  const int64_t first0 = cid * G;
  const int64_t K = (a.B > first0) ? (a.B - first0 + rstride - 1) / rstride : 0;
  PassToken<NTG, G> tok(g, K * (int64_t)(T + 1));
  for (int64_t k = 0; k < K; ++k) {
    const int64_t row = row0 + k * rstride;
    if (row >= a.B) {  // idle slot: keep the token moving
      for (int ph = 0; ph <= T; ++ph) {
        tok.take();
        tok.give();
      }
      continue;
    }
    const int64_t next = row + rstride;
    const bool has_next = next < a.B;
    const int64_t lrow = k;
    // trace: group g uses rows [g*kTraceRows/G, (g+1)*kTraceRows/G) of its CTA's trace block
    long long* tr = (a.trace && lrow < kTraceRows / G)
                        ? a.trace + ((int64_t)blockIdx.x * kTraceRows + g * (kTraceRows / G) + lrow) * kTraceEvents
                        : nullptr;
    PAM_TRACE(tr, 0);
    const Elem* xrow = X + row * a.ldx;
    const Elem k0e = __ldg(xrow);  // shift for the input pass (same in every CTA)
    const double K0 = (double)k0e;
    const Elem k0next = has_next ? __ldg(X + next * a.ldx) : Elem(0);
    tok.take();  // input pass (shift + moments) needs the fp64 pipe

    if (!TMA) {  // unaligned rows: direct loads, no staging
      const Elem* src = xrow + base;
#pragma unroll
      for (int kk = 0; kk < NV; ++kk) {
        const int li0 = (kk * NTG + gtid) * VEC;
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[kk * VEC + j] = (li0 + j < len) ? __ldcs(src + li0 + j) : k0e;
      }
    }
    PAM_TRACE(tr, 2);

    // deferred: once the previous Z store has read buf, prefetch X(next) into it
    auto prefetch_next = [&]() {
      if (need_issue && gtid == 0) {
        ptx::bulk_wait_read_all();
        if (has_next) issue_load(next);
      }
    };

    // ---- input statistics + T CutMax iterations + normaliser + argmax ------------
    double rnorm = 1.0;
    long long amax = -1;
    const int st = cutmax_core<Elem, NTG, G, E, P, true>(
        v, tok, K0, mphantom, rp, a.inv_n, cb, xround, rank, C, g, gtid, base,
        (rank == 0 && gtid == 0 && a.stats) ? a.stats + row * T * 2 : nullptr, rnorm, amax, tr, prefetch_next);
    PAM_TRACE(tr, 20);
    if (rank == 0 && gtid == 0) {
      if (a.argmax) a.argmax[row] = (st == PAM_OK) ? (int32_t)amax : -1;
      if (a.status) a.status[row] = st;
    }

    // ---- Z = Y * inv(sum Y) ------------------------------------------------------
    const Elem re = (Elem)rnorm;
    Elem* zrow = Z + row * a.ldz + base;
    if (TMA) {
      // swap: Z(row) -> buf, X(next) -> registers; then bulk-store buf -> Z(row)
      if (has_next) {
        ptx::mbar_wait_cta(bar_load, load_par);
        load_par ^= 1u;
      }
#pragma unroll
      for (int kk = 0; kk < NV; ++kk) {
        const int li0 = (kk * NTG + gtid) * VEC;
        Elem o[VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) o[j] = v[kk * VEC + j] * re;
        if (li0 + VEC <= len) {
          const V xn = *reinterpret_cast<const V*>(buf + li0);
          *reinterpret_cast<V*>(buf + li0) = *reinterpret_cast<V*>(o);
          *reinterpret_cast<V*>(&v[kk * VEC]) = xn;
        } else {
#pragma unroll
          for (int j = 0; j < VEC; ++j) {
            const Elem xn = (li0 + j < len) ? buf[li0 + j] : k0next;
            if (li0 + j < len) buf[li0 + j] = o[j];
            v[kk * VEC + j] = xn;
          }
        }
      }
      ptx::fence_proxy_async_smem();  // make the Z writes visible to the TMA engine
      group_sync<NTG>(g);
      if (gtid == 0 && !(a.debug_flags & 1)) {
        const uint32_t zbytes = load_bytes;
        const unsigned char* dstb = reinterpret_cast<const unsigned char*>(zrow);
        for (uint32_t off = 0; off < zbytes; off += 32768u) {
          const uint32_t nb = (zbytes - off) < 32768u ? (zbytes - off) : 32768u;
          ptx::bulk_s2g((void*)(dstb + off), ptx::smem_addr(buf) + off, nb, policy);
        }
        ptx::bulk_commit();
      }
    } else if (!(a.debug_flags & 1)) {
#pragma unroll
      for (int kk = 0; kk < NV; ++kk) {
        const int li0 = (kk * NTG + gtid) * VEC;
#pragma unroll
        for (int j = 0; j < VEC; ++j)
          if (li0 + j < len) __stcs(zrow + li0 + j, v[kk * VEC + j] * re);
      }
    }
    PAM_TRACE(tr, 21);
  }
  if (TMA && gtid == 0) ptx::bulk_wait_all();  // Z stores complete before the CTA retires
  ptx::cluster_sync();  // no CTA leaves while a peer may still push into its shared memory
}

}  // namespace pam
