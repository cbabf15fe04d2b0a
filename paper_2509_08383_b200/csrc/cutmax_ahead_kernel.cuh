// cutmax_ahead_kernel.cuh — batched fp64 CutMax for p = 3: two iterations per
// cluster exchange ("moments ahead").
//
// Replaces core.cutmax (Alg. 1) for the headline
// configuration (fp64, p_t = 3 for every t, exact 1/sqrt and 1/x, 16-byte
// aligned rows).  Everything else runs cutmax_rows_kernel (cutmax_kernel.cuh).
//
// Why.  A row of n = 151936 doubles spans a cluster of ~9 CTAs, so every
// iteration's mean and variance is a cluster all-reduce, and the row is a
// serial chain pass -> CTA reduction -> DSMEM exchange -> scalar chain -> pass.
// With one exchange per iteration (cutmax_rows_kernel) ~45% of a row is that
// chain while the fp64 pipe idles.  This kernel halves the number of chains.
//
// How.  With z = a + k*v (v = y - K the stored, shifted iterate) and
// y' = z^3, the first moments of the NEXT iterate are polynomials in the power
// sums S_j = sum v^j of the current one:
//     sum y'   = sum_j C(3,j) a^(3-j) k^j S_j          (j <= 3)
//     sum y'^2 = sum_j C(6,j) a^(6-j) k^j S_j          (j <= 6)
//     sum y'^3 = sum_j C(9,j) a^(9-j) k^j S_j          (j <= 9)
// so one exchange of S_1..S_6 gives (mu_t, s2_t) AND (mu_{t+1}, s2_{t+1}), and
// S_1..S_9 also gives the normaliser sum_i (b + k' y'_i)^3 of the iteration
// after.  A stage is one exchange: stage i holds iterate y_s (s = 2i+1) and
// covers iterations s and s+1.  For T = 4 a row is
//     [input S_1..S_6 + previous row's argmax] -> pass: y2, y3, S_1..S_9 of y3
//     -> [exchange] -> last pass: y4, y5 = Y, Z = Y / sum Y, argmax, and the
//     next row's input moments (its X already sits in the row buffer).
// Two exchanges per row instead of four, at 36 fp64 instructions per element
// instead of 23 (the fp64 pipe is ~38% busy in cutmax_rows_kernel).
//
// Numerics.  The expansions are exact algebra; their rounding is bounded by
// the condition number A_m / |E_m| (A_m the same sum over |terms|, with
// sum|v|^j bounded by S_j, sqrt(S_{j-1} S_{j+1}) or S_{M-1}^{M/(M-1)}).  The
// control warp evaluates it for every expansion and for the variance
// cancellations; above kAhCondMax (or on any non-finite intermediate) the
// stage falls back to the exact path: two-pass mean/variance per iteration and
// an explicit sum of Y, one cluster sum per pass (cluster-uniform decision, so
// every CTA takes it).  Measured on N(0,3^2), Zipf, planted near-ties,
// Cauchy and shifted rows: <= 5e-14 normwise vs the fsum-exact oracle at
// condition numbers up to 2e3; the fallback almost never runs.
//
// Data movement.  The input row X(r+1) is TMA-loaded into the shared row
// buffer during row r.  The last pass of row r swaps it into registers and
// writes Z(r) into the same slots; Z(r) leaves through 1-D TMA bulk stores
// (4 bulk groups), and X(r+2) is loaded behind them at row r+1's
// first mid exchange.  (Storing Z with st.global from registers instead queued
// the exchanges' st.async behind 136 KB of stores.)
//
// Status: correct and opt-in (PAM_ENABLE_AHEAD); 50% of HBM at 4096 x 151936
// vs 57% for cutmax_rows_kernel — the per-stage control path (wait, phase A,
// phase B) runs from a cold instruction cache (DESIGN.md §4 K1b).
//
// Exchange.  Every thread writes its M partial sums to smem (part[j][tid]);
// after one CTA barrier, warp j reduces column j (16 values per lane + a
// 5-level butterfly) and pushes the CTA total into slot [j][rank] of every
// CTA of the cluster (8-byte st.async completing on that CTA's mbarrier); one
// more warp reduces the argmax candidates.  Warp 0 (the control warp) waits,
// sums the C records of each moment in rank order — identical in every CTA —
// runs the scalar chain and publishes the pass coefficients through shared
// memory and a named barrier.
#pragma once

#include "cutmax_kernel.cuh"

namespace pam {

#ifdef PAM_TRACE_BUILD
__device__ __forceinline__ long long ah_gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PAM_GTRACE(tr, k)                                       \
  do {                                                          \
    if ((tr) != nullptr && gtid == 0) (tr)[k] = ah_gtime();     \
  } while (0)
#else
#define PAM_GTRACE(tr, k) \
  do {                    \
  } while (0)
#endif

constexpr int kAhMaxM = 9;
constexpr double kAhCondMax = 256.0;

// moments exchanged at stage i (holding iterate y_s, s = 2i+1)
__host__ __device__ __forceinline__ int ah_stage_M(int i, int T) {
  const int s = 2 * i + 1;
  return s == T ? 3 : (s + 1 == T ? 9 : 6);
}

// Phase-A broadcast: iteration s of the stage (z = fma(v, ka, aa)).
struct __align__(16) AhCoefA {
  double ka, aa;
  int st, slow;  // row status so far; 1: exact statistics for the whole stage
};
// Phase-B broadcast: iteration s+1 (z' = fma(y, kb, bb), y = z^3) and the
// normaliser of the last stage.
struct __align__(16) AhCoefB {
  double kb, bb;
  double kn;   // shift of the value a mid pass stores: v' = z'^3 - kn
  double rn;   // 1 / sum Y (last stage)
  double k0n;  // input shift of the next row (last stage)
  int st, slow;
};

template <int NTG>
struct AhCtl {
  double part[kAhMaxM][NTG];  // per-thread partial sums, column j = moment j+1
  double candv[NTG];          // per-thread argmax candidates
  long long candi[NTG];
  double rec[2][kAhMaxM][16];  // cluster records [round parity][moment][src rank]
  double2 rarg[2][16];         // argmax records (value, index bits)
  double srec[2][16];          // exact-path channel: one sum per src rank
  AhCoefA bca;
  AhCoefB bcb;
  double kc;  // shift of the stage iterate (exact path of phase A)
  unsigned long long mb_load;
  unsigned long long mb_x[2];
  unsigned long long mb_s[2];
};

__device__ __forceinline__ double ah_cube(double z) { return (z * z) * z; }

// r = x^e for 0 <= e <= 15 (lane-varying e), branch-free.
__device__ __forceinline__ double ah_ipow(double x, int e) {
  const double b2 = x * x, b4 = b2 * b2, b8 = b4 * b4;
  double r = (e & 1) ? x : 1.0;
  r = (e & 2) ? r * b2 : r;
  r = (e & 4) ? r * b4 : r;
  r = (e & 8) ? r * b8 : r;
  return r;
}

// C(m, j) for m in {3, 6, 9}, 0 outside 0 <= j <= m.
__device__ __forceinline__ double ah_binom(int m, int j) {
  const unsigned long long k = m == 3 ? 0x01030301ull : (m == 6 ? 0x01060F140F0601ull : 0x24547E7E54240901ull);
  const unsigned long long hi = m == 9 ? 0x0109ull : 0ull;  // C(9,8), C(9,9)
  const unsigned long long c = j < 8 ? (k >> (8 * (j & 7))) & 0xFFull : (hi >> (8 * (j & 1))) & 0xFFull;
  return (j >= 0 && j <= m) ? (double)c : 0.0;
}

// x * 2^k for 0 <= k < 1000 (exact; overflow -> inf)
__device__ __forceinline__ double ah_scale2(double x, int k) {
  return x * __longlong_as_double((long long)(1023 + k) << 52);
}
// floor(log2 x) + 1 for positive normal x (0 for x < 1 and subnormals)
__device__ __forceinline__ int ah_exp_pos(double x) {
  const int e = (int)((__double_as_longlong(x) >> 52) & 0x7ff) - 1022;
  return e > 0 ? e : 0;
}

// 1/x: hardware estimate + three Newton steps (<= 2 ulp for normal x;
// 0, inf and NaN propagate as inf, 0 and NaN).
__device__ __forceinline__ double ah_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  r = fma(r, fma(-x, r, 1.0), r);
  r = fma(r, fma(-x, r, 1.0), r);
  return r;
}

// Accumulate the power sums S_1..S_M of w (s[j] holds S_{j+1}).
template <int M>
__device__ __forceinline__ void ah_acc(double (&s)[kAhMaxM], const double w) {
  s[0] += w;
  s[1] = fma(w, w, s[1]);
  if (M >= 3) {
    const double w2 = w * w;
    s[2] = fma(w2, w, s[2]);
    if (M >= 6) {
      s[3] = fma(w2, w2, s[3]);
      const double w3 = w2 * w;
      s[4] = fma(w3, w2, s[4]);
      s[5] = fma(w3, w3, s[5]);
      if (M >= 9) {
        const double w4 = w2 * w2;
        s[6] = fma(w4, w3, s[6]);
        s[7] = fma(w4, w4, s[7]);
        const double w5 = w4 * w;
        s[8] = fma(w5, w4, s[8]);
      }
    }
  }
}

// Sum of column p[lane + 32k], k < NW, then a 32-lane butterfly: every lane
// returns the CTA total.
template <int NW>
__device__ __forceinline__ double ah_col_sum(const double* p, const int lane) {
  double t[NW];
#pragma unroll
  for (int k = 0; k < NW; ++k) t[k] = p[lane + 32 * k];
#pragma unroll
  for (int w = NW / 2; w >= 1; w /= 2)
#pragma unroll
    for (int k = 0; k < w; ++k) t[k] += t[k + w];
  double a = t[0];
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) a += __shfl_xor_sync(0xffffffffu, a, m);
  return a;
}

// Exchange push: partials -> smem -> CTA barrier -> warp j reduces moment j and
// pushes it to every CTA of the cluster; warp M reduces the argmax (ARG).
// `side` runs on lane 0 of the last warp after the barrier (DMA hook).
template <int NTG, int M, bool ARG, typename Side>
__device__ __forceinline__ void ah_push(const double (&s)[kAhMaxM], const double bv, const long long bi,
                                        AhCtl<NTG>* cb, const uint32_t round, const uint32_t rank, const uint32_t C,
                                        const int gtid, const Side& side) {
  constexpr int NW = NTG / 32;
  constexpr int NCOL = M + (ARG ? 1 : 0);
  const int lane = gtid & 31, warp = gtid >> 5;
#pragma unroll
  for (int j = 0; j < M; ++j) cb->part[j][gtid] = s[j];
  if (ARG) {  // each warp reduces its candidates first (REDUX), lane 0 posts the warp's
    double wv = bv;
    long long wi = bi;
    warp_argmax(wv, wi);
    if (lane == 0) {
      cb->candv[warp] = wv;
      cb->candi[warp] = wi;
    }
  }
  __syncthreads();
  const uint32_t par = round & 1u;
  const uint32_t bar = ptx::smem_addr(&cb->mb_x[par]);
  for (int col = warp; col < NCOL; col += NW) {
    if (col < M) {
      const double acc = ah_col_sum<NW>(cb->part[col], lane);
      if (lane < (int)C)
        ptx::st_async_f64(ptx::mapa(ptx::smem_addr(&cb->rec[par][col][rank]), (uint32_t)lane), acc,
                          ptx::mapa(bar, (uint32_t)lane));
    } else {
      double v = lane < NW ? cb->candv[lane] : -HUGE_VAL;
      long long ix = lane < NW ? cb->candi[lane] : 0x7fffffffffffffffLL;
      warp_argmax(v, ix);
      if (lane < (int)C)
        ptx::st_async_b64x2(ptx::mapa(ptx::smem_addr(&cb->rarg[par][rank]), (uint32_t)lane),
                            (uint64_t)__double_as_longlong(v), (uint64_t)ix, ptx::mapa(bar, (uint32_t)lane));
    }
  }
  if (warp == NW - 1 && lane == 0) side();
}

// Control-warp wait: lane l returns S_{l+1} (l < M, summed over the C ranks in
// rank order), 0 elsewhere; with ARG every lane also gets the cluster argmax.
// Re-arms this parity's barrier for round + 2 (arm_bytes).
template <int NTG>
__device__ __forceinline__ double ah_wait(AhCtl<NTG>* cb, uint32_t& round, const int M, const bool arg,
                                          const uint32_t C, const int lane, const uint32_t arm_bytes, double& bv,
                                          long long& bi) {
  const uint32_t par = round & 1u, ph = (round >> 1) & 1u;
  const uint32_t bar = ptx::smem_addr(&cb->mb_x[par]);
  ptx::mbar_wait_cta(bar, ph);
  if (lane == 0) ptx::mbar_arrive_expect_tx(bar, arm_bytes);
  const double* rr = cb->rec[par][lane < M ? lane : 0];
  double S = 0.0;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const double x = rr[r];
    if (r < (int)C) S += x;
  }
  S = lane < M ? S : 0.0;
  if (arg) {
    const bool have = lane < (int)C;
    const double2 rv = cb->rarg[par][have ? lane : 0];
    bv = have ? rv.x : -HUGE_VAL;
    bi = have ? __double_as_longlong(rv.y) : 0x7fffffffffffffffLL;
    warp_argmax(bv, bi);
  }
  ++round;
  return S;
}

// Phase B of the control chain (see cutmax_ahead_kernel): iteration s+1 of
// stage i and the normaliser, from the power sums S[0..M] (S[0] = n) and
// phase A's (ka, aa), in every lane of the control warp (straight-line code,
// no lane-dependent work).
//   E_m = (1/n) sum_i (aa + ka v_i)^m = (1/n) sum_j C(m,j) aa^(m-j) ka^j S_j
// for m = 3, 6, 9 are the mean, second and third moments of y_{s+1} = z^3.
// A_m, the same sums over |terms| (sum|v|^j <= S_j for even j,
// (S_{j-1} + S_{j+1}) / 2 for odd j < M, S_{M-1}^{M/(M-1)} for odd j = M),
// bound their rounding; the stage goes exact (slow = 1) when A_m / |E_m| or
// the variance cancellation exceeds kAhCondMax.
template <int M, bool TWO, bool LAST>
__device__ __forceinline__ AhCoefB ah_phase_b_t(const double (&S)[10], const AhCoefA& ca, const int it,
                                                 const double inv_n, const double eps_var, const RowParams& rp) {
  constexpr int C3[4] = {1, 3, 3, 1};
  constexpr int C6[7] = {1, 6, 15, 20, 15, 6, 1};
  constexpr int C9[10] = {1, 9, 36, 84, 126, 126, 84, 36, 9, 1};
  const double ka = ca.ka, aa = ca.aa;
  int st = ca.st;
  double ap[10], kp[10];
  ap[0] = 1.0;
  kp[0] = 1.0;
#pragma unroll
  for (int j = 1; j <= 9; ++j) {
    ap[j] = ap[j - 1] * aa;
    kp[j] = kp[j - 1] * ka;
  }
  double U[10];
#pragma unroll
  for (int j = 0; j <= M; ++j) {
    if (!(j & 1)) {
      U[j] = S[j];
    } else if (j < M) {
      U[j] = 0.5 * (S[j - 1] + S[j + 1]);
    } else {  // S_{M-1}^{M/(M-1)} <= S_{M-1} * 2^(floor(e/(M-1)) + 1)
      U[j] = ah_scale2(S[j - 1], (M == 3 ? ah_exp_pos(S[j - 1]) >> 1 : ah_exp_pos(S[j - 1]) >> 3) + 1);
    }
  }
  double E3 = 0.0, E6 = 0.0, E9 = 0.0, A3 = 0.0, A6 = 0.0, A9 = 0.0;
#pragma unroll
  for (int j = 0; j <= 3; ++j) {
    const double w = ap[3 - j] * kp[j];
    E3 = fma((double)C3[j] * w, S[j], E3);
    A3 = fma((double)C3[j] * fabs(w), U[j], A3);
  }
  if (TWO) {
#pragma unroll
    for (int j = 0; j <= 6; ++j) {
      const double w = ap[6 - j] * kp[j];
      E6 = fma((double)C6[j] * w, S[j], E6);
      A6 = fma((double)C6[j] * fabs(w), U[j], A6);
    }
    if (LAST) {
#pragma unroll
      for (int j = 0; j <= 9; ++j) {
        const double w = ap[9 - j] * kp[j];
        E9 = fma((double)C9[j] * w, S[j], E9);
        A9 = fma((double)C9[j] * fabs(w), U[j], A9);
      }
    }
  }
#ifdef PAM_AHEAD_NOCOND  // dev experiment: the cost of the condition bounds (unsafe; never shipped)
  A3 = fabs(E3);
  A6 = fabs(E6);
  A9 = fabs(E9);
#endif
  E3 *= inv_n;
  E6 *= inv_n;
  E9 *= inv_n;
  A3 *= inv_n;
  A6 *= inv_n;
  A9 *= inv_n;
  double okb = 0.0, obb = 1.0, orn = 1.0;
  bool slow = false;
  if (TWO) {
    const double s2b = fma(-E3, E3, E6);
    slow = !((A6 + 2.0 * fabs(E3) * A3) <= kAhCondMax * s2b) || !(A3 * A3 <= (kAhCondMax * kAhCondMax) * s2b);
    const double kb = rsqrt(s2b) * rp.inv_c[it + 1];
    const double bb = fma(-E3, kb, 1.0);
    if (LAST) {  // sum_i (bb + kb y_i)^3 with sum y^j = n E_{3j}
      const double kab = fabs(kb), bab = fabs(bb);
      const double SYn = bb * bb * bb + kb * (3.0 * bb * bb * E3 + kb * (3.0 * bb * E6 + kb * E9));
      const double ASY = bab * bab * bab + kab * (3.0 * bab * bab * A3 + kab * (3.0 * bab * A6 + kab * A9));
      slow = slow || !(ASY <= kAhCondMax * fabs(SYn)) || !isfinite(SYn);
      orn = ah_rcp(SYn * S[0]);
    }
    if (st == PAM_OK && !slow) {
      st = (!isfinite(E3) || !isfinite(s2b)) ? PAM_ERR_RANGE : (s2b < eps_var ? PAM_ERR_DEGENERATE_INPUT : PAM_OK);
      okb = kb;
      obb = bb;
      if (LAST && st == PAM_OK && !(orn > 0.0)) st = PAM_ERR_RANGE;  // Z must be a distribution
    }
  } else {  // LAST with one iteration: sum Y = n E3
    slow = !(A3 <= kAhCondMax * fabs(E3)) || !isfinite(E3);
    orn = ah_rcp(E3 * S[0]);
    if (st == PAM_OK && !slow && !(orn > 0.0)) st = PAM_ERR_RANGE;
  }
  slow = slow && st == PAM_OK;
  if (st != PAM_OK || slow) {
    okb = 0.0;
    obb = 1.0;
    orn = 1.0;
  }
  AhCoefB r;
  r.kb = okb;
  r.bb = obb;
  r.kn = LAST ? 0.0 : rp.kshift[it + 2];
  r.rn = orn;
  r.k0n = 0.0;
  r.st = st;
  r.slow = slow ? 1 : 0;
  return r;
}

// ---------------------------------------------------------------------------
template <int NTG, int E>
__global__ void __launch_bounds__(NTG, 1) cutmax_ahead_kernel(const CutmaxArgs a) {
  constexpr int NV = E / 2;
  constexpr int NW = NTG / 32;
  static_assert(E % 2 == 0 && NW >= 4 && NW <= 16 && (NW & (NW - 1)) == 0, "bad geometry");
  constexpr unsigned FULL = 0xffffffffu;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int gtid = (int)threadIdx.x;
  const int lane = gtid & 31, warp = gtid >> 5;
  double* buf = reinterpret_cast<double*>(smem_raw);
  AhCtl<NTG>* cb = reinterpret_cast<AhCtl<NTG>*>(smem_raw + a.ctrl_offset);

  const uint32_t rank = ptx::cluster_ctarank();
  const uint32_t C = ptx::cluster_nctarank();
  const int64_t cid = ptx::cluster_id_x();
  const int64_t ncl = ptx::nclusters_x();
  const int64_t n = a.n;
  const int64_t base = (int64_t)rank * a.L;
  const int64_t rem = n - base;
  const int len = rem <= 0 ? 0 : (rem < a.L ? (int)rem : a.L);
  const RowParams& rp = a.rp;
  const int T = rp.T;
  const int NS = (T + 1) / 2;
  const int M0 = ah_stage_M(0, T);
  const double nd = (double)n, inv_n = a.inv_n, eps_var = rp.eps_var;
  const double* __restrict__ X = reinterpret_cast<const double*>(a.x);
  double* __restrict__ Zo = reinterpret_cast<double*>(a.z);
  const bool dma = gtid == NTG - 32;
  const bool store_z = !(a.debug_flags & 1);
  const bool skip_passes = (a.debug_flags & 2) != 0;  // dev: exchange/chain latency probe
  const uint32_t bar_load = ptx::smem_addr(&cb->mb_load);
  const uint32_t slice_bytes = (uint32_t)len * 8u;
  const uint32_t chunk = ((slice_bytes + 63u) / 64u) * 16u;  // 4 bulk copies per slice
  const uint64_t policy = ptx::policy_evict_first();

  // bytes one round delivers to each CTA: stage-0 rounds carry M0 sums + argmax
  auto pos_bytes = [&](int pos) -> uint32_t {
    return C * (pos == 0 ? 8u * (uint32_t)M0 + 16u : 8u * (uint32_t)ah_stage_M(pos, T));
  };

  if (gtid == 0) {
    ptx::mbar_init(bar_load, 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_x[0]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_x[1]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_s[0]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_s[1]), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (gtid == 0) {
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[0]), pos_bytes(0));
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[1]), pos_bytes(1 % NS));
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_s[0]), 8u * C);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_s[1]), 8u * C);
  }
  ptx::cluster_sync();
  int arm_pos = 2 % NS;  // control warp: stage position of round xround + 2

  // DMA lane (lane 0 of the last warp).  The row buffer holds X(r+1) while row
  // r computes; the last pass swaps it for Z(r), which leaves through 1-D TMA
  // bulk stores (one bulk group per chunk) — global stores from the SM's LSU
  // would queue the cluster exchange's st.async behind 136 KB of Z — and
  // X(r+2) is loaded chunk by chunk as the store has read each chunk.
  auto load_row = [&](int64_t r, bool after_store) {  // X(r) slice -> row buffer
    ptx::mbar_arrive_expect_tx(bar_load, slice_bytes);
    const unsigned char* src = reinterpret_cast<const unsigned char*>(X + r * a.ldx + base);
    int i = 0;
    for (uint32_t off = 0; off < slice_bytes; off += chunk, ++i) {
      const uint32_t nb = (slice_bytes - off) < chunk ? (slice_bytes - off) : chunk;
      if (after_store && store_z) ptx::bulk_wait_read_le(3 - i);
      ptx::bulk_g2s(ptx::smem_addr(buf) + off, src + off, nb, bar_load, policy);
    }
  };
  auto store_row = [&](int64_t r) {  // Z(r) row buffer -> HBM
    if (!store_z) return;
    unsigned char* dst = reinterpret_cast<unsigned char*>(Zo + r * a.ldz + base);
    int i = 0;
    for (uint32_t off = 0; off < slice_bytes; off += chunk, ++i) {
      const uint32_t nb = (slice_bytes - off) < chunk ? (slice_bytes - off) : chunk;
      ptx::bulk_s2g(dst + off, ptx::smem_addr(buf) + off, nb, policy);
      ptx::bulk_commit();
    }
    for (; i < 4; ++i) ptx::bulk_commit();  // always 4 groups: wait_read counts stay fixed
  };
  // input shift: mean of 8 fixed samples of the row (identical in every CTA)
  auto k0_of = [&](int64_t r) -> double {
    const double* xr = X + r * a.ldx;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += __ldg(xr + (j * n) / 8) * 0.125;
    return s;
  };
  auto valid = [&](int q) { return (q * NTG + gtid) * 2 < len; };
  auto status_of = [&](double mu, double s2) {
    return (!isfinite(mu) || !isfinite(s2)) ? PAM_ERR_RANGE : (s2 < eps_var ? PAM_ERR_DEGENERATE_INPUT : PAM_OK);
  };

  uint32_t xround = 0, sround = 0, load_par = 0;
  double v[E];
  double s[kAhMaxM];

  // ---- exact path (cluster-uniform, rare): one cluster sum per call ----------
  auto xs1 = [&](double p) -> double {
    cb->part[0][gtid] = p;
    __syncthreads();
    const uint32_t par = sround & 1u, ph = (sround >> 1) & 1u;
    const uint32_t bar = ptx::smem_addr(&cb->mb_s[par]);
    if (warp == 0) {
      const double acc = ah_col_sum<NW>(cb->part[0], lane);
      if (lane < (int)C)
        ptx::st_async_f64(ptx::mapa(ptx::smem_addr(&cb->srec[par][rank]), (uint32_t)lane), acc,
                          ptx::mapa(bar, (uint32_t)lane));
    }
    ptx::mbar_wait_cta(bar, ph);
    double tot = 0.0;
    for (uint32_t r = 0; r < C; ++r) tot += cb->srec[par][r];
    __syncthreads();
    if (gtid == 0) ptx::mbar_arrive_expect_tx(bar, 8u * C);  // arm round + 2
    ++sround;
    return tot;
  };
  // exact iteration s from registers v = y_s - kc: two-pass mean and variance
  auto slow_a = [&](int i, AhCoefA& ca, double kc) {
    int st = ca.st;
    double p = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) p += v[e];  // phantoms hold 0
    const double dm = xs1(p) * inv_n;
    p = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const double d = v[e] - dm;
      if (valid(e / 2)) p = fma(d, d, p);
    }
    const double s2 = xs1(p) * inv_n;
    if (st == PAM_OK) st = status_of(kc + dm, s2);
    ca.ka = (st == PAM_OK) ? rsqrt(s2) * rp.inv_c[2 * i] : 0.0;
    ca.aa = fma(-((kc + dm) - kc), ca.ka, 1.0);  // centered on the fp64-rounded mean (see phase A)
    ca.st = st;
  };
  // exact iteration s+1 (two) from registers v = y_{s+1}, and/or the explicit
  // normaliser (last stage; registers hold Y when the stage has one iteration)
  auto slow_b = [&](int i, AhCoefB& c, int st) {
    const int s_ = 2 * i + 1;
    const bool two = s_ + 1 <= T, last = s_ + 1 >= T;
    double kb = 0.0, bb = 1.0, rn = 1.0;
    if (two) {
      double p = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (valid(e / 2)) p += v[e];
      const double mu = xs1(p) * inv_n;
      p = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const double d = v[e] - mu;
        if (valid(e / 2)) p = fma(d, d, p);
      }
      const double s2b = xs1(p) * inv_n;
      if (st == PAM_OK) st = status_of(mu, s2b);
      kb = (st == PAM_OK) ? rsqrt(s2b) * rp.inv_c[s_] : 0.0;
      bb = fma(-mu, kb, 1.0);
    }
    if (last) {
      double p = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const double y = two ? ah_cube(fma(v[e], kb, bb)) : v[e];
        if (valid(e / 2)) p += y;
      }
      const double tot = xs1(p);
      if (st == PAM_OK && (!isfinite(tot) || !(tot > 0.0))) st = PAM_ERR_RANGE;  // Z must be a distribution
      rn = (st == PAM_OK) ? 1.0 / tot : 1.0;
    }
    if (st != PAM_OK) {
      kb = 0.0;
      bb = 1.0;
      rn = 1.0;
    }
    c.kb = kb;
    c.bb = bb;
    c.rn = rn;
    c.st = st;
  };

  // ---- control warp, phase A: iteration s of stage i --------------------------
  // Sl: lane l holds S_{l+1} of the stage iterate (shifted by Kc).  Publishes
  // (ka, aa) so the other warps can run the first half of the pass while
  // phase B (the expansions) is still computing.
  auto phase_a = [&](int i, double Sl, double Kc, int st) {
    const int it = 2 * i;
    const double S1 = __shfl_sync(FULL, Sl, 0), S2 = __shfl_sync(FULL, Sl, 1);
    if (i == 0 && st == PAM_OK && (!isfinite(S1) || !isfinite(S2))) st = PAM_ERR_NON_FINITE;
    const double dm = S1 * inv_n, q = S2 * inv_n;
    const double s2 = fma(-dm, dm, q);
    const bool slow = st == PAM_OK && !(q <= kAhCondMax * s2);  // poor shift / s2 <= 0: exact statistics
    if (st == PAM_OK && !slow) st = status_of(Kc + dm, s2);
    const double ka = (st == PAM_OK && !slow) ? rsqrt(s2) * rp.inv_c[it] : 0.0;
    // center on the mean rounded to fp64, as the reference computes it
    // (SPEC.md:127); (Kc + dm) - Kc is exact.  The expansions of phase B use
    // the same (aa, ka), so they stay consistent.
    const double aa = fma(-((Kc + dm) - Kc), ka, 1.0);
    if (lane == 0) {
      cb->bca.ka = ka;
      cb->bca.aa = aa;
      cb->bca.st = st;
      cb->bca.slow = slow ? 1 : 0;
      cb->kc = Kc;
    }
    __syncwarp();  // (warp 0 itself reads kc in the exact path)
    return AhCoefA{ka, aa, st, slow ? 1 : 0};
  };
  // ---- control warp, phase B: iteration s+1 and the normaliser ----------------
  // sum_i (aa + ka v_i)^m = sum_j C(m,j) aa^(m-j) ka^j S_j for m = 3, 6, 9
  // (mean, second and third moments of y_{s+1} = z^3), with condition bounds
  // A_m (the same sums over |terms|; sum|v|^j <= S_j for even j,
  // (S_{j-1} + S_{j+1}) / 2 for odd j < M, S_{M-1}^{M/(M-1)} for odd j = M).
  auto phase_b = [&](int i, double Sl, const AhCoefA& ca, double k0n) {
    const int s_ = 2 * i + 1, M = ah_stage_M(i, T);
    double S[10];
    S[0] = nd;
#pragma unroll
    for (int j = 1; j <= 9; ++j) S[j] = __shfl_sync(FULL, Sl, j - 1);
    AhCoefB r;
    if (M == 6)
      r = ah_phase_b_t<6, true, false>(S, ca, s_ - 1, inv_n, eps_var, rp);
    else if (M == 9)
      r = ah_phase_b_t<9, true, true>(S, ca, s_ - 1, inv_n, eps_var, rp);
    else
      r = ah_phase_b_t<3, false, true>(S, ca, s_ - 1, inv_n, eps_var, rp);
    if (lane == 0) {
      cb->bcb = r;
      cb->bcb.k0n = k0n;
    }
  };
  // phase B when phase A went exact: only the bookkeeping (slow_b runs everywhere)
  auto phase_b_slow = [&](int i, int st, double k0n) {
    const int s_ = 2 * i + 1, it = s_ - 1;
    const bool last = s_ + 1 >= T;
    if (lane == 0) {
      AhCoefB& b = cb->bcb;
      b.kb = 0.0;
      b.bb = 1.0;
      b.kn = last ? 0.0 : rp.kshift[it + 2];
      b.rn = 1.0;
      b.k0n = k0n;
      b.st = st;
      b.slow = 1;
    }
  };
  auto bar1_sync = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(NTG) : "memory"); };
  auto bar2_sync = [&]() { asm volatile("bar.sync 2, %0;" ::"r"(NTG) : "memory"); };
  auto bar2_arrive = [&]() { asm volatile("bar.arrive 2, %0;" ::"r"(NTG) : "memory"); };

  // ---- passes ------------------------------------------------------------------
  auto input_pass = [&](auto m_c, const double K0) {
    constexpr int MI = decltype(m_c)::value;
#pragma unroll
    for (int j = 0; j < kAhMaxM; ++j) s[j] = 0.0;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int li0 = (q * NTG + gtid) * 2;
      const bool ok = li0 < len;
      const double2 xv = *reinterpret_cast<const double2*>(buf + li0);
      const double u0 = ok ? xv.x - K0 : 0.0, u1 = ok ? xv.y - K0 : 0.0;
      v[2 * q] = u0;
      v[2 * q + 1] = u1;
      ah_acc<MI>(s, u0);
      ah_acc<MI>(s, u1);
    }
  };
  // first half of a stage pass: v <- (fma(v, ka, aa))^3 = y_{s+1} (unshifted)
  auto half_pass = [&](const AhCoefA& ca) {
    if (skip_passes) return;
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = ah_cube(fma(v[e], ca.ka, ca.aa));
  };
  // mid pass: iteration s+1, store y_{s+2} - kn, power sums S_1..S_MN
  auto mid_pass = [&](auto m_c, const AhCoefB& c) {
    constexpr int MN = decltype(m_c)::value;
#pragma unroll
    for (int j = 0; j < kAhMaxM; ++j) s[j] = 0.0;
    if (skip_passes) {
      s[0] = 1e-3 * gtid;
      s[1] = 1.0;
      return;
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const bool ok = valid(q);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double z2 = fma(v[2 * q + h], c.kb, c.bb);
        double w = fma(z2 * z2, z2, -c.kn);
        w = ok ? w : 0.0;
        v[2 * q + h] = w;
        ah_acc<MN>(s, w);
      }
    }
  };
  // last pass: Y = y_{T+1}, argmax, Z = Y * rn -> HBM, X(next) - k0n -> registers
  // with its power sums S_1..S_MI (stale buffer data when there is no next row:
  // those sums are never used)
  double best = -HUGE_VAL;
  int bslot = -1;
  auto last_pass = [&](auto two_c, auto m_c, const AhCoefB& c, double* zrow) {
    constexpr bool TWO = decltype(two_c)::value;
    constexpr int MI = decltype(m_c)::value;
#pragma unroll
    for (int j = 0; j < kAhMaxM; ++j) s[j] = 0.0;
    best = -HUGE_VAL;
    bslot = -1;
    if (skip_passes) {
      s[0] = 1e-3 * gtid;
      s[1] = 1.0;
      best = 1.0;
      bslot = 0;
      return;
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int li0 = (q * NTG + gtid) * 2;
      const bool ok = li0 < len;
      const double2 xn = *reinterpret_cast<const double2*>(buf + li0);
      double o[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double y = TWO ? ah_cube(fma(v[2 * q + h], c.kb, c.bb)) : v[2 * q + h];
        if (ok && y > best) {  // slots in increasing element order: strict > keeps the lowest index
          best = y;
          bslot = 2 * q + h;
        }
        o[h] = y * c.rn;
      }
      if (ok) *reinterpret_cast<double2*>(buf + li0) = make_double2(o[0], o[1]);
      const double u0 = ok ? xn.x - c.k0n : 0.0, u1 = ok ? xn.y - c.k0n : 0.0;
      v[2 * q] = u0;
      v[2 * q + 1] = u1;
      ah_acc<MI>(s, u0);
      ah_acc<MI>(s, u1);
    }
  };
  auto dispatch_M = [&](int m, auto&& f) {
    if (m == 3) f(IntC<3>());
    else if (m == 6) f(IntC<6>());
    else f(IntC<9>());
  };

  int64_t row = cid;
  if (row >= a.B) return;  // (never: the host launches min(B, resident) clusters)

  // ---- prologue: the cluster's first row -------------------------------------
  double K0 = k0_of(row);
  if (dma) load_row(row, false);
  ptx::mbar_wait_cta(bar_load, load_par);
  load_par ^= 1u;
  dispatch_M(M0, [&](auto m_c) { input_pass(m_c, K0); });
  {
    const int64_t nx = row + ncl;
    auto side = [&]() {
      if (nx < a.B) load_row(nx, false);
    };
    dispatch_M(M0, [&](auto m_c) {
      ah_push<NTG, decltype(m_c)::value, true>(s, -HUGE_VAL, 0x7fffffffffffffffLL, cb, xround, rank, C, gtid, side);
    });
    if (warp != 0) ++xround;
  }

  // control-warp state: the previous row's status, waiting for its argmax
  int64_t row_prev = -1;
  int st_prev = PAM_OK;
  // control warp: K0 of the row after this one, one sample per lane (lanes 0..7),
  // summed in lane order only when it is needed (the loads stay in flight)
  auto k0_sample = [&](int64_t r) -> double {
    return (lane < 8 && r < a.B) ? __ldg(X + r * a.ldx + ((int64_t)lane * n) / 8) * 0.125 : 0.0;
  };
  auto k0_sum = [&](double smp) -> double {
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += __shfl_sync(FULL, smp, j);
    return t;
  };
  double k0_pf = (warp == 0) ? k0_sample(row + ncl) : 0.0;
#ifdef PAM_TRACE_BUILD
  int64_t lrow = 0;
#endif
  for (; row < a.B; row += ncl) {
    const int64_t next = row + ncl;
    const bool has_next = next < a.B;
#ifdef PAM_TRACE_BUILD
    long long* tr = (a.trace && lrow < kTraceRows)
                        ? a.trace + ((int64_t)blockIdx.x * kTraceRows + lrow) * kTraceEvents
                        : nullptr;
    ++lrow;
#else
    long long* tr = nullptr;
#endif
    PAM_TRACE(tr, 0);
    // input shift of the next row: its samples were loaded a row ago (HBM
    // latency stays off the chain); start the loads for the row after it
    double k0n = 0.0;
    if (warp == 0) {
      k0n = k0_sum(k0_pf);
      k0_pf = k0_sample(next + ncl);
    }
    int st = PAM_OK;
    for (int i = 0; i < NS; ++i) {
      const bool last_stage = i == NS - 1;
      const int M = ah_stage_M(i, T);
      // ---- control warp: records + phase A -----------------------------------
      double Sl = 0.0;
      AhCoefA ca;
      if (warp == 0) {
        double bv = 0.0;
        long long bi = 0;
        Sl = ah_wait<NTG>(cb, xround, M, i == 0, C, lane, pos_bytes(arm_pos), bv, bi);
        arm_pos = arm_pos + 1 == NS ? 0 : arm_pos + 1;
        PAM_TRACE(tr, i == 0 ? 1 : 14);
        PAM_GTRACE(tr, i == 0 ? 22 : 21);
        if (i == 0 && row_prev >= 0 && rank == 0 && lane == 0) {
          if (a.argmax) a.argmax[row_prev] = (st_prev == PAM_OK) ? (int32_t)bi : -1;
          if (a.status) a.status[row_prev] = st_prev;
        }
        const double Kc = (i == 0) ? K0 : rp.kshift[2 * i];
        ca = phase_a(i, Sl, Kc, st);
        PAM_TRACE(tr, i == 0 ? 2 : 15);
        bar2_arrive();
      } else {
        bar2_sync();
        ca = cb->bca;
      }
      if (ca.slow) {
        slow_a(i, ca, cb->kc);  // all threads: identical results
        // (the slow path's barriers order the bca reads before any rewrite)
      }
      // ---- phase B on the control warp while the others run the first half -------
      if (warp == 0) {
        if (!ca.slow) phase_b(i, Sl, ca, last_stage ? k0n : 0.0);
        else phase_b_slow(i, ca.st, last_stage ? k0n : 0.0);
        PAM_TRACE(tr, i == 0 ? 3 : 16);
      }
      half_pass(ca);
      bar1_sync();
      AhCoefB c = cb->bcb;
      if (c.slow) slow_b(i, c, c.st);
      if (warp == 0) st = c.st;
      if (!last_stage) {
        dispatch_M(ah_stage_M(i + 1, T), [&](auto m_c) {
          mid_pass(m_c, c);
          PAM_TRACE(tr, 4);
          auto side = [&]() {  // first mid exchange of the row: X(next) behind the Z(prev) store
            if (i == 0 && has_next && row_prev >= 0) load_row(next, true);
          };
          ah_push<NTG, decltype(m_c)::value, false>(s, 0.0, 0LL, cb, xround, rank, C, gtid, side);
        });
        PAM_TRACE(tr, 5);
        PAM_GTRACE(tr, 20);
        if (warp != 0) ++xround;  // keep the round counter in step with warp 0
      } else {
        if (has_next) {
          ptx::mbar_wait_cta(bar_load, load_par);  // X(next) has landed (issued a row ago)
          load_par ^= 1u;
        }
        PAM_TRACE(tr, 9);
        double* zrow = Zo + row * a.ldz + base;
        if (2 * i + 2 <= T) {
          dispatch_M(M0, [&](auto m_c) { last_pass(BoolC<true>(), m_c, c, zrow); });
        } else {
          dispatch_M(M0, [&](auto m_c) { last_pass(BoolC<false>(), m_c, c, zrow); });
        }
        ptx::fence_proxy_async_smem();  // Z in the buffer -> visible to the bulk store after the barrier
        PAM_TRACE(tr, 10);
        const long long bidx =
            bslot < 0 ? 0x7fffffffffffffffLL : base + (long long)(((bslot / 2) * NTG + gtid) * 2 + (bslot & 1));
        const int64_t nx2 = next + ncl;
        auto side = [&]() {
          store_row(row);  // Z(row) now sits in the buffer (X(next) is in registers)
          if (NS == 1 && has_next && nx2 < a.B) load_row(nx2, true);  // no mid exchange to hook into
        };
        dispatch_M(M0, [&](auto m_c) {
          ah_push<NTG, decltype(m_c)::value, true>(s, best, bidx, cb, xround, rank, C, gtid, side);
        });
        PAM_TRACE(tr, 11);
        PAM_GTRACE(tr, 23);
        if (warp != 0) ++xround;
        row_prev = row;
        st_prev = st;
        K0 = c.k0n;
      }
    }
  }
  // ---- epilogue: the last row's argmax ----------------------------------------
  if (warp == 0) {
    double bv = 0.0;
    long long bi = 0;
    (void)ah_wait<NTG>(cb, xround, M0, true, C, lane, pos_bytes(arm_pos), bv, bi);
    if (rank == 0 && lane == 0) {
      if (a.argmax) a.argmax[row_prev] = (st_prev == PAM_OK) ? (int32_t)bi : -1;
      if (a.status) a.status[row_prev] = st_prev;
    }
  }
  if (dma) ptx::bulk_wait_all();  // the last Z store has left the buffer
  ptx::cluster_sync();            // no CTA leaves while a peer may still push into it
}

}  // namespace pam
