// cutmax_kernel.cuh — fused, row-resident batched CutMax for sm_100a.
//
// Replaces core.cutmax / core.cutmaxStep (Alg. 1).
//
// Geometry.  One logit row is owned by one thread-block cluster of C CTAs
// (C = 1..16).  CTA `rank` owns the contiguous slice [rank*L, min(n,(rank+1)*L)).
// Each of the NTG threads keeps E elements of the slice in registers for all T
// iterations: HBM is read once (1-D TMA bulk copy into the CTA's shared-memory
// row buffer, prefetched one row ahead) and written once (TMA bulk store).
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
// Exchange.  Each warp butterfly-reduces its lanes into a per-warp partial;
// after a CTA barrier warp 0 combines the partials and pushes ONE 32-byte
// record (sums + argmax candidate) into slot [rank] of every CTA of the
// cluster with st.async (DSMEM), completing on the destination's mbarrier;
// every warp then combines the C records in the same butterfly order.
// xor-butterflies leave bit-identical values in every lane (IEEE addition is
// commutative), so all CTAs compute identical mu and s2 without a broadcast.
//
// Row pipeline (TMA path).  Per row, T exchanges — the input statistics ride
// on the previous row's last exchange:
//   pass t (t < T-1): update + moments            -> exchange t
//   pass T-1: Y^(T+1), sum Y, argmax             -> push (no wait)
//   swap: unnormalised Y(r) -> row buffer, X(r+1) - K0(r+1) -> registers,
//         moments of X(r+1)                       -> push; wait both
//   row r+1, pass 0 also scales the buffer by inv(sum Y(r)) = Z(r); the DMA
//   thread then streams Z(r) out (4 bulk-store chunks) and, chunk by chunk as
//   the store has read them, streams X(r+2) in.
// Normalising one pass late lets the row-boundary exchange carry both rows,
// and the prologue's input pass + exchange is needed only for a cluster's
// first row.
//
// Element update (z = (y-mu)/(c sigma) + 1, y' = z^p):
//     z = fma(v, k, b)  with k = inv_sigma/c, b = 1 - dm*k
//     v' = z^p - K'     (p = 3: fma(z*z, z, -K'))
// which is 5 fp64 instructions per element per iteration including the two
// accumulations (the oracle evaluates the same algebra in textbook order; the
// difference is rounding only and is covered by the 1e-12 normwise tolerance).
#pragma once

#include <stdint.h>
#include <stdio.h>
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
  double eps_stop;  // early stop when max Y / sum Y >= 1 - eps_stop; 0 = off (generic flow only)
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
  int32_t ctrl_offset;  // byte offset of the control block (after the row buffer)
  int32_t tma;          // 1: TMA bulk loads/stores (16-byte aligned rows), 0: direct loads/stores
  double inv_n;         // 1/n
  long long* trace;     // debug: per-CTA phase timestamps (pam_set_trace_buffer), normally null
  RowParams rp;
};

// One 32-byte exchange record per (cluster rank): partial sums (a, b) and an
// argmax candidate (value, index) used by the last exchange of a row.
struct __align__(16) XchRecord {
  double2 ab;
  double2 cand;  // (value, index bits)
#ifdef PAM_CHECKED_BUILD
  double2 tag;   // checked build: (round, sender rank), verified by the receiver
#endif
};
// tx bytes one sender completes on a receiver's exchange mbarrier
#ifdef PAM_CHECKED_BUILD
constexpr uint32_t kXchBytes = 48;
#else
constexpr uint32_t kXchBytes = 32;
#endif

// Checked build (make checked -> libpam_checked.so; compute-sanitizer is closed
// on the GPU pool): protocol and bounds assertions that trap with a message.
#ifdef PAM_CHECKED_BUILD
#define PAM_CHECK(cond)                                                                                  \
  do {                                                                                                   \
    if (!(cond)) {                                                                                       \
      printf("PAM_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, (int)blockIdx.x, \
             (int)threadIdx.x);                                                                          \
      __trap();                                                                                          \
    }                                                                                                    \
  } while (0)
#else
#define PAM_CHECK(cond) \
  do {                  \
  } while (0)
#endif

// Coefficients the control warp publishes for the next pass (p = 3 flow).
struct __align__(16) Bcast {
  double ke, be, dm, re;
  int flag;  // 1: the exact second pass about dm is needed first
  int st;    // row status so far (generic flow)
  int pad[2];
};

struct __align__(16) ControlBlock {
  XchRecord xch[2][16];  // exchange slots per cluster rank, double-buffered by round parity
  Bcast bc;              // control-warp broadcast (p = 3 flow)
  double2 xin[16];       // next row's input sums per cluster rank (row-boundary exchange)
  double2 wred[32];      // per-warp partial sums (CTA pre-reduction; sampler token gather)
  double2 wcand[32];     // per-warp argmax candidates
  double2 wred2[32];     // per-warp partials of the next row's input sums
  double2 gat[16][2];    // all-gather records (sampler: token candidate + max x)
  double2 tin[2][16];    // input top-2 records (TieWarning) per cluster rank, by local row parity
  double2 wt2[32];       // per-warp top-2 partials
  unsigned long long mb_t[2];
  long long unc_rows[16];  // rows whose TieWarning the key screen left undecided (settled at kernel end)
  int unc_n;               // their count (> 16: re-scan every row of the cluster)
  // control warp: a finished row whose argmax / status is written in the next
  // row's first exchange wait (kept here, not in registers)
  long long fin_row, fin_best;
  int fin_st, fin_pending;
  // control warp's scalar state of the lean p = 3 kernel (cutmax_p3_kernel.cuh)
  double p3_S, p3_Q, p3_R, p3_dm, p3_s2, p3_m3, p3_e1, p3_w;
  int p3_st;
  unsigned long long mb_load;
  unsigned long long mb_x[2];
  unsigned long long mb_g;
  unsigned long long mb_in;
};

// Debug phase tracing (builds with -DPAM_TRACE_BUILD only; tools/trace.py):
// thread 0 of each CTA stamps clock64() at phase boundaries of its first
// kTraceRows rows.  Compiled out otherwise so it costs no registers.
constexpr int kTraceRows = 8, kTraceEvents = 32;
#ifdef PAM_TRACE_BUILD
#define PAM_TRACE(tr, k)                                   \
  do {                                                     \
    if ((tr) != nullptr && gtid == 0) (tr)[k] = clock64(); \
  } while (0)
#define PAM_TRACE_DMA(tr, k)                 \
  do {                                       \
    if ((tr) != nullptr) (tr)[k] = clock64(); \
  } while (0)
#else
#define PAM_TRACE(tr, k) \
  do {                   \
  } while (0)
#define PAM_TRACE_DMA(tr, k) \
  do {                       \
  } while (0)
#endif

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

__device__ __forceinline__ int lane_of(int tid) { return tid & 31; }

__device__ __forceinline__ bool cand_better(double v, long long i, double bv, long long bi) {
  return (v > bv) || (v == bv && i < bi);
}

// xor-butterfly over aligned WIDTH-lane groups (WIDTH a power of two <= 32):
// every lane ends with the combination of its group, and because IEEE addition
// and the argmax rule are commutative, all lanes of a group hold bit-identical
// values.
template <int WIDTH>
__device__ __forceinline__ void bfly_sum1(double& a) {
#pragma unroll
  for (int m = WIDTH / 2; m > 0; m >>= 1) a += __shfl_xor_sync(0xffffffffu, a, m);
}

template <int WIDTH>
__device__ __forceinline__ void bfly_sum2(double& a, double& b) {
#pragma unroll
  for (int m = WIDTH / 2; m > 0; m >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, m);
    b += __shfl_xor_sync(0xffffffffu, b, m);
  }
}

// Warp argmax in the (value desc, index asc) order of cand_better with three
// REDUX steps on a monotone 64-bit key of the value (+0.0 and -0.0 compare
// equal; NaN candidates never occur: the passes only admit y > best).  Every
// lane returns the winner.  Indices must be < 2^32 - 1 (n <= 2^30); the
// sentinel index (> that) survives only when every candidate carries it.
__device__ __forceinline__ void warp_argmax(double& v, long long& ix) {
  constexpr unsigned FULL = 0xffffffffu;
  unsigned long long b = (unsigned long long)__double_as_longlong(v + 0.0);
  b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
  const unsigned mhi = __reduce_max_sync(FULL, hi);
  const unsigned mlo = __reduce_max_sync(FULL, hi == mhi ? lo : 0u);
  const bool win = hi == mhi && lo == mlo;
  const unsigned i32 = (win && ix >= 0 && ix < 0xffffffffLL) ? (unsigned)ix : 0xffffffffu;
  const unsigned mi = __reduce_min_sync(FULL, i32);
  unsigned long long k = ((unsigned long long)mhi << 32) | mlo;
  k = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  v = __longlong_as_double((long long)k);
  ix = mi == 0xffffffffu ? 0x7fffffffffffffffLL : (long long)mi;
}

// Argmax over aligned WIDTH-lane groups.  Every caller fills the lanes outside
// a group with copies of the group or neutral candidates, so the whole-warp
// REDUX form (warp_argmax) gives each group's result.
template <int WIDTH>
__device__ __forceinline__ void bfly_argmax(double& best, long long& besti) {
  warp_argmax(best, besti);
}

// ---------------------------------------------------------------------------
// Input top-2 (TieWarning: the top-2 gap of the input < 1e-9).
// (m1, m2) = the largest and second-largest entry of the multiset (a
// duplicated maximum gives m2 = m1), exactly as the oracle's orc_tie_warning.
// min/max are exact and commutative, so every merge order gives the same pair.
__device__ __forceinline__ double emax(double a, double b) { return fmax(a, b); }
__device__ __forceinline__ double emin(double a, double b) { return fmin(a, b); }
__device__ __forceinline__ float emax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ float emin(float a, float b) { return fminf(a, b); }
template <typename Elem>
__device__ __forceinline__ void top2_add(Elem& m1, Elem& m2, Elem x) {
  m2 = emax(m2, emin(m1, x));
  m1 = emax(m1, x);
}
__device__ __forceinline__ void top2_merge(double& a1, double& a2, double b1, double b2) {
  a2 = fmax(fmin(a1, b1), fmax(a2, b2));
  a1 = fmax(a1, b1);
}
template <int WIDTH>
__device__ __forceinline__ void bfly_top2(double& a1, double& a2) {
#pragma unroll
  for (int m = WIDTH / 2; m > 0; m >>= 1) {
    const double b1 = __shfl_xor_sync(0xffffffffu, a1, m), b2 = __shfl_xor_sync(0xffffffffu, a2, m);
    top2_merge(a1, a2, b1, b2);
  }
}
__device__ __forceinline__ int tie_flag(int st, double2 t) {
  return (st == PAM_OK && t.x - t.y < 1e-9) ? PAM_ROW_FLAG_TIE : 0;
}

// ---------------------------------------------------------------------------
// Input top-2 screen of the rows kernel (TieWarning).  Each
// thread keeps the top-2 of a 32-bit image of its inputs -- the high word of a
// double (sign, exponent, 20 mantissa bits), or a whole float -- on the FP32
// pipe (hiword_f below) instead of three fp64 min/max per element on the DP
// pipe the passes saturate; warps combine signed order keys of those images
// (fkey) with REDUX.  For fp32 rows the image is exact; for fp64 each key
// brackets its value, and tie_decide() turns the cluster's top-2 keys
// (K1 >= K2) into a certain flag or "undecided" (the brackets straddle the
// 1e-9 threshold, e.g. a duplicated maximum), which the kernel settles with an
// exact fp64 re-scan of the row at its end.
__device__ __forceinline__ void top2k_add(int& k1, int& k2, int k) {
  k2 = max(k2, min(k1, k));
  k1 = max(k1, k);
}
// The per-element screen runs on the FP32 pipe: the high word of a double,
// read as an fp32 bit pattern (sign, 8 of the 11 exponent bits, ...), orders
// exactly like the double's high word (sign-magnitude both ways).  Patterns
// that read as fp32 Inf / NaN need |x| >= 2^1017, where the row's variance
// overflows (status RANGE, no TieWarning).  fp32 rows use the value itself.
__device__ __forceinline__ float hiword_f(double x) { return __int_as_float(__double2hiint(x)); }
__device__ __forceinline__ float hiword_f(float x) { return x; }
__device__ __forceinline__ void top2f_add(float& m1, float& m2, float x) {
  m2 = fmaxf(m2, fminf(m1, x));
  m1 = fmaxf(m1, x);
}
// order key of a screen value (int order = value order; -inf -> a finite key)
__device__ __forceinline__ int fkey(float f) {
  const int h = __float_as_int(f);
  return h ^ ((h >> 31) & 0x7fffffff);
}
// Multiset top-2 of the lanes' (k1 >= k2) pairs; every lane gets the result.
// Lanes without data must hold INT_MIN (the key of no finite value).
__device__ __forceinline__ void top2k_warp(int& k1, int& k2) {
  constexpr unsigned FULL = 0xffffffffu;
  const int m1 = __reduce_max_sync(FULL, k1);
  const unsigned dup = __ballot_sync(FULL, k1 == m1);
  const int m2 = __reduce_max_sync(FULL, k1 == m1 ? k2 : k1);
  k2 = __popc(dup) > 1 ? m1 : m2;
  k1 = m1;
}
__device__ __forceinline__ unsigned long long pack_keys(int k1, int k2) {
  return ((unsigned long long)(unsigned)k1 << 32) | (unsigned)k2;
}
__device__ __forceinline__ int2 unpack_keys(unsigned long long u) {
  return make_int2((int)(unsigned)(u >> 32), (int)(unsigned)u);
}
// Bracket [lo, hi] of the values whose key is k (fp64 high-word keys).
__device__ __forceinline__ void key_bracket(int k, double& lo, double& hi) {
  const int h = k ^ ((k >> 31) & 0x7fffffff);  // the map is an involution
  const double a = __hiloint2double(h, 0), b = __hiloint2double(h, (int)0xffffffff);
  lo = fmin(a, b);
  hi = fmax(a, b);
}
// 0: no tie, 1: tie (oracle: m1 - m2 < 1e-9), 2: undecided (fp64 only).
// fl() is monotone, so a bound on the exact gap bounds the oracle's rounded one.
template <typename Elem>
__device__ __forceinline__ int tie_decide(int st, int K1, int K2) {
  if (st != PAM_OK) return 0;
  if (sizeof(Elem) == 4) {  // exact keys: the float values themselves
    const int h1 = K1 ^ ((K1 >> 31) & 0x7fffffff), h2 = K2 ^ ((K2 >> 31) & 0x7fffffff);
    return ((double)__int_as_float(h1) - (double)__int_as_float(h2) < 1e-9) ? 1 : 0;
  }
  double l1, h1, l2, h2;
  key_bracket(K1, l1, h1);
  key_bracket(K2, l2, h2);
  if (l1 - h2 >= 1e-9) return 0;
  if (h1 - l2 < 1e-9) return 1;
  return 2;
}
// The same decision from the keys of the SHIFTED input v = fl(x - K0) (the
// lean p = 3 kernel screens its first pass, where v is in registers).  v is a
// monotone function of x, so the top-2 of v are the images of the top-2 of x,
// and x1 - x2 = (v1 - v2) + (e1 - e2) with |e_i| <= ulp(v_i) / 2 (fp32 rows:
// fp32 ulps).  The slack below covers those and the rounding of this bound.
template <typename Elem>
__device__ __forceinline__ int tie_decide_shifted(int st, int K1, int K2) {
  if (st != PAM_OK) return 0;
  double l1, h1, l2, h2;
  if (sizeof(Elem) == 4) {
    const int a1 = K1 ^ ((K1 >> 31) & 0x7fffffff), a2 = K2 ^ ((K2 >> 31) & 0x7fffffff);
    l1 = h1 = (double)__int_as_float(a1);
    l2 = h2 = (double)__int_as_float(a2);
  } else {
    key_bracket(K1, l1, h1);
    key_bracket(K2, l2, h2);
  }
  const double rel = sizeof(Elem) == 4 ? 0x1p-22 : 0x1p-50;
  const double slack = (fabs(l1) + fabs(h1) + fabs(l2) + fabs(h2)) * rel + 0x1p-1000;
  if ((l1 - h2) - slack >= 1e-9) return 0;
  if ((h1 - l2) + slack < 1e-9) return 1;
  return 2;
}

struct KeyPush {
  bool on;
  int k1, k2;
  uint32_t slot;
  bool stashed = false;  // the warps already stashed their records (wt2): only the CTA combine + send remain
};
// Top-2 side record of an exchange: the CTA's pair, butterflied over each
// warp, goes to slot `slot` (the row's local parity) of every CTA with its own
// mbarrier mb_t[slot]; top2_wait (warp 0, at the row's status write) combines
// the C records.  Exactly one record per row, so no phase is ever skipped.
struct Top2Push {
  bool on;
  double m1, m2;
  uint32_t slot;
};
__device__ __forceinline__ Top2Push no_top2() { return Top2Push{false, 0.0, 0.0, 0u}; }

// `phases` holds the current mbarrier phase of slot s in bit s.
__device__ __forceinline__ double2 top2_wait(ControlBlock* cb, const uint32_t slot, uint32_t& phases,
                                             const uint32_t C, const int gtid) {
  const int lane = gtid & 31;
  ptx::mbar_wait_cta(ptx::smem_addr(&cb->mb_t[slot]), (phases >> slot) & 1u);
  phases ^= 1u << slot;
  const int src = lane & 15;
  const bool have = src < (int)C;
  const double2 rec = cb->tin[slot][have ? src : 0];
  __syncwarp();
  if (gtid == 0) ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_t[slot]), C * 16u);  // arm row + 2
  double m1 = have ? rec.x : -HUGE_VAL, m2 = have ? rec.y : -HUGE_VAL;
  bfly_top2<16>(m1, m2);
  return make_double2(m1, m2);
}

// Row lr's input top-2 keys: slot lr & 1, the (lr >> 1)-th phase of that slot's
// mbarrier (stateless, so any warp can wait; lane 0 of the caller re-arms).
__device__ __forceinline__ int2 top2k_wait_row(ControlBlock* cb, const int64_t lr, const uint32_t C, const int lane) {
  const uint32_t slot = (uint32_t)(lr & 1);
  ptx::mbar_wait_cta(ptx::smem_addr(&cb->mb_t[slot]), (uint32_t)((lr >> 1) & 1));
  const bool have = lane < (int)C;
  const int2 rec = unpack_keys((unsigned long long)__double_as_longlong(cb->tin[slot][have ? lane : 0].x));
  __syncwarp();
  if (lane == 0) ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_t[slot]), C * 16u);  // arm row + 2
  int k1 = have ? rec.x : INT_MIN, k2 = have ? rec.y : INT_MIN;
  top2k_warp(k1, k2);
  return make_int2(k1, k2);
}
__device__ __forceinline__ int2 top2k_wait(ControlBlock* cb, const uint32_t slot, uint32_t& phases, const uint32_t C,
                                           const int gtid) {
  const int lane = gtid & 31;
  ptx::mbar_wait_cta(ptx::smem_addr(&cb->mb_t[slot]), (phases >> slot) & 1u);
  phases ^= 1u << slot;
  const bool have = lane < (int)C;
  const int2 rec = unpack_keys((unsigned long long)__double_as_longlong(cb->tin[slot][have ? lane : 0].x));
  __syncwarp();
  if (gtid == 0) ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_t[slot]), C * 16u);  // arm row + 2
  int k1 = have ? rec.x : INT_MIN, k2 = have ? rec.y : INT_MIN;
  top2k_warp(k1, k2);
  return make_int2(k1, k2);
}

// Per-warp stash and CTA-level push of a top-2 side record: exact fp64 pairs
// (Top2Push, sampler) or order keys (KeyPush, rows kernel).
__device__ __forceinline__ bool t2_stashed(const Top2Push&) { return false; }
__device__ __forceinline__ bool t2_stashed(const KeyPush& t) { return t.stashed; }
__device__ __forceinline__ void t2_warp(Top2Push& t) { bfly_top2<32>(t.m1, t.m2); }
__device__ __forceinline__ void t2_warp(KeyPush& t) { top2k_warp(t.k1, t.k2); }
__device__ __forceinline__ void t2_stash(ControlBlock* cb, int warp, const Top2Push& t) {
  cb->wt2[warp] = make_double2(t.m1, t.m2);
}
__device__ __forceinline__ void t2_stash(ControlBlock* cb, int warp, const KeyPush& t) {
  cb->wt2[warp] = make_double2(__longlong_as_double((long long)pack_keys(t.k1, t.k2)), 0.0);
}
template <int NW>
__device__ __forceinline__ void t2_send(ControlBlock* cb, int lane, uint32_t rank, uint32_t C, const Top2Push& t) {
  const double2 w2 = cb->wt2[lane & (NW - 1)];
  double m1 = w2.x, m2 = w2.y;
  bfly_top2<NW>(m1, m2);
  if (lane < (int)C)
    ptx::st_async_f64x2(ptx::mapa(ptx::smem_addr(&cb->tin[t.slot][rank]), (uint32_t)lane), m1, m2,
                        ptx::mapa(ptx::smem_addr(&cb->mb_t[t.slot]), (uint32_t)lane));
}
template <int NW>
__device__ __forceinline__ void t2_send(ControlBlock* cb, int lane, uint32_t rank, uint32_t C, const KeyPush& t) {
  int k1 = INT_MIN, k2 = INT_MIN;
  if (lane < NW) {
    const int2 r = unpack_keys((unsigned long long)__double_as_longlong(cb->wt2[lane].x));
    k1 = r.x;
    k2 = r.y;
  }
  top2k_warp(k1, k2);
  if (lane < (int)C)
    ptx::st_async_b64x2(ptx::mapa(ptx::smem_addr(&cb->tin[t.slot][rank]), (uint32_t)lane), pack_keys(k1, k2), 0ull,
                        ptx::mapa(ptx::smem_addr(&cb->mb_t[t.slot]), (uint32_t)lane));
}

// ---------------------------------------------------------------------------
// Cluster exchange, split in two so independent work can run between the push
// and the wait.  All NTG threads of the CTA call both halves.
//
// xch_push: warp butterfly -> per-warp partial in smem -> CTA barrier -> warp 0
// combines the NW partials and pushes one 32-byte record into slot [rank] of
// every CTA (st.async, complete_tx on the destination's mbarrier).  `side` runs
// on lane 0 of the last warp right after the barrier (the DMA thread's hook:
// bulk stores / loads issued there stay off warp 0's critical path).
struct NoSide {
  __device__ __forceinline__ void operator()() const {}
};

// Exchange payloads: two sums; three sums (the third rides in the candidate
// slot); or two sums plus the lexicographic (value desc, index asc) argmax.
enum XchMode { kSum2 = 0, kSum3 = 1, kArgmax = 2, kTop2 = 3 };  // kTop2: (a, b) = exact top-2 pair

// kSum3 with third == false behaves as kSum2 (one code copy for both in the p = 3 row loop).
template <int NTG, int MODE, typename Ch, typename Side = NoSide, typename T2 = Top2Push>
__device__ __forceinline__ void xch_push(double a, double b, double c, long long ci_, Ch* cb,
                                         const uint32_t round, const uint32_t rank, const uint32_t C, const int gtid,
                                         const Side& side = Side(), const bool third = true,
                                         T2 t2 = T2{false}) {
  constexpr int NW = NTG / 32;
  const int lane = gtid & 31, warp = gtid >> 5;
  long long ci = ci_;
  if (MODE == kTop2)
    bfly_top2<32>(a, b);
  else
    bfly_sum2<32>(a, b);
  if (MODE == kArgmax) bfly_argmax<32>(c, ci);
  if (MODE == kSum3 && third) bfly_sum1<32>(c);
  if (t2.on && !t2_stashed(t2)) t2_warp(t2);
  if (lane == 0) {
    cb->wred[warp] = make_double2(a, b);
    if (MODE == kArgmax || (MODE == kSum3 && third)) cb->wcand[warp] = make_double2(c, __longlong_as_double(ci));
    if (t2.on && !t2_stashed(t2)) t2_stash(cb, warp, t2);
  }
  __syncthreads();
  const uint32_t par = round & 1u;
  if (warp == 0) {
    const double2 w = cb->wred[lane & (NW - 1)];
    double ca = w.x, cbv = w.y;
    if (MODE == kTop2)
      bfly_top2<NW>(ca, cbv);
    else
      bfly_sum2<NW>(ca, cbv);
    double cv = -HUGE_VAL;
    long long cix = 0x7fffffffffffffffLL;
    if (MODE == kArgmax || (MODE == kSum3 && third)) {
      const double2 wc = cb->wcand[lane & (NW - 1)];
      cv = wc.x;
      cix = __double_as_longlong(wc.y);
      if (MODE == kArgmax) bfly_argmax<NW>(cv, cix);
      if (MODE == kSum3) bfly_sum1<NW>(cv);
    }
    if (lane < (int)C) {
      const uint32_t bar = ptx::mapa(ptx::smem_addr(&cb->mb_x[par]), (uint32_t)lane);
      ptx::st_async_f64x2(ptx::mapa(ptx::smem_addr(&cb->xch[par][rank].ab), (uint32_t)lane), ca, cbv, bar);
      ptx::st_async_b64x2(ptx::mapa(ptx::smem_addr(&cb->xch[par][rank].cand), (uint32_t)lane),
                          (uint64_t)__double_as_longlong(cv), (uint64_t)cix, bar);
#ifdef PAM_CHECKED_BUILD
      ptx::st_async_b64x2(ptx::mapa(ptx::smem_addr(&cb->xch[par][rank].tag), (uint32_t)lane), (uint64_t)round,
                          (uint64_t)rank, bar);
#endif
    }
    if (t2.on) t2_send<NW>(cb, lane, rank, C, t2);
  } else if (warp == NW - 1 && lane == 0) {
    side();
  }
}

// xch_wait: wait for the C records of this round, re-arm the barrier for
// round + 2 and combine the records (16-lane butterfly, same order everywhere).
// Returns (a, b); c / ci receive the third sum or the argmax.
template <int MODE, typename Ch>
__device__ __forceinline__ double2 xch_wait(double& c, long long& ci, Ch* cb, uint32_t& round,
                                            const uint32_t C, const int gtid, const bool third = true) {
  const int lane = gtid & 31;
  const uint32_t par = round & 1u, ph = (round >> 1) & 1u;
  ptx::mbar_wait_cta(ptx::smem_addr(&cb->mb_x[par]), ph);
  if (gtid == 0) ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[par]), C * kXchBytes);  // arm round+2
  const int src = lane & 15;
  const bool have = src < (int)C;
  const XchRecord rec = cb->xch[par][have ? src : 0];
#ifdef PAM_CHECKED_BUILD
  if (have) {  // the record of every sender is this round's
    PAM_CHECK((uint64_t)__double_as_longlong(rec.tag.x) == (uint64_t)round);
    PAM_CHECK((uint64_t)__double_as_longlong(rec.tag.y) == (uint64_t)src);
  }
#endif
  double a = have ? rec.ab.x : (MODE == kTop2 ? -HUGE_VAL : 0.0);
  double b = have ? rec.ab.y : (MODE == kTop2 ? -HUGE_VAL : 0.0);
  if (MODE == kTop2)
    bfly_top2<16>(a, b);
  else
    bfly_sum2<16>(a, b);
  if (MODE == kArgmax) {
    c = have ? rec.cand.x : -HUGE_VAL;
    ci = have ? __double_as_longlong(rec.cand.y) : 0x7fffffffffffffffLL;
    bfly_argmax<16>(c, ci);
  }
  if (MODE == kSum3 && third) {
    c = have ? rec.cand.x : 0.0;
    bfly_sum1<16>(c);
  }
  ++round;
  return make_double2(a, b);
}

template <int NTG, bool ARGMAX, typename Ch, typename T2 = Top2Push>
__device__ __forceinline__ double2 cluster_reduce(double a, double b, double& best, long long& besti, Ch* cb,
                                                  uint32_t& round, const uint32_t rank, const uint32_t C,
                                                  const int gtid, T2 t2 = T2{false}) {
  constexpr int M = ARGMAX ? kArgmax : kSum2;
  xch_push<NTG, M>(a, b, best, besti, cb, round, rank, C, gtid, NoSide(), true, t2);
  return xch_wait<M>(best, besti, cb, round, C, gtid);
}

template <int NTG, typename Ch, typename T2 = Top2Push>
__device__ __forceinline__ double2 cluster_sum2(double a, double b, Ch* cb, uint32_t& round,
                                                const uint32_t rank, const uint32_t C, const int gtid,
                                                T2 t2 = T2{false}) {
  double bv = 0.0;
  long long bi = 0;
  return cluster_reduce<NTG, false>(a, b, bv, bi, cb, round, rank, C, gtid, t2);
}

// Three cluster sums in one exchange.
template <int NTG, typename Ch, typename T2 = Top2Push>
__device__ __forceinline__ double3 cluster_sum3(double a, double b, double c, Ch* cb, uint32_t& round,
                                                const uint32_t rank, const uint32_t C, const int gtid,
                                                T2 t2 = T2{false}) {
  long long ci = 0;
  xch_push<NTG, kSum3>(a, b, c, ci, cb, round, rank, C, gtid, NoSide(), true, t2);
  const double2 r = xch_wait<kSum3>(c, ci, cb, round, C, gtid);
  return make_double3(r.x, r.y, c);
}

// Exact top-2 of (m1, m2) pairs over the cluster (every thread calls it).
template <int NTG, typename Ch>
__device__ __forceinline__ double2 cluster_top2(double m1, double m2, Ch* cb, uint32_t& round, const uint32_t rank,
                                                const uint32_t C, const int gtid) {
  double c = 0.0;
  long long ci = 0;
  xch_push<NTG, kTop2>(m1, m2, c, ci, cb, round, rank, C, gtid);
  return xch_wait<kTop2>(c, ci, cb, round, C, gtid);
}

// Next row's input sums (row-boundary exchange, second record): own per-warp
// slots, own records and mbarrier (mb_in, one phase per row).
template <int NTG>
__device__ __forceinline__ void xin_push(double s, double q, ControlBlock* cb, const uint32_t rank, const uint32_t C,
                                         const int gtid, KeyPush t2) {
  constexpr int NW = NTG / 32;
  const int lane = gtid & 31, warp = gtid >> 5;
  bfly_sum2<32>(s, q);
  t2_warp(t2);
  if (lane == 0) {
    cb->wred2[warp] = make_double2(s, q);
    t2_stash(cb, warp, t2);
  }
  __syncthreads();
  if (warp == 0) {
    const double2 w = cb->wred2[lane & (NW - 1)];
    double cs = w.x, cq = w.y;
    bfly_sum2<NW>(cs, cq);
    if (lane < (int)C) {
      const uint32_t bar = ptx::mapa(ptx::smem_addr(&cb->mb_in), (uint32_t)lane);
      ptx::st_async_f64x2(ptx::mapa(ptx::smem_addr(&cb->xin[rank]), (uint32_t)lane), cs, cq, bar);
    }
    t2_send<NW>(cb, lane, rank, C, t2);
  }
}

__device__ __forceinline__ double2 xin_wait(ControlBlock* cb, uint32_t& in_par, const uint32_t C, const int gtid) {
  const int lane = gtid & 31;
  ptx::mbar_wait_cta(ptx::smem_addr(&cb->mb_in), in_par);
  in_par ^= 1u;
  if (gtid == 0) ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_in), C * 16u);  // arm the next row
  const int src = lane & 15;
  const bool have = src < (int)C;
  const double2 rec = cb->xin[have ? src : 0];
  double s = have ? rec.x : 0.0, q = have ? rec.y : 0.0;
  bfly_sum2<16>(s, q);
  return make_double2(s, q);
}

// ---------------------------------------------------------------------------
// The affine step z = (v - dm) * k + 1 of one element.
//   fp64: z = fma(v, k, b) with b = 1 - dm*k (one instruction; b's rounding
//         error 2^-53 stays far inside the 1e-12 tolerance after p^T growth).
//   fp32: z = fma(v - dm, k, 1): rounding b to fp32 would put a 2^-24 offset
//         into every z (amplified ~p^T), so dm is subtracted first, like the
//         oracle's (z - mu) * k + 1 (oracle.c orc_cutmax_f32).
// `b` is the per-type coefficient from affine_coef().
__device__ __forceinline__ double affine_e(double v, double k, double b) { return fma(v, k, b); }
__device__ __forceinline__ float affine_e(float v, float k, float dm) { return fmaf(v - dm, k, 1.0f); }
template <typename Elem>
__device__ __forceinline__ Elem affine_coef(double bd, double dm) {
  return sizeof(Elem) == 8 ? (Elem)bd : (Elem)dm;
}

// One element update z = affine(v), v' = z^p - K'.  Used for the register
// slice and for the scalar phantom trajectory, so both round identically.
template <typename Elem, int P>
__device__ __forceinline__ Elem cutmax_update(Elem v, Elem k, Elem b, Elem kn, int p) {
  const Elem zz = affine_e(v, k, b);
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

// Input pass: shift the slice by K0 in place and return this thread's
// (sum v, sum v^2).  Phantom slots hold K0 and so contribute exactly 0.
template <typename Elem, int E>
__device__ __forceinline__ double2 input_pass(Elem (&v)[E], const double K0) {
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
  return make_double2((double)sa + (double)sb, (double)qa + (double)qb);
}

// Input pass with the third power sum as well (the p = 3 analytic normaliser
// needs the third central moment of the iterate feeding the last iteration;
// for T = 1 that is the input).
template <typename Elem, int E>
__device__ __forceinline__ double3 input_pass3(Elem (&v)[E], const double K0) {
  const Elem k0 = (Elem)K0;
  Elem sa = 0, sb = 0, qa = 0, qb = 0, ra = 0, rb = 0;
#pragma unroll
  for (int i = 0; i < E; i += 2) {
    const Elem d0 = v[i] - k0, d1 = v[i + 1] - k0;
    v[i] = d0;
    v[i + 1] = d1;
    sa += d0;
    sb += d1;
    const Elem e0 = d0 * d0, e1 = d1 * d1;
    qa += e0;
    qb += e1;
    ra = fma_e(e0, d0, ra);
    rb = fma_e(e1, d1, rb);
  }
  return make_double3((double)sa + (double)sb, (double)qa + (double)qb, (double)ra + (double)rb);
}

// Hooks the caller threads into the iterations:
//   pass0_on / pass0(kk): side work fused into the first pass, per vector slot kk
//   side(e):               DMA hook, run inside exchange e's push (see xch_push)
//   final_xch(sy, best, besti) -> raw cluster sum of Y^(T+1); performs the last
//                          exchange (and whatever the caller overlaps with it)
template <typename P0, typename SD, typename FX>
struct IterHooks {
  bool pass0_on;
  P0 pass0;
  SD side;
  FX final_xch;
};
template <typename P0, typename SD, typename FX>
__device__ __forceinline__ IterHooks<P0, SD, FX> make_hooks(bool on, P0 p0, SD sd, FX fx) {
  return IterHooks<P0, SD, FX>{on, p0, sd, fx};
}

template <bool B>
struct BoolC {
  static constexpr bool value = B;
};
template <int I>
struct IntC {
  static constexpr int value = I;
};

// ---------------------------------------------------------------------------
// CutMax iterations on a register-resident, K0-shifted row slice.
//
// (S_in, Q_in) are the cluster sums of the shifted input.  `len` real elements
// are followed by phantom slots (beyond the slice) that start as copies of
// element 0 (0 in the shifted representation) and get the same updates, so the
// element passes need no per-element control flow.  All phantoms of the row
// carry one common value w_t, tracked as a scalar, and
//   fp64: their total contribution mph*w (mph = phantom slots in the cluster)
//         is subtracted from the cluster sums — no predicate in the passes;
//   fp32: they are left out of the sums by a per-slot predicate (mph = 0): the
//         fp32 partial sums would round the mph identical terms coherently,
//         ~1e-6 relative in the variance and ~1e-5 in Z after p^T growth.
//
// With ARGMAX, the last iteration's pass also tracks the argmax of Y^(T+1)
// (pin A7: equals argmax Z for the positive normaliser) and the last exchange
// carries it.  Phantoms are exact copies of element 0 (shift K0 = x[0]), so
// they can never beat it (equal value, larger index): no predicate needed.
//
// On exit rnorm is the normaliser inv(sum Y) (1 when PAM_F_NO_NORMALIZE).
// v holds Y^(T+1) unless final_xch reused the registers.  Returns the row
// status, identical in every CTA.
//
// STOP (early stopping): after every non-final pass the exchange
// also carries the row maximum; when max Y / sum Y >= 1 - eps_stop (the
// oracle's test, oracle.c orc_cutmax) the remaining iterations are replaced by
// one terminal pass Y = v + K (undo the storage shift) that feeds the usual
// final exchange, normaliser and argmax.  The decision is made by every CTA's
// control warp from identical exchanged sums, so it is cluster-uniform.
template <typename Elem, int NTG, int E, int P, bool ARGMAX, typename Hooks, bool STOP = false>
__device__ __forceinline__ int cutmax_iterate(Elem (&v)[E], const double S_in, const double Q_in, const double K0,
                                              const int len, const double mph, const RowParams& rp,
                                              const double inv_n, const double nd,
                                              ControlBlock* cb, uint32_t& xround, const uint32_t rank,
                                              const uint32_t C, const int gtid, const int64_t gbase,
                                              double* stats_row, double& rnorm, long long& argmax_out, Hooks& h,
                                              long long* tr) {
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
  // slot i holds an element (fp32 only; fp64 corrects by mph * w instead)
  auto real = [&](int i) { return sizeof(Elem) == 8 || ((i / VEC) * NTG + gtid) * VEC + (i % VEC) < len; };

  // exact second pass about dm when the shifted one-pass moments cancelled
  auto guard = [&](double S, double Q, double w, double& dm, double& s2) {
    moments_from_sums(S, Q, inv_n, dm, s2);
    if (st == PAM_OK && isfinite(Q) && Q * inv_n > kGuard * s2) {
      const Elem dme = (Elem)dm;
      Elem q2a = 0, q2b = 0;
#pragma unroll
      for (int i = 0; i < E; i += 2) {
        const Elem d0 = v[i] - dme, d1 = v[i + 1] - dme;
        if (real(i)) q2a = fma_e(d0, d0, q2a);
        if (real(i + 1)) q2b = fma_e(d1, d1, q2b);
      }
      const double2 r2 = cluster_sum2<NTG>((double)q2a + (double)q2b, 0.0, cb, xround, rank, C, gtid);
      const Elem dw = (Elem)w - dme;
      s2 = (r2.x - mph * (double)dw * (double)dw) * inv_n;
    }
  };

  // per-iteration constants, loaded ahead of the exchange they follow
  double c_inv = rp.inv_c[0], knext = rp.kshift[1];
  int pcur = rp.p[0];

  double dm, s2;
  if (!isfinite(S_in) || !isfinite(Q_in)) st = PAM_ERR_NON_FINITE;
  guard(S_in, Q_in, 0.0, dm, s2);
  PAM_TRACE(tr, 4);
  double kcur = K0;
  Elem w = 0;  // phantom value (shifted representation)

  // one element pass; FIRST: fused pass-0 side work, LAST: argmax, no moments;
  // TERM (early stop): y = v + ke, the stored shift undone, instead of an update
  auto pass = [&](auto first_c, auto last_c, auto term_c, Elem ke, Elem be, Elem kn, int p, Elem& sa, Elem& sb,
                  Elem& qa, Elem& qb, Elem& bestv, int& besto) {
    constexpr bool FIRST = decltype(first_c)::value, LAST = decltype(last_c)::value;
    constexpr bool TERM = decltype(term_c)::value;
    constexpr bool TRACK = (LAST && ARGMAX) || (STOP && !LAST);  // STOP: the row max of every iterate
#pragma unroll
    for (int i = 0; i < E; i += 2) {
      if (FIRST && (i % VEC) == 0) h.pass0(i / VEC);
      const Elem d0 = TERM ? v[i] + ke : cutmax_update<Elem, P>(v[i], ke, be, kn, p);
      const Elem d1 = TERM ? v[i + 1] + ke : cutmax_update<Elem, P>(v[i + 1], ke, be, kn, p);
      v[i] = d0;
      v[i + 1] = d1;
      if (real(i)) {
        sa += d0;
        if (!LAST) qa = fma_e(d0, d0, qa);
      }
      if (real(i + 1)) {
        sb += d1;
        if (!LAST) qb = fma_e(d1, d1, qb);
      }
      if (TRACK) {  // slots in increasing element order: strict > keeps the lowest index
        if (d0 > bestv) { bestv = d0; besto = i; }
        if (d1 > bestv) { bestv = d1; besto = i + 1; }
      }
    }
    if (FIRST) ptx::fence_proxy_async_smem();  // side writes -> visible to the TMA engine after the barrier
  };
  auto slot_index = [&](int besto) {
    return gbase + (long long)(((besto / VEC) * NTG + gtid) * VEC + (besto % VEC));
  };

  // scalar chain of iteration t from (kcur, dm, s2): status, 1/sigma, k, b
  auto chain = [&](int t, double& kd, double& bd) {
    const double mu = kcur + dm;
    // Center the input iteration on the fp64 mean, as the reference computes it
    // (SPEC.md:127): mu is rounded to the double grid of the logits, and
    // mu - kcur is exact (Sterbenz).  For rows whose |mean| / sigma is huge
    // (e.g. 1e9 + N(0, 1e-2)) that rounding, not the summation, sets the result.
    if (t == 0) dm = mu - kcur;
    // status: first failure wins (branch-free on the common path)
    const bool bad_range = !isfinite(mu) || !isfinite(s2);
    st = (st != PAM_OK) ? st : (bad_range ? PAM_ERR_RANGE : (s2 < eps_var ? PAM_ERR_DEGENERATE_INPUT : PAM_OK));
    if (stats_row) {
      stats_row[t * 2 + 0] = mu;
      stats_row[t * 2 + 1] = s2;
    }
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
    kd = (st == PAM_OK) ? inv_sigma * c_inv : 0.0;
    bd = fma(-dm, kd, 1.0);
  };
  // control warp: warp 0 alone waits for each exchange, runs the moments, the
  // guard decision and the chain, and broadcasts (k, b, dm, status) through
  // shared memory (named barrier 1); see the p = 3 flow of cutmax_rows_kernel
  const int warp = gtid >> 5;
  auto bar1 = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(NTG) : "memory"); };
  auto publish = [&](double kd, double bd, int flag) {
    if ((gtid & 31) == 0) {
      cb->bc.ke = kd;
      cb->bc.be = bd;
      cb->bc.dm = dm;
      cb->bc.flag = flag;
      cb->bc.st = st;
    }
  };

  // ---- T iterations; the last one (no variance; argmax) is peeled -----------
  double total = 0.0;
  double kd, bd;
  bool stopped = false;  // STOP: eps_stop reached, the next pass is the terminal one
  chain(0, kd, bd);  // every warp: identical inputs
  for (int t = 0; t < T; ++t) {
    const Elem ke = (Elem)kd, be = affine_coef<Elem>(bd, dm), kn = (Elem)(-knext);
    const int p = pcur;
    if (!stopped) w = cutmax_update<Elem, P>(w, ke, be, kn, p);
    const double kthis = knext;
    const bool first = (t == 0) && h.pass0_on;
    Elem sa = 0, sb = 0, qa = 0, qb = 0, bestv = -INFINITY;
    int besto = 0;  // register slot of the best element (compile-time immediates)
    if (t + 1 < T && !stopped) {
      if (first)
        pass(BoolC<true>(), BoolC<false>(), BoolC<false>(), ke, be, kn, p, sa, sb, qa, qb, bestv, besto);
      else
        pass(BoolC<false>(), BoolC<false>(), BoolC<false>(), ke, be, kn, p, sa, sb, qa, qb, bestv, besto);
      c_inv = rp.inv_c[t + 1];  // prefetch next iteration's constants
      knext = rp.kshift[t + 2];
      pcur = rp.p[t + 1];
      PAM_TRACE(tr, 5 + 2 * t);
      constexpr int XM = STOP ? kArgmax : kSum2;
      xch_push<NTG, XM>((double)sa + (double)sb, (double)qa + (double)qb, (double)bestv, slot_index(besto), cb,
                        xround, rank, C, gtid, [&]() { h.side(t); });
      kcur = kthis;
      const double wd = (double)w;
      if (warp == 0) {
        double bv = 0.0;
        long long bi = 0;
        const double2 r = xch_wait<XM>(bv, bi, cb, xround, C, gtid);
        const double Q = r.y - mph * wd * wd;
        moments_from_sums(r.x - mph * wd, Q, inv_n, dm, s2);
        // stop when the top mass max Y / sum Y reaches 1 - eps_stop
        const bool stop_here = STOP && st == PAM_OK && (bv + kcur) / fma(nd, kcur, r.x - mph * wd) >= 1.0 - rp.eps_stop;
        if (stop_here) {
          publish(0.0, 0.0, 2);
        } else if (st == PAM_OK && isfinite(Q) && Q * inv_n > kGuard * s2) {
          publish(0.0, 0.0, 1);  // exact second pass first
        } else {
          chain(t + 1, kd, bd);
          publish(kd, bd, 0);
        }
      } else {
        ++xround;  // keep the round counter in step with warp 0
      }
      bar1();
      Bcast b = cb->bc;
      if (STOP && b.flag == 2) {  // cluster-uniform: the next iteration is the terminal pass
        stopped = true;
        st = b.st;
        PAM_TRACE(tr, 6 + 2 * t);
        continue;
      }
      if (b.flag) {  // exact second pass about dm (cluster-uniform, rare)
        dm = b.dm;
        const Elem dme = (Elem)dm;
        Elem q2a = 0, q2b = 0;
#pragma unroll
        for (int i = 0; i < E; i += 2) {
          const Elem d0 = v[i] - dme, d1 = v[i + 1] - dme;
          if (real(i)) q2a = fma_e(d0, d0, q2a);
          if (real(i + 1)) q2b = fma_e(d1, d1, q2b);
        }
        const double2 r2 = cluster_sum2<NTG>((double)q2a + (double)q2b, 0.0, cb, xround, rank, C, gtid);
        if (warp == 0) {
          const Elem dw = (Elem)w - dme;
          s2 = (r2.x - mph * (double)dw * (double)dw) * inv_n;
          chain(t + 1, kd, bd);
          publish(kd, bd, 0);
        }
        bar1();
        b = cb->bc;
      }
      kd = b.ke;
      bd = b.be;
      dm = b.dm;
      st = b.st;
      PAM_TRACE(tr, 6 + 2 * t);
    } else {
      if (STOP && stopped) {
        const Elem kk = (Elem)kcur;  // Y = v + K: the shift of the stored iterate undone
        w = w + kk;
        pass(BoolC<false>(), BoolC<true>(), BoolC<true>(), kk, be, kn, p, sa, sb, qa, qb, bestv, besto);
      } else if (first) {
        pass(BoolC<true>(), BoolC<true>(), BoolC<false>(), ke, be, kn, p, sa, sb, qa, qb, bestv, besto);
      } else {
        pass(BoolC<false>(), BoolC<true>(), BoolC<false>(), ke, be, kn, p, sa, sb, qa, qb, bestv, besto);
      }
      double best = (double)bestv;
      long long besti = slot_index(besto);
      PAM_TRACE(tr, 5 + 2 * t);
      const double ty = h.final_xch((double)sa + (double)sb, best, besti);
      PAM_TRACE(tr, 6 + 2 * t);
      total = ty - mph * (double)w;  // kshift[T] == 0 (or the terminal pass): v holds Y itself
      argmax_out = besti;
      break;
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

// Resident CTAs per SM the register budget allows without spilling the slice
// (launch-bounds hint; MINB > 0 in the variant table overrides it).
template <typename Elem, int NT, int E>
constexpr int min_blocks_for() {
  constexpr int est = E * (int)sizeof(Elem) / 4 + 60;  // slice registers + ~60 of state
  constexpr int regs = est < 96 ? 96 : est;
  constexpr int b = 65536 / (NT * regs);
  return b < 1 ? 1 : (b > 8 ? 8 : b);
}

// ---------------------------------------------------------------------------
template <typename Elem, int NTG, int E, int P, int MINB = 0, bool STOP = false>
__global__ void __launch_bounds__(NTG, (MINB > 0 ? MINB : min_blocks_for<Elem, NTG, E>()))
    cutmax_rows_kernel(const CutmaxArgs a) {
  static_assert(!STOP || P == 0, "early stopping runs on the generic flow");
  using Tr = ElemTraits<Elem>;
  using V = typename Tr::V;
  constexpr int VEC = Tr::VEC;
  constexpr int NV = E / VEC;
  constexpr int NW = NTG / 32;
  static_assert(E % VEC == 0 && E % 2 == 0, "E must be a multiple of the vector width");
  static_assert(NTG % 32 == 0 && NW >= 2 && NW <= 16 && (NW & (NW - 1)) == 0, "bad CTA size");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int gtid = (int)threadIdx.x;
  Elem* buf = reinterpret_cast<Elem*>(smem_raw);  // row buffer: NTG*E elements (TMA path)
  ControlBlock* cb = reinterpret_cast<ControlBlock*>(smem_raw + a.ctrl_offset);

  const uint32_t rank = ptx::cluster_ctarank();
  const uint32_t C = ptx::cluster_nctarank();
  const int64_t cid = ptx::cluster_id_x();
  const int64_t ncl = ptx::nclusters_x();
  const int64_t n = a.n;
  const int64_t base = (int64_t)rank * a.L;
  const int64_t rem = n - base;
  const int len = rem <= 0 ? 0 : (rem < a.L ? (int)rem : a.L);
  const bool TMA = a.tma != 0;
  const bool dma = gtid == NTG - 32;  // lane 0 of the last warp issues every bulk copy
  // phantom handling (see cutmax_iterate): fp64 subtracts mph * w from the
  // cluster sums, fp32 predicates the accumulation on real(i)
  const double mph = sizeof(Elem) == 8 ? (double)((int64_t)C * NTG * E - n) : 0.0;
  auto real = [&](int i) { return sizeof(Elem) == 8 || ((i / VEC) * NTG + gtid) * VEC + (i % VEC) < len; };
  const RowParams& rp = a.rp;
  const int T = rp.T;
  const Elem* __restrict__ X = reinterpret_cast<const Elem*>(a.x);
  Elem* __restrict__ Z = reinterpret_cast<Elem*>(a.z);

  const uint32_t bar_load = ptx::smem_addr(&cb->mb_load);
  const uint32_t slice_bytes = (uint32_t)len * (uint32_t)sizeof(Elem);
  // bulk copies move the slice in 4 chunks so a row's load can chase the
  // previous row's store through the buffer chunk by chunk
  const uint32_t chunk = ((slice_bytes + 63u) / 64u) * 16u;
  const int nch = chunk ? (int)((slice_bytes + chunk - 1) / chunk) : 0;
  uint64_t policy = 0;
  if (TMA) policy = ptx::policy_evict_first();

  if (gtid == 0) {
    cb->unc_n = 0;
    cb->fin_pending = 0;
    ptx::mbar_init(bar_load, 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_x[0]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_x[1]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_in), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_t[0]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb->mb_t[1]), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (gtid == 0) {
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[0]), C * kXchBytes);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_x[1]), C * kXchBytes);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_in), C * 16u);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_t[0]), C * 16u);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb->mb_t[1]), C * 16u);
  }
  ptx::cluster_sync();

#ifdef PAM_CHECKED_BUILD
  PAM_CHECK(len <= NTG * E && a.L <= NTG * E);
  if (TMA) {
    PAM_CHECK(len % VEC == 0 && (uintptr_t)a.x % 16 == 0 && (uintptr_t)a.z % 16 == 0 && a.ldx % VEC == 0);
    for (int i = gtid; i < NTG * E; i += NTG) buf[i] = Elem(NAN);  // poison (see cutmax_p3_kernel.cuh)
    ptx::fence_proxy_async_smem();
  }
  __syncthreads();
#endif
  // ---- DMA-thread helpers ----------------------------------------------------
  auto load_chunk = [&](int64_t row, int i) {
    const unsigned char* src = reinterpret_cast<const unsigned char*>(X + row * a.ldx + base);
    const uint32_t off = (uint32_t)i * chunk;
    const uint32_t nb = (slice_bytes - off) < chunk ? (slice_bytes - off) : chunk;
    PAM_CHECK(row >= 0 && row < a.B && ((uintptr_t)(src + off) & 15) == 0 && nb % 16 == 0);
    ptx::bulk_g2s(ptx::smem_addr(buf) + off, src + off, nb, bar_load, policy);
  };
  auto store_all = [&](int64_t row) {  // buf -> Z(row), one bulk group per chunk
    unsigned char* dst = reinterpret_cast<unsigned char*>(Z + row * a.ldz + base);
    for (int i = 0; i < nch; ++i) {
      const uint32_t off = (uint32_t)i * chunk;
      const uint32_t nb = (slice_bytes - off) < chunk ? (slice_bytes - off) : chunk;
      ptx::bulk_s2g(dst + off, ptx::smem_addr(buf) + off, nb, policy);
      ptx::bulk_commit();
    }
  };
  auto load_after_store = [&](int64_t row) {  // X(row) -> buf as the outstanding store frees each chunk
    ptx::mbar_arrive_expect_tx(bar_load, slice_bytes);
    for (int i = 0; i < nch; ++i) {
      ptx::bulk_wait_read_le(nch - 1 - i);
      load_chunk(row, i);
    }
  };

  int64_t row = cid;
  uint32_t xround = 0, load_par = 0, in_par = 0;
  uint32_t t2_ph = 0u;           // mb_t phases, bit s = slot s (warp 0)
  int64_t lrow = 0;              // local row counter: the parity selects the top-2 record slot
  Elem v[E];
  // top-2 screen values (hiword_f) of the real input elements of this thread's
  // slots (TieWarning); phantom slots are copies of x[0] and must not count
  float t1 = -INFINITY, t2 = -INFINITY;
  auto load_direct = [&](const Elem* src, Elem k0e) {  // unaligned rows: direct loads, no staging
#pragma unroll
    for (int kk = 0; kk < NV; ++kk) {
      const int li0 = (kk * NTG + gtid) * VEC;
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        const bool in = li0 + j < len;
        const Elem xv = in ? __ldcs(src + li0 + j) : k0e;
        v[kk * VEC + j] = xv;
        if (in) top2f_add(t1, t2, hiword_f(xv));
      }
    }
  };

  // warp 0, once per row: the row's input top-2 keys -> TieWarning decision;
  // rank 0 writes argmax and status, undecided rows are queued (every CTA
  // queues identically: the keys are cluster-uniform)
  auto finish_row = [&](int64_t r, int st, long long amax, uint32_t slot) {
    const int2 kk = top2k_wait(cb, slot, t2_ph, C, gtid);
    const int td = tie_decide<Elem>(st, kk.x, kk.y);
    if (rank == 0 && gtid == 0) {
      if (a.argmax) a.argmax[r] = (st == PAM_OK) ? (int32_t)amax : -1;
      if (a.status) a.status[r] = st | (td == 1 ? PAM_ROW_FLAG_TIE : 0);
    }
    if (td == 2 && gtid == 0) {
      const int q = cb->unc_n;
      if (q < 16) cb->unc_rows[q] = r;
      cb->unc_n = q + 1;
    }
  };

  // ---- prologue: the cluster's first row -> registers -------------------------
  if (TMA && row < a.B) {
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
      if (li0 + VEC <= len) {
        *reinterpret_cast<V*>(&v[k * VEC]) = *reinterpret_cast<const V*>(buf + li0);
#pragma unroll
        for (int j = 0; j < VEC; ++j) top2f_add(t1, t2, hiword_f(v[k * VEC + j]));
      } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          const bool in = li0 + j < len;
          v[k * VEC + j] = in ? buf[li0 + j] : k0;  // phantoms = K0
          if (in) top2f_add(t1, t2, hiword_f(v[k * VEC + j]));
        }
      }
    }
    __syncthreads();  // buf free
  }

  if constexpr (P == 3) {
    // ===== p = 3 every iteration: analytic normaliser =======================
    // sum_i (1 + k d_i)^3 = n + 3k sum d + 3k^2 sum d^2 + k^3 sum d^3 with
    // d = y - mu of the iterate feeding the last iteration, so inv(sum Y) is
    // known BEFORE the last pass.  The last pass then writes Z = Y*inv directly
    // into the row buffer while pulling X(next) - K0(next) into registers and
    // summing its moments; ONE exchange closes the row (argmax + next row's
    // input sums) and the Z store streams out right behind it.  The third
    // power sum rides on the exchange of pass T-2 (or the input for T = 1).
    // A non-finite analytic total (third powers overflowing) falls back to an
    // explicit sum of Y (extra pass + exchange).
    //
    // Control warp.  Between two passes only warp 0 waits for the exchange,
    // combines the C records and runs the scalar chain (moments, status,
    // 1/sigma, normaliser); it publishes the pass coefficients in shared memory
    // and the other warps pick them up at a named barrier.  Replicating that
    // latency-bound scalar work in all 16 warps cost ~25% of each gap.
    constexpr double kGuard = sizeof(Elem) == 8 ? 16.0 : 2.0;
    const int warp = gtid >> 5;
    const double nd = (double)n;
    const double inv_n = a.inv_n;
    const bool normalize = !(rp.flags & PAM_F_NO_NORMALIZE);
    const bool poly_invsqrt = rp.invsqrt_mode == PAM_MODE_POLY;
    const double eps_var = rp.eps_var;
    bool in_ready = false;  // registers hold the K0-shifted row; warp 0 holds its cluster sums
    double S_c = 0.0, Q_c = 0.0, R_c = 0.0;  // warp 0: cluster sums of the current iterate
    Elem k0_cur = row < a.B ? __ldg(X + row * a.ldx) : Elem(0);
    auto bar1 = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(NTG) : "memory"); };
    for (; row < a.B; row += ncl, ++lrow) {
      const int64_t next = row + ncl;
      const bool has_next = next < a.B;
      const bool merged = TMA && has_next;  // the closing exchange carries the next row's input sums
#ifdef PAM_TRACE_BUILD
      long long* tr = (a.trace && lrow < kTraceRows)
                          ? a.trace + ((int64_t)blockIdx.x * kTraceRows + lrow) * kTraceEvents
                          : nullptr;
#else
      long long* tr = nullptr;
#endif
      PAM_TRACE(tr, 0);
      const Elem* xrow = X + row * a.ldx;
      const Elem k0e = k0_cur;  // shift for the input (same in every CTA)
      const double K0 = (double)k0e;
      // x[next][0]: loaded a row ahead, first used by the last pass
      const Elem k0next = has_next ? __ldg(X + next * a.ldx) : Elem(0);
      if (!in_ready) {
        if (!TMA) {
          t1 = t2 = -INFINITY;
          load_direct(xrow + base, k0e);
        }
        const double3 part = input_pass3<Elem, E>(v, K0);
        const double3 r = cluster_sum3<NTG>(part.x, part.y, part.z, cb, xround, rank, C, gtid,
                                            KeyPush{true, fkey(t1), fkey(t2), (uint32_t)(lrow & 1)});
        S_c = r.x;
        Q_c = r.y;
        R_c = r.z;
      }
      PAM_TRACE(tr, 2);

      // DMA thread: X(next) -> buffer, chunk by chunk behind the previous row's Z store
      int issued = 0;
      bool armed = false;
      auto issue_upto = [&](int upto) {
        if (!merged) return;
        if (!armed) {
          ptx::mbar_arrive_expect_tx(bar_load, slice_bytes);
          armed = true;
        }
        for (; issued < upto; ++issued) {
          ptx::bulk_wait_read_le(nch - 1 - issued);
          load_chunk(next, issued);
        }
      };
      auto side = [&](int e) {
        if (e == 0) issue_upto(nch / 2);
        if (e == 1) issue_upto(nch);
        if (e < 2) PAM_TRACE_DMA(tr, 25 + e);
      };

      // ---- warp 0's scalar state ---------------------------------------------------
      int st = PAM_OK;
      double dm = 0.0, s2 = 0.0, m3 = 0.0, e1 = 0.0;
      double kcur = K0, c_inv = rp.inv_c[0], knext = rp.kshift[1];
      Elem w = 0;  // phantom value (shifted representation)
      double* stats_row = (rank == 0 && gtid == 0 && a.stats) ? a.stats + row * T * 2 : nullptr;
      if (!isfinite(S_c) || !isfinite(Q_c)) st = PAM_ERR_NON_FINITE;

      // moments of iterate t from its (phantom-corrected) cluster sums; returns
      // false when the one-pass form cancelled and the exact pass is needed
      auto moments = [&](double S, double Q, double R, bool need3) -> bool {
        dm = S * inv_n;
        const double qn = Q * inv_n;
        s2 = fma(-dm, dm, qn);
        if (need3) {
          e1 = fma(-nd, dm, S);
          m3 = fma(dm, fma(2.0 * dm, dm, -3.0 * qn), R * inv_n);
        }
        return !(st == PAM_OK && isfinite(Q) && qn > kGuard * s2);
      };
      // scalar chain of iteration t (+ the analytic normaliser for the last one)
      auto chain = [&](int t, double& kd, double& bd, double& rnorm) {
        const double mu = kcur + dm;
        // input iteration: center on the reference's fp64-rounded mean (see the
        // generic chain); T = 1 keeps dm, because its analytic normaliser uses
        // the moments about dm
        if (t == 0 && T > 1) dm = mu - kcur;
        const bool bad_range = !isfinite(mu) || !isfinite(s2);
        st = (st != PAM_OK) ? st : (bad_range ? PAM_ERR_RANGE : (s2 < eps_var ? PAM_ERR_DEGENERATE_INPUT : PAM_OK));
        if (stats_row) {
          stats_row[t * 2 + 0] = mu;
          stats_row[t * 2 + 1] = s2;
        }
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
        kd = (st == PAM_OK) ? inv_sigma * c_inv : 0.0;
        bd = fma(-dm, kd, 1.0);
        rnorm = 1.0;
        if (t == T - 1) {
          const double total = nd + kd * (3.0 * e1 + kd * (3.0 * nd * s2 + kd * nd * m3));
          if (st == PAM_OK && !isfinite(total)) {
            rnorm = NAN;  // explicit sum needed (rare): signalled to the CTA
            return;
          }
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
        }
      };
      // final normaliser from an explicit total (rare fallback)
      auto finish_total = [&](double total, double& rnorm) {
        rnorm = 1.0;
        if (st == PAM_OK && !isfinite(total)) st = PAM_ERR_RANGE;
        if (st == PAM_OK && normalize) {
          if (!(total > 0.0)) {
            st = PAM_ERR_RANGE;
          } else if (rp.inv_mode == PAM_MODE_POLY) {
            const pam_approx_config& ac = rp.inv;
            const int rs = inv_rescaled(total, ac.iterations, ac.rescale, ac.scale_log2, ac.lo, ac.hi, &rnorm);
            if (rs) st = rs;
          } else {
            rnorm = 1.0 / total;
          }
        }
      };
      // control step for pass t (warp 0 computes, everyone receives): returns the
      // affine coefficients (ke, be) and, for the last pass, the normaliser re.
      auto control = [&](int t, Elem& ke, Elem& be, Elem& re) {
        const bool need3 = (t == T - 1);
        if (warp == 0) {
          const bool ok = moments(S_c, Q_c, R_c, need3);
          Bcast& bc = cb->bc;
          if (ok) {
            double kd, bd, rn;
            chain(t, kd, bd, rn);
            if (lane_of(gtid) == 0) {
              bc.ke = kd;
              bc.be = bd;
              bc.dm = dm;
              bc.re = rn;
              bc.flag = 0;
            }
          } else if (lane_of(gtid) == 0) {
            bc.dm = dm;
            bc.flag = 1;
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
            const double dw = (double)((Elem)w - dme);
            s2 = (r2.x - mph * dw * dw) * inv_n;
            if (need3) m3 = (r2.y - mph * dw * dw * dw) * inv_n;
            double kd, bd, rn;
            chain(t, kd, bd, rn);
            if (lane_of(gtid) == 0) {
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

      // pass t < T-1: update + shifted moments (+ third power sum on pass T-2)
      auto pass = [&](auto r_c, Elem ke, Elem be, Elem kn, double3& out) {
        constexpr bool R3 = decltype(r_c)::value;
        Elem sa = 0, sb = 0, qa = 0, qb = 0, ra = 0, rb = 0;
#pragma unroll
        for (int i = 0; i < E; i += 2) {
          const Elem d0 = cutmax_update<Elem, 3>(v[i], ke, be, kn, 3);
          const Elem d1 = cutmax_update<Elem, 3>(v[i + 1], ke, be, kn, 3);
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
        out = make_double3((double)sa + (double)sb, (double)qa + (double)qb, (double)ra + (double)rb);
      };

      for (int t = 0; t + 1 < T; ++t) {
        Elem ke, be, re_unused;
        control(t, ke, be, re_unused);
        const Elem kn = (Elem)(-knext);
        PAM_TRACE(tr, 13 + t);
        const bool need3 = (t + 2 == T);
        double3 part;
        if (need3)
          pass(BoolC<true>(), ke, be, kn, part);
        else
          pass(BoolC<false>(), ke, be, kn, part);
        PAM_TRACE(tr, 5 + 2 * t);
#ifdef PAM_TRACE_BUILD
        if (tr != nullptr && t == 1) {  // pass-end stamps of warps 0, 5, 10, 15 (intra-CTA skew)
          if (gtid == 5 * 32) tr[30] = clock64();
          if (gtid == 10 * 32) tr[31] = clock64();
          if (gtid == NTG - 32) tr[19] = clock64();
        }
#endif
        if (need3)
          xch_push<NTG, kSum3>(part.x, part.y, part.z, 0LL, cb, xround, rank, C, gtid, [&]() { side(t); });
        else
          xch_push<NTG, kSum2>(part.x, part.y, 0.0, 0LL, cb, xround, rank, C, gtid, [&]() { side(t); });
        PAM_TRACE(tr, 16 + t);
        if (warp == 0) {
          if (t == 0 && cb->fin_pending) {  // previous row's argmax / status, in the exchange's idle window
            finish_row(cb->fin_row, cb->fin_st, cb->fin_best, (uint32_t)((lrow - 1) & 1));
            __syncwarp();
            if (gtid == 0) cb->fin_pending = 0;
          }
          double r3 = 0.0;
          long long ci = 0;
          const double2 r = need3 ? xch_wait<kSum3>(r3, ci, cb, xround, C, gtid)
                                  : xch_wait<kSum2>(r3, ci, cb, xround, C, gtid);
          w = cutmax_update<Elem, 3>(w, ke, be, kn, 3);
          const double wd = (double)w;
          S_c = r.x - mph * wd;
          Q_c = r.y - mph * wd * wd;
          R_c = r3 - mph * wd * wd * wd;
          kcur = knext;
          c_inv = rp.inv_c[t + 1];
          knext = rp.kshift[t + 2];
        } else {
          ++xround;  // keep the round counter in step with warp 0
        }
        PAM_TRACE(tr, 6 + 2 * t);
      }

      // ---- last iteration: normaliser first, then the fused pass ---------------
      Elem ke, be, re;
      control(T - 1, ke, be, re);
      const Elem kz = (Elem)0;  // kshift[T] = 0
      if (!(re == re)) {  // analytic total not finite: explicit sum of Y (rare, cluster-uniform)
        Elem ta = 0, tb = 0;
#pragma unroll
        for (int i = 0; i < E; i += 2) {
          const Elem y0 = cutmax_update<Elem, 3>(v[i], ke, be, kz, 3);
          const Elem y1 = cutmax_update<Elem, 3>(v[i + 1], ke, be, kz, 3);
          if (real(i)) ta += y0;
          if (real(i + 1)) tb += y1;
        }
        const double tot = cluster_sum2<NTG>((double)ta + (double)tb, 0.0, cb, xround, rank, C, gtid).x -
                           mph * (double)cutmax_update<Elem, 3>(w, ke, be, kz, 3);
        if (warp == 0) {
          double rn;
          finish_total(tot, rn);
          if (lane_of(gtid) == 0) cb->bc.re = rn;
        }
        bar1();
        re = (Elem)cb->bc.re;
      }
      PAM_TRACE(tr, 22);
      if (merged) {
        if (dma) issue_upto(nch);  // small T: whatever the hooks did not issue yet
        ptx::mbar_wait_cta(bar_load, load_par);  // X(next) has landed
        load_par ^= 1u;
      } else if (TMA) {
        if (dma) ptx::bulk_wait_read_all();  // the previous Z store has read the buffer
        __syncthreads();
      }
      PAM_TRACE(tr, 23);

      // fused last pass: Y = z^3 (argmax), Z = Y * inv(sum Y) -> buffer / HBM,
      // and (merged) X(next) - K0(next) -> registers with its moments
      Elem bestv = -INFINITY;
      int besto = 0;  // register slot of the best element (compile-time immediates)
      double3 nxt = make_double3(0.0, 0.0, 0.0);
      Elem* zrow = Z + row * a.ldz + base;
      t1 = t2 = -INFINITY;  // top-2 of X(next) (merged)
      auto last = [&](auto mode_c, auto r_c) {
        constexpr int MODE = decltype(mode_c)::value;  // 0: swap (merged), 1: Z -> buffer, 2: Z -> HBM
        constexpr bool R3 = decltype(r_c)::value;
        Elem sa = 0, sb = 0, qa = 0, qb = 0, ra = 0, rb = 0;
#pragma unroll
        for (int kk = 0; kk < NV; ++kk) {
          const int li0 = (kk * NTG + gtid) * VEC;
          Elem o[VEC];
#pragma unroll
          for (int j = 0; j < VEC; ++j) {
            const Elem y = cutmax_update<Elem, 3>(v[kk * VEC + j], ke, be, kz, 3);
            if (y > bestv) {  // slots in increasing element order: strict > keeps the lowest index
              bestv = y;
              besto = kk * VEC + j;
            }
            o[j] = y * re;
          }
          if (MODE == 2) {
#pragma unroll
            for (int j = 0; j < VEC; ++j)
              if (li0 + j < len) __stcs(zrow + li0 + j, o[j]);
            continue;
          }
          if (li0 + VEC <= len) {
            V xn;
            if (MODE == 0) xn = *reinterpret_cast<const V*>(buf + li0);
            *reinterpret_cast<V*>(buf + li0) = *reinterpret_cast<const V*>(o);
            if (MODE == 0) {
              const Elem* xe = reinterpret_cast<const Elem*>(&xn);
#pragma unroll
              for (int j = 0; j < VEC; ++j) {
                v[kk * VEC + j] = xe[j] - k0next;
                top2f_add(t1, t2, hiword_f(xe[j]));
              }
            }
          } else {
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
              const bool in = li0 + j < len;
              Elem xv = k0next;  // phantoms: K0(next) -> 0
              if (MODE == 0 && in) {
                xv = buf[li0 + j];
                top2f_add(t1, t2, hiword_f(xv));
              }
              if (in) buf[li0 + j] = o[j];
              if (MODE == 0) v[kk * VEC + j] = xv - k0next;
            }
          }
          if (MODE == 0) {
#pragma unroll
            for (int j = 0; j < VEC; j += 2) {
              const Elem d0 = v[kk * VEC + j], d1 = v[kk * VEC + j + 1];
              sa += d0;
              sb += d1;
              if (R3) {
                const Elem f0 = d0 * d0, f1 = d1 * d1;
                qa += f0;
                qb += f1;
                ra = fma_e(f0, d0, ra);
                rb = fma_e(f1, d1, rb);
              } else {
                qa = fma_e(d0, d0, qa);
                qb = fma_e(d1, d1, qb);
              }
            }
          }
        }
        nxt = make_double3((double)sa + (double)sb, (double)qa + (double)qb, (double)ra + (double)rb);
      };
      if (merged) {
        if (T == 1)
          last(IntC<0>(), BoolC<true>());
        else
          last(IntC<0>(), BoolC<false>());
      } else if (TMA) {
        last(IntC<1>(), BoolC<false>());
      } else {
        last(IntC<2>(), BoolC<false>());
      }
      if (TMA) ptx::fence_proxy_async_smem();  // Z writes -> visible to the TMA engine after the barrier
      PAM_TRACE(tr, 24);
      double best = (double)bestv;
      long long besti = base + (long long)(((besto / VEC) * NTG + gtid) * VEC + (besto % VEC));
      const int64_t zr = row;
      xch_push<NTG, kArgmax>(
          nxt.x, nxt.y, best, besti, cb, xround, rank, C, gtid,
          [&]() { if (TMA) store_all(zr); }, true,
          KeyPush{merged, fkey(t1), fkey(t2), (uint32_t)((lrow + 1) & 1)});
      if (merged && T == 1) {
        // T = 1 needs the next input's third power sum too (one more exchange)
        if (warp == 0) {
          const double2 rn = xch_wait<kArgmax>(best, besti, cb, xround, C, gtid);
          S_c = rn.x;
          Q_c = rn.y;
        } else {
          ++xround;
        }
        const double r3 = cluster_sum2<NTG>(nxt.z, 0.0, cb, xround, rank, C, gtid).x;
        if (warp == 0) R_c = r3;
      } else if (warp == 0) {
        const double2 rn = xch_wait<kArgmax>(best, besti, cb, xround, C, gtid);
        S_c = rn.x;
        Q_c = rn.y;
      } else {
        ++xround;
      }
      PAM_TRACE(tr, 6 + 2 * (T - 1));
      in_ready = merged;
      k0_cur = k0next;
      if (warp == 0) {
        // argmax / status / TieWarning of this row: deferred to the next row's
        // first exchange wait (the input top-2 records arrived long ago, but the
        // wait and the decision would sit on the control warp's critical path)
        if (T == 1 || !merged) {
          finish_row(row, st, besti, (uint32_t)(lrow & 1));
        } else if (gtid == 0) {
          cb->fin_row = row;
          cb->fin_st = st;
          cb->fin_best = besti;
          cb->fin_pending = 1;
        }
      }
      PAM_TRACE(tr, 21);
    }
  } else {
    // ===== generic p: one-pass-late normalisation (see header) ==============
    bool in_ready = false;  // registers hold the K0-shifted row and (S_in, Q_in) its cluster sums
    double S_in = 0.0, Q_in = 0.0;
    Elem k0_cur = row < a.B ? __ldg(X + row * a.ldx) : Elem(0);
    bool zpend = false;  // buf holds the previous row's unnormalised Y: scale in pass 0, then store
    Elem rn_prev = 1;
    int64_t zrow_prev = 0;
    const int pf_ex = T >= 3 ? 1 : 0;  // exchange whose DMA hook issues the next row's load
    const int warp = gtid >> 5;
    for (; row < a.B; row += ncl, ++lrow) {
      const int64_t next = row + ncl;
      const bool has_next = next < a.B;
      const bool merged = TMA && has_next;  // row-boundary exchange carries the next row's input sums
  #ifdef PAM_TRACE_BUILD
      long long* tr =
          (a.trace && lrow < kTraceRows) ? a.trace + ((int64_t)blockIdx.x * kTraceRows + lrow) * kTraceEvents : nullptr;
  #else
      long long* tr = nullptr;
  #endif
      PAM_TRACE(tr, 0);
      const Elem* xrow = X + row * a.ldx;
      const Elem k0e = k0_cur;  // shift for the input (same in every CTA)
      const double K0 = (double)k0e;
      // x[next][0]: loaded a row ahead, first used by the last pass
      const Elem k0next = has_next ? __ldg(X + next * a.ldx) : Elem(0);

      if (!in_ready) {
        if (!TMA) {
          t1 = t2 = -INFINITY;
          load_direct(xrow + base, k0e);
        }
        const double2 part = input_pass<Elem, E>(v, K0);
        const double2 r = cluster_sum2<NTG>(part.x, part.y, cb, xround, rank, C, gtid,
                                            KeyPush{true, fkey(t1), fkey(t2), (uint32_t)(lrow & 1)});
        S_in = r.x;
        Q_in = r.y;
      }
      PAM_TRACE(tr, 2);

      const bool scale_now = zpend;
      const Elem rsc = rn_prev;
      const int64_t zrow_p = zrow_prev;
      auto pass0 = [&](int kk) {  // Z(prev) = Y(prev) * inv(sum Y(prev)), in the row buffer
        V* p = reinterpret_cast<V*>(buf) + kk * NTG + gtid;
        V t = *p;
        Elem* te = reinterpret_cast<Elem*>(&t);
  #pragma unroll
        for (int j = 0; j < VEC; ++j) te[j] *= rsc;
        *p = t;
      };
      auto side = [&](int e) {  // DMA thread, inside exchange e
        if (!TMA) return;
        if (e == 0 && scale_now) {
          store_all(zrow_p);
          PAM_TRACE_DMA(tr, 25);
        }
        if (e == pf_ex && has_next) {
          PAM_TRACE_DMA(tr, 26);
          load_after_store(next);
          PAM_TRACE_DMA(tr, 27);
        }
      };
      auto final_xch = [&](double sy, double& best, long long& besti) -> double {
        xch_push<NTG, kArgmax>(sy, 0.0, best, besti, cb, xround, rank, C, gtid, [&]() { side(T - 1); });
        if (merged) {
          PAM_TRACE(tr, 22);
          ptx::mbar_wait_cta(bar_load, load_par);  // X(next) has landed
          load_par ^= 1u;
          PAM_TRACE(tr, 23);
          // swap: Y -> buf, X(next) - K0(next) -> registers (+ its moments and top-2)
          Elem sa = 0, sb = 0, qa = 0, qb = 0;
          t1 = t2 = -INFINITY;
  #pragma unroll
          for (int kk = 0; kk < NV; ++kk) {
            const int li0 = (kk * NTG + gtid) * VEC;
            if (li0 + VEC <= len) {
              const V xn = *reinterpret_cast<const V*>(buf + li0);
              *reinterpret_cast<V*>(buf + li0) = *reinterpret_cast<const V*>(&v[kk * VEC]);
              const Elem* xe = reinterpret_cast<const Elem*>(&xn);
  #pragma unroll
              for (int j = 0; j < VEC; ++j) {
                v[kk * VEC + j] = xe[j] - k0next;
                top2f_add(t1, t2, hiword_f(xe[j]));
              }
            } else {
  #pragma unroll
              for (int j = 0; j < VEC; ++j) {
                const bool in = li0 + j < len;
                const Elem xv = in ? buf[li0 + j] : k0next;  // phantoms: K0(next) -> 0
                if (in) {
                  buf[li0 + j] = v[kk * VEC + j];
                  top2f_add(t1, t2, hiword_f(xv));
                }
                v[kk * VEC + j] = xv - k0next;
              }
            }
  #pragma unroll
            for (int j = 0; j < VEC; j += 2) {
              const Elem d0 = v[kk * VEC + j], d1 = v[kk * VEC + j + 1];
              sa += d0;
              sb += d1;
              qa = fma_e(d0, d0, qa);
              qb = fma_e(d1, d1, qb);
            }
          }
          xin_push<NTG>((double)sa + (double)sb, (double)qa + (double)qb, cb, rank, C, gtid,
                        KeyPush{true, fkey(t1), fkey(t2), (uint32_t)((lrow + 1) & 1)});
          PAM_TRACE(tr, 24);
        }
        double2 r = xch_wait<kArgmax>(best, besti, cb, xround, C, gtid);
        if (merged) {
          const double2 in = xin_wait(cb, in_par, C, gtid);
          S_in = in.x;
          Q_in = in.y;
        }
        return r.x;
      };
      auto hooks = make_hooks(scale_now, pass0, side, final_xch);

      double rnorm = 1.0;
      long long amax = -1;
      const int st = cutmax_iterate<Elem, NTG, E, P, true, decltype(hooks), STOP>(
          v, S_in, Q_in, K0, len, mph, rp, a.inv_n, (double)n, cb, xround, rank, C, gtid, base,
          (rank == 0 && gtid == 0 && a.stats) ? a.stats + row * T * 2 : nullptr, rnorm, amax, hooks, tr);
      PAM_TRACE(tr, 20);
      if (warp == 0) finish_row(row, st, amax, (uint32_t)(lrow & 1));

      const Elem re = (Elem)rnorm;
      if (merged) {
        zpend = true;  // Z(row) = buf * re, written during the next row's pass 0
        rn_prev = re;
        zrow_prev = row;
        in_ready = true;
      } else {
        zpend = false;
        in_ready = false;
        if (TMA) {
          // last row of this cluster: Z from registers through the buffer
          if (dma) ptx::bulk_wait_read_all();  // the previous Z store has read buf
          __syncthreads();
  #pragma unroll
          for (int kk = 0; kk < NV; ++kk) {
            const int li0 = (kk * NTG + gtid) * VEC;
            Elem o[VEC];
  #pragma unroll
            for (int j = 0; j < VEC; ++j) o[j] = v[kk * VEC + j] * re;
            if (li0 + VEC <= len) {
              *reinterpret_cast<V*>(buf + li0) = *reinterpret_cast<V*>(o);
            } else {
  #pragma unroll
              for (int j = 0; j < VEC; ++j)
                if (li0 + j < len) buf[li0 + j] = o[j];
            }
          }
          ptx::fence_proxy_async_smem();  // make the Z writes visible to the TMA engine
          __syncthreads();
          if (dma) store_all(row);
        } else {
          Elem* zrow = Z + row * a.ldz + base;
  #pragma unroll
          for (int kk = 0; kk < NV; ++kk) {
            const int li0 = (kk * NTG + gtid) * VEC;
  #pragma unroll
            for (int j = 0; j < VEC; ++j)
              if (li0 + j < len) __stcs(zrow + li0 + j, v[kk * VEC + j] * re);
          }
        }
      }
      k0_cur = k0next;
      PAM_TRACE(tr, 21);
    }
  }
  // ---- TieWarning rows the key screen left undecided: exact fp64 top-2 -------
  // (rare: the two largest inputs share their high word, e.g. a duplicated
  // maximum).  The queue is identical in every CTA of the cluster.
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
  if (TMA && dma) ptx::bulk_wait_all();  // Z stores complete before the CTA retires
  ptx::cluster_sync();  // no CTA leaves while a peer may still push into its shared memory
}

}  // namespace pam
