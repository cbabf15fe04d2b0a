// nucleus_set.cu — the top-p nucleus itself (cutoff logit, size, mass) by a
// cluster-wide radix select: the cumulative-mass step of SPEC.md:464 ("softmax
// probabilities sorted descending, smallest prefix with cumulative mass >= p,
// ties included"; top-p definition) as a histogram + scan over a
// thread-block cluster, with no sort.  SURVEY.md §8 row a11 (the full cutoff /
// nucleus size form of the membership test fused into nucleus_kernel.cuh).
//
// Definition (restated in oracle.c orc_nucleus_set, which sorts):
//   m   = max x;  w_i = floor(exp_t(x_i - m) * 2^40 + 1/2)  (0 when x_i < m - 64):
//         the softmax masses as 40-bit fixed-point integers, so every sum below
//         is an exact integer and does not depend on the order of summation;
//   W   = sum w_i;  A(v) = sum of w_k over {x_k > v};
//   v is inside the nucleus  <=>  (double)A(v) < p * (double)W   (ties share A);
//   cutoff = the smallest inside value, size = #{x_i >= cutoff, w_i > 0},
//   mass = (A(cutoff) + weight of the entries equal to cutoff) / W.
// inside() is monotone in v, so the cutoff is found by descending first (small
// clusters) 1024 linear buckets of max - x, then the bits of an
// order-preserving 64-bit key of x, 8 bits per level: each CTA histograms
// the weights and counts of its slice's candidates (shared atomics; the two most
// common digits of each warp step are pre-summed with REDUX), the cluster's histograms are summed through
// distributed shared memory, and one warp scans the 256 buckets from the top for
// the lowest non-empty bucket whose entries can still be inside; once at most 32
// entries survive, they are gathered into one warp, which finishes exactly
// (all-pairs mass above each, smallest inside key).  Integer
// arithmetic throughout: every CTA takes the same decision, and the result is
// bit-identical to the oracle's.
//
// One row per cluster (C = 1..16 CTAs of <= 11264 entries, slice keys and weights
// resident in shared memory: 16 bytes per element), rows strided over the persistent
// clusters.  HBM traffic: 8n bytes read per row, 24 bytes written.
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "../../include/pam_c_api.h"
#include "pam_ptx.cuh"
#include "pam_scalar.h"

extern "C" void pam_internal_count_launch(void);   // pam_api.cu: kernel_launch_count()
extern "C" int pam_internal_cuda_fail(int e, const char* what);

namespace pam {
namespace {

typedef unsigned long long u64;
constexpr int kNT = 512;
constexpr int kLcap = 11264;  // elements per CTA: 2 x 88 KB of shared memory
constexpr int kWBits = 40;

struct NucSetArgs {
  const double* x;
  int64_t ldx, B, n;
  int32_t L;
  double p;
  double* cutoff;
  int32_t* size;
  double* mass;
  int32_t* status;
  long long* dbg;  // dev: phase clocks of cluster 0 / CTA 0's first row (pam_dev_nucleus_set_clocks)
};

#define NS_STAMP(k)                                                        \
  do {                                                                     \
    if (a.dbg && blockIdx.x == 0 && tid == 0 && row == cid) a.dbg[k] = clock64(); \
  } while (0)

struct NucSetCtl {
  // weight histogram of the level in three 14-bit pieces (native 32-bit shared
  // atomics; a 64-bit shared add is a CAS loop), double-buffered by level parity
  uint32_t hp[2][3][256];
  uint32_t hc[2][256];  // count histogram
  u64 tw[256];          // cluster totals of the current level
  uint32_t tc[256];
  u64 tw2[256];         // (second half of the gather)
  uint32_t tc2[256];
  // level A: histogram over 1024 linear buckets of max - x (1/16 wide): three
  // 14-bit mass pieces and a count per bucket
  uint32_t ha[4][1024];
  u64 scan_w[16];       // level A block scan: per-warp totals
  uint32_t scan_c[16];
  int scan_b[16];
  u64 cand_k[32];       // the last <= 32 candidates of this CTA's slice (key, mass) for the final gather
  u64 cand_q[32];
  uint32_t cand_n;
  u64 pmax;             // this CTA's max key / total weight / non-finite flag
  u64 pw;
  uint32_t pbad;
  int sel_b;            // the scan's decision
  u64 sel_above, sel_w;
  uint32_t sel_cabove, sel_c;
};

__device__ __forceinline__ u64 key_of(double x) {
  const u64 b = (u64)__double_as_longlong(x + 0.0);  // -0 -> +0
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double value_of(u64 k) {
  const u64 b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}
__device__ __forceinline__ u64 ld_dsmem_u64(const void* local, uint32_t rank) {
  u64 v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(ptx::mapa(ptx::smem_addr(local), rank)));
  return v;
}
__device__ __forceinline__ uint32_t ld_dsmem_u32(const void* local, uint32_t rank) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(ptx::mapa(ptx::smem_addr(local), rank)));
  return v;
}

__global__ void __launch_bounds__(kNT, 1) nucleus_set_kernel(const NucSetArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  u64* key = reinterpret_cast<u64*>(smem_raw);
  u64* qw = key + kLcap;
  NucSetCtl* c = reinterpret_cast<NucSetCtl*>(qw + kLcap);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = ptx::cluster_ctarank();
  const uint32_t C = ptx::cluster_nctarank();
  const int64_t cid = ptx::cluster_id_x();
  const int64_t ncl = ptx::nclusters_x();
  const int64_t base = (int64_t)rank * a.L;
  const int64_t rem = a.n - base;
  const int len = rem <= 0 ? 0 : (rem < a.L ? (int)rem : a.L);
  // level A pays for its 1024-bucket gather only in clusters of up to 8 CTAs (16 peers: 128
  // DSMEM loads per thread); larger ones run the key descent from the top byte
  const bool useA = C <= 8;

  for (int64_t row = cid; row < a.B; row += ncl) {
    if (tid == 0) {
      c->pmax = 0;
      c->pw = 0;
      c->pbad = 0;
    }
    if (useA)
      for (int b = tid; b < 4 * 1024; b += kNT) (&c->ha[0][0])[b] = 0u;
    __syncthreads();
    NS_STAMP(0);
    // ---- keys, row maximum, non-finite check ---------------------------------
    {
      const double* xr = a.x + row * a.ldx + base;
      u64 kmx = 0;
      uint32_t bad = 0;
      for (int i = tid; i < len; i += kNT) {
        const double x = __ldcs(xr + i);
        bad |= !isfinite(x);
        const u64 k = key_of(x);
        key[i] = k;
        kmx = k > kmx ? k : kmx;
      }
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) {
        const u64 o = __shfl_xor_sync(0xffffffffu, kmx, m);
        kmx = o > kmx ? o : kmx;
      }
      bad = __any_sync(0xffffffffu, bad);
      if (lane == 0) {
        atomicMax(&c->pmax, kmx);
        if (bad) atomicOr(&c->pbad, 1u);
      }
    }
    NS_STAMP(1);
    ptx::cluster_sync();  // every CTA's partials are visible cluster-wide
    NS_STAMP(2);
    // lane r reads CTA r's partials (one DSMEM round trip), every warp combines them
    u64 kmax = lane < (int)C ? ld_dsmem_u64(&c->pmax, (uint32_t)lane) : 0ull;
    uint32_t bad = lane < (int)C ? ld_dsmem_u32(&c->pbad, (uint32_t)lane) : 0u;
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) {
      const u64 o = __shfl_xor_sync(0xffffffffu, kmax, m);
      kmax = o > kmax ? o : kmax;
    }
    bad = __any_sync(0xffffffffu, bad);
    if (bad) {  // cluster-uniform
      if (rank == 0 && tid == 0) {
        if (a.cutoff) a.cutoff[row] = (double)NAN;
        if (a.size) a.size[row] = 0;
        if (a.mass) a.mass[row] = (double)NAN;
        if (a.status) a.status[row] = PAM_ERR_NON_FINITE;
      }
      ptx::cluster_sync();  // nobody resets its partials while a peer still reads them
      continue;
    }
    // ---- fixed-point softmax masses and their total ----------------------------
    const double mx = value_of(kmax);
    {
      u64 ws = 0;
#pragma unroll 4
      for (int i = tid; i < len; i += kNT) {
        const double t = value_of(key[i]) - mx;
        // exp_t_core = exp_t on [-708, 709] (no special case can occur on [-64, 0])
        const double e = exp_t_core(t < -64.0 ? -64.0 : t, PAM_EXPT_E2);
        const u64 q = t < -64.0 ? 0ull : (u64)(e * 0x1p40 + 0.5);
        qw[i] = q;
        ws += q;
        if (useA && q > 0) {  // level A histogram (q > 0 => t > -29: bucket < 1024)
          const int bA = (int)(-t * 16.0);
          atomicAdd(&c->ha[0][bA], (uint32_t)q & 0x3fffu);
          atomicAdd(&c->ha[1][bA], (uint32_t)(q >> 14) & 0x3fffu);
          atomicAdd(&c->ha[2][bA], (uint32_t)(q >> 28));
          atomicAdd(&c->ha[3][bA], 1u);
        }
      }
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, m);
      if (lane == 0) atomicAdd(&c->pw, ws);
    }
    NS_STAMP(3);
    ptx::cluster_sync();
    NS_STAMP(4);
    u64 W = lane < (int)C ? ld_dsmem_u64(&c->pw, (uint32_t)lane) : 0ull;
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) W += __shfl_xor_sync(0xffffffffu, W, m);
    const double pW = a.p * (double)W;

    // ---- level A: 1024 linear buckets of max - x (value space) -------------------
    // The top bytes of the key are sign and exponent: nearly every entry shares
    // them, so two radix levels would pass over the whole slice for nothing.  A
    // monotone value-space split spreads the entries instead; the key descent
    // then starts below the bytes the chosen bucket's bounds have in common.
    u64 prefix = 0, above = 0;  // above = A(everything in the current bucket's range)
    uint32_t cabove = 0;
    u64 eq_w = 0;
    uint32_t eq_c = 0;
    int selA = 0;
    if (useA) {
      // thread t gathers buckets 2t and 2t + 1 (ascending bucket = descending x)
      u64 w2[2] = {0, 0};
      uint32_t c2[2] = {0, 0};
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int b = 2 * tid + j;
        for (uint32_t r0 = 0; r0 < C; r0 += 4) {
          uint32_t v[4][4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int q = 0; q < 4; ++q) v[u][q] = r0 + u < C ? ld_dsmem_u32(&c->ha[q][b], r0 + u) : 0u;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            w2[j] += (u64)v[u][0] + ((u64)v[u][1] << 14) + ((u64)v[u][2] << 28);
            c2[j] += v[u][3];
          }
        }
      }
      // block exclusive scan of (mass, count) over the 1024 buckets
      u64 iw = w2[0] + w2[1];
      uint32_t ic = c2[0] + c2[1];
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        const u64 ow = __shfl_up_sync(0xffffffffu, iw, m);
        const uint32_t oc = __shfl_up_sync(0xffffffffu, ic, m);
        if (lane >= m) {
          iw += ow;
          ic += oc;
        }
      }
      if (lane == 31) {
        c->scan_w[warp] = iw;
        c->scan_c[warp] = ic;
      }
      __syncthreads();
      u64 xw = iw - (w2[0] + w2[1]);  // exclusive within the warp
      uint32_t xc = ic - (c2[0] + c2[1]);
      for (int w = 0; w < warp; ++w) {
        xw += c->scan_w[w];
        xc += c->scan_c[w];
      }
      // the largest bucket index that is non-empty and whose top entry is inside
      int mine = -1;
      if (c2[0] > 0 && (double)xw < pW) mine = 2 * tid;
      if (c2[1] > 0 && (double)(xw + w2[0]) < pW) mine = 2 * tid + 1;
      const int wmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)(mine + 1)) - 1;
      if (lane == 0) c->scan_b[warp] = wmax;
      __syncthreads();
      int sel = -1;
      for (int w = 0; w < kNT / 32; ++w) sel = c->scan_b[w] > sel ? c->scan_b[w] : sel;
      if (mine == sel && sel >= 0) {
        const int j = sel & 1;
        c->sel_b = sel;
        c->sel_above = xw + (j ? w2[0] : 0ull);
        c->sel_cabove = xc + (j ? c2[0] : 0u);
        c->sel_w = w2[j];
        c->sel_c = c2[j];
      }
      __syncthreads();
      selA = c->sel_b;
      above = c->sel_above;
      cabove = c->sel_cabove;
      eq_w = c->sel_w;
      eq_c = c->sel_c;
    }
    auto in_selA = [&](const u64 k) { return !useA || (int)((mx - value_of(k)) * 16.0) == selA; };
    // ---- key descent inside that bucket: 8 key bits per level ---------------------
    int done_bits = 64;  // key bits fixed by the descent (64: all levels ran; 0: level A alone)
    int lvl0 = 0;
    if (!useA) {
      // (the descent starts at the top byte with every entry of positive mass a candidate)
    } else if (eq_c <= 32u) {
      done_bits = 0;
      lvl0 = 8;
    } else {  // the bucket's entries lie in [lo, hi] (bounds widened past any rounding of max - x)
      const double delta = (fabs(mx) + 64.0) * 0x1p-48;
      const u64 klo = key_of(mx - (double)(selA + 1) * 0.0625 - delta), khi = key_of(mx - (double)selA * 0.0625 + delta);
      const int shared = (klo == khi) ? 64 : __clzll((long long)(klo ^ khi));
      lvl0 = shared / 8 > 7 ? 7 : shared / 8;
      prefix = lvl0 ? khi >> (64 - 8 * lvl0) : 0ull;
    }
    for (int lvl = lvl0; lvl < 8; ++lvl) {
      const int shift = 56 - 8 * lvl;
      uint32_t* h0 = c->hp[lvl & 1][0];
      uint32_t* h1 = c->hp[lvl & 1][1];
      uint32_t* h2 = c->hp[lvl & 1][2];
      uint32_t* hc = c->hc[lvl & 1];
      for (int b = tid; b < 256; b += kNT) {
        h0[b] = 0;
        h1[b] = 0;
        h2[b] = 0;
        hc[b] = 0;
      }
      __syncthreads();
#pragma unroll 2
      for (int i0 = 0; i0 < len; i0 += kNT) {
        const int i = i0 + tid;
        u64 k = 0, q = 0;
        if (i < len) {
          k = key[i];
          q = qw[i];
        }
        const bool cand = q > 0 && (lvl == 0 || (k >> (shift + 8)) == prefix) && in_selA(k);
        const uint32_t cm = __ballot_sync(0xffffffffu, cand);
        if (cm == 0u) continue;  // warp-uniform
        const uint32_t d = (uint32_t)(k >> shift) & 255u;
        // few distinct digits in the warp (the exponent levels, tie groups): one
        // REDUX pair and one atomic per digit; many: the buckets are spread and
        // direct atomics do not contend (a REDUX per distinct digit would serialise)
        // (a group is worth its three REDUX only from 8 lanes up)
        const uint32_t d0 = __shfl_sync(0xffffffffu, d, __ffs(cm) - 1);
        uint32_t m0 = __ballot_sync(0xffffffffu, cand && d == d0);
        const uint32_t rest = cm & ~m0;
        if (__popc(m0) < 8) m0 = 0u;
        uint32_t m1 = 0u, d1 = 0u;
        if (__popc(rest) >= 8) {  // warp-uniform
          d1 = __shfl_sync(0xffffffffu, d, __ffs(rest) - 1);
          m1 = __ballot_sync(0xffffffffu, cand && d == d1);
          if (__popc(m1) < 8) m1 = 0u;
        }
        // q < 2^41 in three 14-bit pieces: a CTA's bucket sums stay below 2^32
        const uint32_t q0 = (uint32_t)q & 0x3fffu, q1 = (uint32_t)(q >> 14) & 0x3fffu, q2 = (uint32_t)(q >> 28);
        if (m0) {  // warp-uniform
          const bool in0 = (m0 >> lane) & 1u;
          const uint32_t s0 = __reduce_add_sync(0xffffffffu, in0 ? q0 : 0u);
          const uint32_t s1 = __reduce_add_sync(0xffffffffu, in0 ? q1 : 0u);
          const uint32_t s2 = __reduce_add_sync(0xffffffffu, in0 ? q2 : 0u);
          if (lane == 0) {
            atomicAdd(&h0[d0], s0);
            atomicAdd(&h1[d0], s1);
            atomicAdd(&h2[d0], s2);
            atomicAdd(&hc[d0], (uint32_t)__popc(m0));
          }
        }
        if (m1) {  // warp-uniform
          const bool in1 = (m1 >> lane) & 1u;
          const uint32_t s0 = __reduce_add_sync(0xffffffffu, in1 ? q0 : 0u);
          const uint32_t s1 = __reduce_add_sync(0xffffffffu, in1 ? q1 : 0u);
          const uint32_t s2 = __reduce_add_sync(0xffffffffu, in1 ? q2 : 0u);
          if (lane == 0) {
            atomicAdd(&h0[d1], s0);
            atomicAdd(&h1[d1], s1);
            atomicAdd(&h2[d1], s2);
            atomicAdd(&hc[d1], (uint32_t)__popc(m1));
          }
        }
        if (cand && !(((m0 | m1) >> lane) & 1u)) {  // the remaining digits: direct
          atomicAdd(&h0[d], q0);
          atomicAdd(&h1[d], q1);
          atomicAdd(&h2[d], q2);
          atomicAdd(&hc[d], 1u);
        }
      }
      NS_STAMP(5 + 4 * lvl);
      ptx::cluster_sync();  // the cluster's histograms of this level are complete
      NS_STAMP(6 + 4 * lvl);
      {  // thread (b, h) gathers bucket b of the CTAs r = h, h + 2, ...: all loads in flight at once
        const int b = tid & 255, h = tid >> 8;
        uint32_t v0[8], v1[8], v2[8], nv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t r = (uint32_t)(h + 2 * j);
          v0[j] = r < C ? ld_dsmem_u32(&h0[b], r) : 0u;
          v1[j] = r < C ? ld_dsmem_u32(&h1[b], r) : 0u;
          v2[j] = r < C ? ld_dsmem_u32(&h2[b], r) : 0u;
          nv[j] = r < C ? ld_dsmem_u32(&hc[b], r) : 0u;
        }
        u64 w = 0;
        uint32_t n_ = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          w += (u64)v0[j] + ((u64)v1[j] << 14) + ((u64)v2[j] << 28);
          n_ += nv[j];
        }
        if (h == 1) {
          c->tw2[b] = w;
          c->tc2[b] = n_;
        }
        __syncthreads();
        if (h == 0) {
          c->tw[b] = w + c->tw2[b];
          c->tc[b] = n_ + c->tc2[b];
        }
      }
      __syncthreads();
      NS_STAMP(7 + 4 * lvl);
      if (warp == 0) {
        // lane l owns buckets 8l .. 8l+7; suffix sums over the lanes above it
        u64 sw = 0;
        uint32_t sc = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          sw += c->tw[8 * lane + j];
          sc += c->tc[8 * lane + j];
        }
        u64 aw = sw;  // inclusive suffix scan (lanes >= l)
        uint32_t ac = sc;
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
          const u64 ow = __shfl_down_sync(0xffffffffu, aw, m);
          const uint32_t oc = __shfl_down_sync(0xffffffffu, ac, m);
          if (lane + m < 32) {
            aw += ow;
            ac += oc;
          }
        }
        u64 rw = above + (aw - sw);  // weight strictly above this lane's top bucket
        uint32_t rc = cabove + (ac - sc);
        int best = 256;
        u64 best_rw = 0;
        uint32_t best_rc = 0;
#pragma unroll
        for (int j = 7; j >= 0; --j) {
          const int b = 8 * lane + j;
          const u64 w = c->tw[b];
          const uint32_t n_ = c->tc[b];
          if (n_ > 0 && (double)rw < pW) {  // the bucket's largest entry is inside
            best = b;
            best_rw = rw;
            best_rc = rc;
          }
          rw += w;
          rc += n_;
        }
        const int sel = (int)__reduce_min_sync(0xffffffffu, (unsigned)best);
        if (best == sel && sel < 256) {
          c->sel_b = sel;
          c->sel_above = best_rw;
          c->sel_cabove = best_rc;
          c->sel_w = c->tw[sel];
          c->sel_c = c->tc[sel];
        }
      }
      __syncthreads();
      NS_STAMP(8 + 4 * lvl);
      prefix = (prefix << 8) | (u64)(uint32_t)c->sel_b;
      above = c->sel_above;
      cabove = c->sel_cabove;
      eq_w = c->sel_w;
      eq_c = c->sel_c;
      // (the next level zeroes the other histogram buffer: a peer that still reads
      //  this level's has not reached the next cluster barrier)
      if (lvl < 7 && eq_c <= 32u) {  // cluster-uniform: few survivors, finish without more levels
        done_bits = 8 * (lvl + 1);
        break;
      }
    }
    if (done_bits < 64) {
      // ---- final gather: the <= 32 entries whose key starts with `prefix` ----------
      const int sh = 64 - done_bits;
      if (tid == 0) c->cand_n = 0;
      __syncthreads();
      for (int i = tid; i < len; i += kNT) {
        const u64 k = key[i], q = qw[i];
        if (q > 0 && (done_bits == 0 || (k >> sh) == prefix) && in_selA(k)) {
          const uint32_t slot = atomicAdd(&c->cand_n, 1u);
          if (slot < 32u) {
            c->cand_k[slot] = k;
            c->cand_q[slot] = q;
          }
        }
      }
      ptx::cluster_sync();
      if (rank == 0 && warp == 0) {
        // lane l takes the l-th candidate of the cluster (CTA order, then slot order)
        const uint32_t cn = lane < (int)C ? ld_dsmem_u32(&c->cand_n, (uint32_t)lane) : 0u;
        uint32_t inc = cn;
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
          const uint32_t o = __shfl_up_sync(0xffffffffu, inc, m);
          if (lane >= m) inc += o;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
        uint32_t rr = 0, jj = 0;
        for (uint32_t r = 0; r < C; ++r) {
          const uint32_t e = __shfl_sync(0xffffffffu, inc - cn, (int)r), n_ = __shfl_sync(0xffffffffu, cn, (int)r);
          if ((uint32_t)lane >= e && (uint32_t)lane < e + n_) {
            rr = r;
            jj = (uint32_t)lane - e;
          }
        }
        const bool have = (uint32_t)lane < total;
        const u64 kl = have ? ld_dsmem_u64(&c->cand_k[jj], rr) : 0ull;
        const u64 ql = have ? ld_dsmem_u64(&c->cand_q[jj], rr) : 0ull;
        u64 al = above;  // mass strictly above this candidate
        for (int m = 0; m < 32; ++m) {
          const u64 km = __shfl_sync(0xffffffffu, kl, m), qm = __shfl_sync(0xffffffffu, ql, m);
          if ((uint32_t)m < total && km > kl) al += qm;
        }
        const bool in = have && (double)al < pW;
        u64 kc = in ? kl : ~0ull;  // the smallest inside key (the largest candidate is always inside)
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) {
          const u64 o = __shfl_xor_sync(0xffffffffu, kc, m);
          kc = o < kc ? o : kc;
        }
        const bool ge = have && kl >= kc;
        u64 mq = ge ? ql : 0ull;
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) mq += __shfl_xor_sync(0xffffffffu, mq, m);
        const uint32_t cnt = (uint32_t)__popc(__ballot_sync(0xffffffffu, ge));
        if (lane == 0) {
          if (a.cutoff) a.cutoff[row] = value_of(kc);
          if (a.size) a.size[row] = (int32_t)(cabove + cnt);
          if (a.mass) a.mass[row] = (double)(above + mq) / (double)W;
          if (a.status) a.status[row] = PAM_OK;
        }
      }
    } else if (rank == 0 && tid == 0) {
      if (a.cutoff) a.cutoff[row] = value_of(prefix);
      if (a.size) a.size[row] = (int32_t)(cabove + eq_c);
      if (a.mass) a.mass[row] = (double)(above + eq_w) / (double)W;
      if (a.status) a.status[row] = PAM_OK;
    }
    ptx::cluster_sync();  // partials and histograms are reset only after every peer is done
  }
}

}  // namespace
}  // namespace pam

static long long* g_nucset_dbg = nullptr;
extern "C" void pam_dev_nucleus_set_clocks(long long* d_buf40) { g_nucset_dbg = d_buf40; }

extern "C" int pam_nucleus_set_batch_f64(const double* d_x, int64_t ld_x, int64_t B, int64_t n, double p,
                                         double* d_cutoff, int32_t* d_size, double* d_mass, int32_t* d_row_status,
                                         void* stream) {
  using namespace pam;
  if (B < 0 || n < 1 || ld_x < n || (B > 0 && !d_x)) return PAM_ERR_BAD_ARGUMENT;
  if (!(p > 0.0 && p < 1.0)) return PAM_ERR_DOMAIN;
  if (B == 0) return PAM_OK;
  if (n > (int64_t)16 * kLcap) return PAM_ERR_UNSUPPORTED;  // 180224 entries per row
  int C = 1;
  while ((int64_t)C * kLcap < n) C *= 2;
  NucSetArgs ka;
  ka.x = d_x;
  ka.ldx = ld_x;
  ka.B = B;
  ka.n = n;
  ka.L = (int32_t)((n + C - 1) / C);
  ka.p = p;
  ka.cutoff = d_cutoff;
  ka.size = d_size;
  ka.mass = d_mass;
  ka.status = d_row_status;
  ka.dbg = g_nucset_dbg;
  const int smem = 2 * kLcap * 8 + (int)sizeof(NucSetCtl);
  const void* fn = (const void*)nucleus_set_kernel;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return pam_internal_cuda_fail((int)e, "cudaFuncSetAttribute(nucleus set smem)");
  if (C > 8) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return pam_internal_cuda_fail((int)e, "cudaFuncSetAttribute(nucleus set cluster)");
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kNT);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = (cudaStream_t)stream;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3((unsigned)C);
  int maxcl = 0;
  e = cudaOccupancyMaxActiveClusters(&maxcl, fn, &cfg);
  if (e != cudaSuccess || maxcl <= 0)
    return pam_internal_cuda_fail((int)(e != cudaSuccess ? e : cudaErrorInvalidConfiguration),
                                  "cudaOccupancyMaxActiveClusters(nucleus set)");
  const int64_t clusters = B < maxcl ? B : maxcl;
  cfg.gridDim = dim3((unsigned)(clusters * C));
  void* args[] = {&ka};
  e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e != cudaSuccess) return pam_internal_cuda_fail((int)e, "cudaLaunchKernelExC(nucleus set)");
  pam_internal_count_launch();
  return PAM_OK;
}
