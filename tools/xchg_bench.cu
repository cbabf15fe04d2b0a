// xchg_bench.cu — microbenchmark of cluster all-reduce designs (dev tool).
// Measures clock64 cycles per exchange of two doubles across a cluster with
// no other work, for:
//   0: warp-direct push (every warp pushes its partial to every CTA; every warp
//      reduces C*NW slots)
//   1: CTA pre-reduce (named barrier, warp 0 reduces, one slot per CTA; every
//      warp reduces C slots)
//   2: barrier.cluster + DSMEM loads (CTA partial in own smem, cluster barrier,
//      every warp reads C remote partials)
//   3: CTA pre-reduce, but only warp 0 receives and broadcasts via smem + barrier
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2509_08383_b200/csrc/pam_ptx.cuh"

using namespace pam;

struct __align__(16) Ctl {
  double2 slots[2][256];
  double2 wred[32];
  double2 bcast;
  double2 mine[2];
  unsigned long long mb[2];
};

__device__ __forceinline__ void bfly(double& a, double& b) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, m);
    b += __shfl_xor_sync(0xffffffffu, b, m);
  }
}

template <int NT, int MODE>
__global__ void xk(long long* out, int iters) {
  constexpr int NW = NT / 32;
  __shared__ Ctl cb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = ptx::cluster_ctarank(), C = ptx::cluster_nctarank();
  const uint32_t per = (MODE == 0) ? C * NW * 16u : C * 16u;
  if (tid == 0) {
    ptx::mbar_init(ptx::smem_addr(&cb.mb[0]), 1);
    ptx::mbar_init(ptx::smem_addr(&cb.mb[1]), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0 && MODE != 2) {
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb.mb[0]), per);
    ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb.mb[1]), per);
  }
  ptx::cluster_sync();
  double a = tid * 1e-3 + rank, b = 1.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t par = it & 1, ph = (it >> 1) & 1;
    if (MODE == 0) {
      bfly(a, b);
      if (lane < (int)C)
        ptx::st_async_f64x2(ptx::mapa(ptx::smem_addr(&cb.slots[par][rank * NW + warp]), lane), a, b,
                            ptx::mapa(ptx::smem_addr(&cb.mb[par]), lane));
      ptx::mbar_wait_cta(ptx::smem_addr(&cb.mb[par]), ph);
      if (tid == 0) ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb.mb[par]), per);
      a = 0; b = 0;
      for (int s = lane; s < (int)C * NW; s += 32) { double2 c = cb.slots[par][s]; a += c.x; b += c.y; }
      bfly(a, b);
    } else if (MODE == 1 || MODE == 3) {
      bfly(a, b);
      if (lane == 0) cb.wred[warp] = make_double2(a, b);
      __syncthreads();
      if (warp == 0) {
        double2 w = lane < NW ? cb.wred[lane] : make_double2(0, 0);
        a = w.x; b = w.y;
        bfly(a, b);
        if (lane < (int)C)
          ptx::st_async_f64x2(ptx::mapa(ptx::smem_addr(&cb.slots[par][rank]), lane), a, b,
                              ptx::mapa(ptx::smem_addr(&cb.mb[par]), lane));
      }
      if (MODE == 1) {
        ptx::mbar_wait_cta(ptx::smem_addr(&cb.mb[par]), ph);
        if (tid == 0) ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb.mb[par]), per);
        double2 c = lane < (int)C ? cb.slots[par][lane] : make_double2(0, 0);
        a = c.x; b = c.y;
        bfly(a, b);
      } else {
        if (warp == 0) {
          ptx::mbar_wait_cta(ptx::smem_addr(&cb.mb[par]), ph);
          if (lane == 0) ptx::mbar_arrive_expect_tx(ptx::smem_addr(&cb.mb[par]), per);
          double2 c = lane < (int)C ? cb.slots[par][lane] : make_double2(0, 0);
          a = c.x; b = c.y;
          bfly(a, b);
          if (lane == 0) cb.bcast = make_double2(a, b);
        }
        __syncthreads();
        a = cb.bcast.x; b = cb.bcast.y;
      }
    } else {  // MODE 2: cluster barrier + DSMEM reads
      bfly(a, b);
      if (lane == 0) cb.wred[warp] = make_double2(a, b);
      __syncthreads();
      if (warp == 0) {
        double2 w = lane < NW ? cb.wred[lane] : make_double2(0, 0);
        a = w.x; b = w.y;
        bfly(a, b);
        if (lane == 0) cb.mine[par] = make_double2(a, b);
      }
      ptx::cluster_sync();
      double2 c = make_double2(0, 0);
      if (lane < (int)C) {
        uint32_t ra = ptx::mapa(ptx::smem_addr(&cb.mine[par]), lane);
        asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(c.x), "=d"(c.y) : "r"(ra) : "memory");
      }
      a = c.x; b = c.y;
      bfly(a, b);
    }
    a *= 1e-9; b *= 1e-9;
  }
  long long t1 = clock64();
  ptx::cluster_sync();
  if (tid == 0) out[blockIdx.x] = (t1 - t0) / iters;
  if (tid == 0 && a == 12345.0) out[0] = 0;
}

template <int NT, int MODE>
void run(int C) {
  long long* d;
  cudaMalloc(&d, 1024 * 8);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(C * 4);
  cfg.blockDim = dim3(NT);
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaFuncSetAttribute(xk<NT, MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int iters = 2000;
  for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, xk<NT, MODE>, d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[64];
  cudaMemcpy(h, d, 8 * C * 4, cudaMemcpyDeviceToHost);
  long long mx = 0, mn = 1 << 30;
  for (int i = 0; i < C * 4; ++i) { mx = h[i] > mx ? h[i] : mx; mn = h[i] < mn ? h[i] : mn; }
  printf("mode=%d NT=%d C=%2d: %lld..%lld cycles/exchange %s\n", MODE, NT, C, mn, mx, e ? cudaGetErrorString(e) : "");
  cudaFree(d);
}

int main() {
  for (int C : {1, 2, 4, 8, 16}) {
    run<512, 0>(C); run<512, 1>(C); run<512, 2>(C); run<512, 3>(C);
    run<256, 0>(C); run<256, 1>(C); run<256, 3>(C);
  }
  return 0;
}
