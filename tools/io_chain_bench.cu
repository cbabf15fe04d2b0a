// io_chain_bench.cu — upper bound of the rows kernel's I/O structure (dev tool).
// Each CTA owns one slice position of its cluster's rows and moves slices
// HBM -> shared memory -> HBM with TMA bulk copies and NO compute:
//   chain: wait X(r) landed -> [delay D cycles] -> store Z(r) in nch chunks ->
//          X(r+1) chunk i is loaded as soon as store chunk i has been read.
// NBUF independent chains per CTA (own buffer + mbarrier + DMA thread each) show
// what a deeper I/O queue would buy.  Prints GB/s (read + write) per setting.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../paper_2509_08383_b200/csrc/pam_ptx.cuh"
using namespace pam;

__global__ void __launch_bounds__(512, 1)
    chain(const double* x, double* z, long long n, long long B, int C, int L, int nbuf, int nch, int delay,
          long long* cyc) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ unsigned long long mb[4];
  const int rank = blockIdx.x % C, cid = blockIdx.x / C, ncl = gridDim.x / C;
  const long long base = (long long)rank * L;
  const long long rem = n - base;
  const int len = rem <= 0 ? 0 : (rem < L ? (int)rem : L);
  const uint32_t bytes = (uint32_t)len * 8u;
  const uint32_t bufsz = ((uint32_t)L * 8u + 127u) & ~127u;
  if (threadIdx.x == 0) {
    for (int k = 0; k < nbuf; ++k) ptx::mbar_init(ptx::smem_addr(&mb[k]), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const long long t0 = clock64();
  const int k = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && k < nbuf) {
    const uint64_t pol = ptx::policy_evict_first();
    const uint32_t bar = ptx::smem_addr(&mb[k]);
    const uint32_t buf = ptx::smem_addr(sm) + k * bufsz;
    const uint32_t chunk = ((bytes / nch + 15u) / 16u) * 16u;
    auto ld = [&](long long r, int i) {
      const uint32_t off = i * chunk;
      if (off >= bytes) return;
      const uint32_t nb = bytes - off < chunk ? bytes - off : chunk;
      ptx::bulk_g2s(buf + off, (const unsigned char*)(x + r * n + base) + off, nb, bar, pol);
    };
    uint32_t par = 0;
    long long r = cid + (long long)ncl * k;
    const long long step = (long long)ncl * nbuf;
    if (r < B) {
      ptx::mbar_arrive_expect_tx(bar, bytes);
      for (int i = 0; i < nch; ++i) ld(r, i);
    }
    for (; r < B; r += step) {
      ptx::mbar_wait_cta(bar, par);
      par ^= 1u;
      if (delay > 0) {
        const long long s = clock64();
        while (clock64() - s < delay) {
        }
      }
      for (int i = 0; i < nch; ++i) {
        const uint32_t off = i * chunk;
        if (off >= bytes) break;
        const uint32_t nb = bytes - off < chunk ? bytes - off : chunk;
        ptx::bulk_s2g((unsigned char*)(z + r * n + base) + off, buf + off, nb, pol);
        ptx::bulk_commit();
      }
      const long long nx = r + step;
      if (nx < B) {
        ptx::mbar_arrive_expect_tx(bar, bytes);
        for (int i = 0; i < nch; ++i) {
          ptx::bulk_wait_read_le(nch - 1 - i);
          ld(nx, i);
        }
      }
    }
    ptx::bulk_wait_all();
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main(int argc, char** argv) {
  const long long n = 151936, B = 4096;
  double *x, *z;
  long long* cyc;
  cudaMalloc(&x, n * B * 8);
  cudaMalloc(&z, n * B * 8);
  cudaMalloc(&cyc, 296 * 8);
  cudaMemset(x, 0, n * B * 8);
  cudaFuncSetAttribute(chain, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int C, ctas, nbuf, nch, delay; };
  const Cfg cfgs[] = {
      {9, 135, 1, 4, 0},   {9, 135, 1, 8, 0},    {9, 135, 1, 4, 2000}, {9, 135, 1, 4, 4000}, {9, 135, 1, 4, 6000},
      {18, 144, 2, 4, 0},  {18, 144, 2, 4, 4000}, {18, 144, 2, 4, 8000}, {27, 135, 3, 4, 0},   {27, 135, 3, 4, 8000},
      {8, 144, 1, 4, 0},   {6, 132, 1, 4, 0},     {6, 132, 1, 8, 0},     {16, 144, 2, 4, 0},
  };
  for (const Cfg& c : cfgs) {
    int L = (int)((n + c.C - 1) / c.C);
    L = (L + 1) & ~1;
    const size_t smem = (size_t)c.nbuf * (((size_t)L * 8 + 127) & ~127) + 128;
    if (smem > 220 * 1024) { printf("C=%d nbuf=%d: smem %zu too large\n", c.C, c.nbuf, smem); continue; }
    float best = 1e9f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      chain<<<c.ctas, 512, smem>>>(x, z, n, B, c.C, L, c.nbuf, c.nch, c.delay, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    const double gbs = 2.0 * n * B * 8 / (best * 1e-3) / 1e9;
    const double rows_per_chain = (double)B / (c.ctas / c.C) / c.nbuf;
    printf("C=%2d ctas=%3d chains/CTA=%d chunks=%d delay=%5d: %.3f ms  %7.1f GB/s  (%.0f cycles per slice per chain) %s\n",
           c.C, c.ctas, c.nbuf, c.nch, c.delay, best, gbs, best * 1e-3 * 1.965e9 / rows_per_chain,
           err ? cudaGetErrorString(err) : "");
  }
  return 0;
}
