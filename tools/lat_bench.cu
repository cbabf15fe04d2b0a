// lat_bench.cu — dependent-chain latencies of the primitives the exchange uses (dev tool).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2509_08383_b200/csrc/pam_ptx.cuh"
using namespace pam;

__global__ void __cluster_dims__(1, 1, 1) lat(long long* out, double x, int n) {
  __shared__ unsigned long long mb;
  __shared__ double2 slot[4];
  double a = x + threadIdx.x, b = 1.0;
  long long t0, t1;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = a + b; a = a + b; a = a + b; a = a + b; }
  t1 = clock64(); if (threadIdx.x == 0) out[0] = (t1 - t0) / (4 * n);
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = fma(a, b, x); a = fma(a, b, x); a = fma(a, b, x); a = fma(a, b, x); }
  t1 = clock64(); if (threadIdx.x == 0) out[1] = (t1 - t0) / (4 * n);
  // FADD chain (fp32)
  float f = a, g = 1.0f;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { f = f + g; f = f + g; f = f + g; f = f + g; }
  t1 = clock64(); if (threadIdx.x == 0) out[2] = (t1 - t0) / (4 * n);
  // SHFL chain (64-bit)
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = __shfl_xor_sync(~0u, a, 1); a = __shfl_xor_sync(~0u, a, 2); a = __shfl_xor_sync(~0u, a, 4); a = __shfl_xor_sync(~0u, a, 8); }
  t1 = clock64(); if (threadIdx.x == 0) out[3] = (t1 - t0) / (4 * n);
  // shfl + dadd butterfly level
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) a += __shfl_xor_sync(~0u, a, m);
  }
  t1 = clock64(); if (threadIdx.x == 0) out[4] = (t1 - t0) / (5 * n);
  // mbarrier self arrive + wait (1 thread)
  if (threadIdx.x == 0) { ptx::mbar_init(ptx::smem_addr(&mb), 1); ptx::fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(ptx::smem_addr(&mb)) : "memory");
      ptx::mbar_wait_cta(ptx::smem_addr(&mb), i & 1);
    }
    t1 = clock64(); out[5] = (t1 - t0) / n;
    // st.async to self + wait
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
      ptx::mbar_arrive_expect_tx(ptx::smem_addr(&mb), 16);
      ptx::st_async_f64x2(ptx::mapa(ptx::smem_addr(&slot[0]), 0), a, b, ptx::mapa(ptx::smem_addr(&mb), 0));
      ptx::mbar_wait_cta(ptx::smem_addr(&mb), (n + i) & 1);
      a += slot[0].x;
    }
    t1 = clock64(); out[6] = (t1 - t0) / n;
  }
  __syncthreads();
  // __syncthreads cost (all threads)
  t0 = clock64();
  for (int i = 0; i < n; ++i) { __syncthreads(); }
  t1 = clock64(); if (threadIdx.x == 0) out[7] = (t1 - t0) / n;
  // rsqrt(double) latency
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = rsqrt(a + 2.0); }
  t1 = clock64(); if (threadIdx.x == 0) out[8] = (t1 - t0) / n;
  // division latency
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = 1.0 / (a + 2.0); }
  t1 = clock64(); if (threadIdx.x == 0) out[9] = (t1 - t0) / n;
  // LDS latency chain
  __shared__ int idx[64];
  if (threadIdx.x < 64) idx[threadIdx.x] = (threadIdx.x + 1) & 63;
  __syncthreads();
  int k = threadIdx.x & 63;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { k = idx[k]; k = idx[k]; k = idx[k]; k = idx[k]; }
  t1 = clock64(); if (threadIdx.x == 0) out[10] = (t1 - t0) / (4 * n);
  if (a == 12345.0 || f == 1.0f || k == 999) out[11] = 1;
}

int main() {
  long long* d; cudaMalloc(&d, 64 * 8);
  const char* names[] = {"DADD", "DFMA", "FADD", "SHFL64 chain (per shfl)", "butterfly level (shfl+dadd)", "mbarrier arrive+wait",
                         "st.async self + wait", "__syncthreads (256 thr)", "rsqrt(double)", "1.0/x double", "LDS chain"};
  for (int threads : {32, 256}) {
    lat<<<1, threads>>>(d, 0.5, 1000);
    lat<<<1, threads>>>(d, 0.5, 1000);
    cudaError_t e = cudaDeviceSynchronize(); if (e) printf("err %s\n", cudaGetErrorString(e));
    long long h[12]; cudaMemcpy(h, d, 12 * 8, cudaMemcpyDeviceToHost);
    printf("threads=%d\n", threads);
    for (int i = 0; i < 11; ++i) printf("  %-32s %lld cycles\n", names[i], h[i]);
  }
  return 0;
}
