// load_bench.cu — per-SM load bandwidth: TMA bulk G2S (chunked) vs LDG.128 (dev tool).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2509_08383_b200/csrc/pam_ptx.cuh"
using namespace pam;

constexpr int BYTES = 135168;  // ~135 KB per CTA (one C=9 fp64 slice)

__global__ void tma_load(const double* in, long long* cyc, int nchunk, int reps, size_t stride) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ unsigned long long bar;
  if (threadIdx.x == 0) {
    ptx::mbar_init(ptx::smem_addr(&bar), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int chunk = ((BYTES / nchunk) + 15) / 16 * 16;
  uint64_t pol = ptx::policy_evict_first();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const unsigned char* src = (const unsigned char*)in + ((size_t)blockIdx.x * reps + r) * stride;
    if (threadIdx.x == 0) {
      ptx::mbar_arrive_expect_tx(ptx::smem_addr(&bar), BYTES);
      for (int off = 0; off < BYTES; off += chunk) {
        int nb = BYTES - off < chunk ? BYTES - off : chunk;
        ptx::bulk_g2s(ptx::smem_addr(sm) + off, src + off, nb, ptx::smem_addr(&bar), pol);
      }
    }
    ptx::mbar_wait_cta(ptx::smem_addr(&bar), r & 1);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}

__global__ void ldg_load(const double* in, long long* cyc, int reps, size_t stride, double* sink) {
  double2 acc = make_double2(0, 0);
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const double2* src = (const double2*)((const unsigned char*)in + ((size_t)blockIdx.x * reps + r) * stride);
    double2 v[17];
#pragma unroll
    for (int i = 0; i < 17; ++i) v[i] = __ldcs(src + i * blockDim.x + threadIdx.x);
#pragma unroll
    for (int i = 0; i < 17; ++i) {
      acc.x += v[i].x;
      acc.y += v[i].y;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
  if (acc.x == 12345.0) sink[0] = acc.y;
}

int main() {
  const int reps = 8;
  const size_t stride = 139264;
  double* in;
  long long* cyc;
  double* sink;
  size_t total = (size_t)148 * reps * stride + 4096;
  cudaMalloc(&in, total);
  cudaMemset(in, 0, total);
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(tma_load, cudaFuncAttributeMaxDynamicSharedMemorySize, BYTES + 1024);
  long long h[148];
  for (int blocks : {1, 16, 74, 135, 148}) {
    for (int nch : {1, 4, 8, 16, 33}) {
      for (int w = 0; w < 2; ++w) tma_load<<<blocks, 512, BYTES + 1024>>>(in, cyc, nch, reps, stride);
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, 8 * blocks, cudaMemcpyDeviceToHost);
      long long mx = 0, s = 0;
      for (int i = 0; i < blocks; ++i) {
        mx = h[i] > mx ? h[i] : mx;
        s += h[i];
      }
      printf("TMA G2S blocks=%3d chunks=%2d: max %6lld avg %6lld cycles per 135KB (%.1f B/clk/SM)\n", blocks, nch, mx,
             s / blocks, (double)BYTES / (s / blocks));
    }
    for (int w = 0; w < 2; ++w) ldg_load<<<blocks, 512>>>(in, cyc, reps, stride, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 8 * blocks, cudaMemcpyDeviceToHost);
    long long s = 0;
    for (int i = 0; i < blocks; ++i) s += h[i];
    printf("LDG.128 blocks=%3d          : avg %6lld cycles per 139KB (%.1f B/clk/SM)\n", blocks, s / blocks,
           139264.0 / (s / blocks));
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
