// store_bench.cu — per-SM store bandwidth: TMA bulk S2G vs STG.128 (dev tool).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2509_08383_b200/csrc/pam_ptx.cuh"
using namespace pam;

constexpr int BYTES = 151552;  // ~152 KB per CTA

__global__ void tma_store(double* out, long long* cyc, int chunk, int reps) {
  extern __shared__ __align__(128) unsigned char sm[];
  for (int i = threadIdx.x * 16; i < BYTES; i += blockDim.x * 16) *(double2*)(sm + i) = make_double2(i, 1);
  ptx::fence_proxy_async_smem();
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    uint64_t pol = ptx::policy_evict_first();
    for (int r = 0; r < reps; ++r) {
      unsigned char* dst = (unsigned char*)(out) + ((size_t)blockIdx.x * reps + r) * BYTES;
      for (int off = 0; off < BYTES; off += chunk) {
        int nb = BYTES - off < chunk ? BYTES - off : chunk;
        ptx::bulk_s2g(dst + off, ptx::smem_addr(sm) + off, nb, pol);
      }
      ptx::bulk_commit();
      ptx::bulk_wait_read_all();
    }
    ptx::bulk_wait_all();
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}

__global__ void stg_store(double* out, long long* cyc, int reps) {
  double2 v[19];
#pragma unroll
  for (int i = 0; i < 19; ++i) v[i] = make_double2(threadIdx.x + i, 1);
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    double2* dst = (double2*)((unsigned char*)(out) + ((size_t)blockIdx.x * reps + r) * BYTES);
#pragma unroll
    for (int i = 0; i < 19; ++i) __stcs(dst + i * blockDim.x + threadIdx.x, v[i]);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}

int main() {
  double* out;
  long long* cyc;
  size_t total = (size_t)148 * 8 * BYTES;
  cudaMalloc(&out, total);
  cudaMalloc(&cyc, 148 * 8);
  cudaFuncSetAttribute(tma_store, cudaFuncAttributeMaxDynamicSharedMemorySize, BYTES + 1024);
  long long h[148];
  for (int blocks : {1, 8, 74, 148}) {
    for (int chunk : {8192, 32768, BYTES}) {
      tma_store<<<blocks, 512, BYTES + 1024>>>(out, cyc, chunk, 8);
      tma_store<<<blocks, 512, BYTES + 1024>>>(out, cyc, chunk, 8);
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, 8 * blocks, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("TMA S2G blocks=%3d chunk=%6d: %6lld cycles per 152KB (%.1f B/clk/SM)\n", blocks, chunk, mx,
             (double)BYTES / mx);
    }
    stg_store<<<blocks, 512>>>(out, cyc, 8);
    stg_store<<<blocks, 512>>>(out, cyc, 8);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 8 * blocks, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("STG.128   blocks=%3d            : %6lld cycles per 152KB (%.1f B/clk/SM)\n", blocks, mx, (double)BYTES / mx);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
