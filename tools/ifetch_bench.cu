// ifetch_bench.cu — does a straight-line per-row code footprint above the
// 32 KB L1.5 instruction cache slow a 512-thread CTA down? (dev tool)
// Each "row" executes N FFMA (8 independent chains, distinct immediates) once;
// 135 CTAs x 512 threads, R rows.  Issue-bound time is 4*N cycles per row
// (4 warps per SMSP); a fetch-bound kernel takes longer.
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
__global__ void __launch_bounds__(512, 1) body(float* out, long long* cyc, int R) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < R; ++r) {
#pragma unroll
    for (int i = 0; i < N; ++i) a[i & 7] = fmaf(a[i & 7], 1.0f + (float)i * 1e-7f, (float)(i & 15) * 1e-3f);
    __syncthreads();
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * 512 + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / R;
}

template <int N>
void run(float* out, long long* cyc) {
  long long h[135];
  body<N><<<135, 512>>>(out, cyc, 50);
  body<N><<<135, 512>>>(out, cyc, 50);
  cudaDeviceSynchronize();
  cudaMemcpy(h, cyc, 135 * 8, cudaMemcpyDeviceToHost);
  long long m = 0;
  for (int i = 0; i < 135; ++i) m += h[i];
  m /= 135;
  printf("N=%5d (%5.1f KB of FFMA): %7lld cycles/row, %.2f cycles per instruction per SMSP-warp-slot (issue bound 4.00)\n",
         N, N * 16 / 1024.0, m, (double)m / N);
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 135 * 512 * 4);
  cudaMalloc(&cyc, 135 * 8);
  run<500>(out, cyc);
  run<1000>(out, cyc);
  run<1500>(out, cyc);
  run<1900>(out, cyc);
  run<2200>(out, cyc);
  run<3000>(out, cyc);
  run<4000>(out, cyc);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
