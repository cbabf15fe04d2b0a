// pass_bench.cu — cycles per element pass of the ahead kernel's mid / last
// passes in isolation (512 threads x E=34 registers, 1 CTA per SM), plus
// fp64 scalar-op latencies used by the control chain (dev tool).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2509_08383_b200/csrc/cutmax_ahead_kernel.cuh"
using namespace pam;

constexpr int NTG = 512, E = 34;

template <int MODE>
__global__ void __launch_bounds__(NTG, 1) passk(double* out, long long* cyc, int reps, double ka, double aa, double kb,
                                                double bb, double kn) {
  double v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = 1e-3 * (threadIdx.x + e);
  double s[kAhMaxM];
  const int len = 17000;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll
  for (int j = 0; j < kAhMaxM; ++j) s[j] = 0.0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int q = 0; q < E / 2; ++q) {
      const bool ok = (q * NTG + (int)threadIdx.x) * 2 < len;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (MODE == 0) {  // ahead mid pass, S_1..S_9
          const double y = ah_cube(fma(v[2 * q + h], ka, aa));
          const double z2 = fma(y, kb, bb);
          double w = fma(z2 * z2, z2, -kn);
          w = ok ? w : 0.0;
          v[2 * q + h] = w;
          ah_acc<9>(s, w);
        } else if (MODE == 1) {  // old kernel pass: update + 2 sums
          const double z = fma(v[2 * q + h], ka, aa);
          const double w = fma(z * z, z, -kn);
          v[2 * q + h] = w;
          s[h] += w;
          s[2 + h] = fma(w, w, s[2 + h]);
        } else {  // mid pass without the phantom select
          const double y = ah_cube(fma(v[2 * q + h], ka, aa));
          const double z2 = fma(y, kb, bb);
          const double w = fma(z2 * z2, z2, -kn);
          v[2 * q + h] = w;
          ah_acc<9>(s, w);
        }
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  double acc = 0;
#pragma unroll
  for (int j = 0; j < kAhMaxM; ++j) acc += s[j];
#pragma unroll
  for (int e = 0; e < E; ++e) acc += v[e];
  out[blockIdx.x * NTG + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}

__global__ void lat(long long* out, double x, int n) {
  double a = x + threadIdx.x, b = 1.000001;
  long long t0, t1;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = fma(a, b, x); a = fma(a, b, x); a = fma(a, b, x); a = fma(a, b, x); }
  t1 = clock64(); out[0] = (t1 - t0) / (4 * n);
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = x / a; }
  t1 = clock64(); out[1] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = sqrt(a) + x; }
  t1 = clock64(); out[2] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = rsqrt(a) + x; }
  t1 = clock64(); out[3] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = a * a; a = a * b; a = a * a; a = a * b; }
  t1 = clock64(); out[4] = (t1 - t0) / (4 * n);
  out[5] = (long long)a;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 148 * NTG * 8);
  cudaMalloc(&cyc, 148 * 8);
  long long h[148];
  const char* nm[3] = {"ahead mid pass (S1..S9, select)", "old pass (2 sums)", "ahead mid pass (no select)"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int blocks : {1, 135}) {
      for (int it = 0; it < 2; ++it) {
        if (mode == 0) passk<0><<<blocks, NTG>>>(out, cyc, 20, 0.2, 0.9, 0.3, 0.7, 1.12);
        if (mode == 1) passk<1><<<blocks, NTG>>>(out, cyc, 20, 0.2, 0.9, 0.3, 0.7, 1.12);
        if (mode == 2) passk<2><<<blocks, NTG>>>(out, cyc, 20, 0.2, 0.9, 0.3, 0.7, 1.12);
      }
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, 8 * blocks, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("%-36s blocks=%3d: %6lld cycles per pass of %d elements (%.3f clk/elem/SM)\n", nm[mode], blocks, mx,
             NTG * E, (double)mx / (NTG * E));
    }
  }
  lat<<<1, 32>>>(cyc, 1.5, 1000);
  cudaDeviceSynchronize();
  cudaMemcpy(h, cyc, 8 * 6, cudaMemcpyDeviceToHost);
  printf("latency cycles: DFMA %lld  ddiv %lld  dsqrt(+dadd) %lld  rsqrt(+dadd) %lld  DMUL %lld\n", h[0], h[1], h[2],
         h[3], h[4]);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
