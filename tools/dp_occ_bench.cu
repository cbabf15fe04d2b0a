// dp_occ_bench.cu — fp64 pass throughput vs warps per SM (dev tool).
// Each thread keeps E doubles in registers and runs the CutMax element update
// (z = fma(v,k,b); v = fma(z*z, z, -K); s += v; q = fma(v,v,q)) R times.
#include <cstdio>
#include <cuda_runtime.h>

template <int E, int ACC>
__global__ void __launch_bounds__(1024, 1) pass_kernel(double* out, int R, double k, double b, double kn) {
  double v[E];
#pragma unroll
  for (int i = 0; i < E; ++i) v[i] = (threadIdx.x + i) * 1e-3;
  double s[ACC], q[ACC];
#pragma unroll
  for (int a = 0; a < ACC; ++a) { s[a] = 0; q[a] = 0; }
  long long t0 = clock64();
  for (int r = 0; r < R; ++r) {
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const double z = fma(v[i], k, b);
      const double z2 = z * z;
      const double d = fma(z2, z, kn);
      v[i] = d * 1e-3;
      s[i % ACC] += d;
      q[i % ACC] = fma(d, d, q[i % ACC]);
    }
  }
  long long t1 = clock64();
  double acc = 0;
#pragma unroll
  for (int a = 0; a < ACC; ++a) acc += s[a] + q[a];
#pragma unroll
  for (int i = 0; i < E; ++i) acc += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) out[1024 * 1024 + blockIdx.x] = (double)(t1 - t0);
}

template <int E, int ACC>
void run(int threads) {
  double* d;
  cudaMalloc(&d, (1024 * 1024 + 1024) * 8);
  int R = 200;
  pass_kernel<E, ACC><<<148, threads>>>(d, R, 0.1, 1.0, -1.1);
  pass_kernel<E, ACC><<<148, threads>>>(d, R, 0.1, 1.0, -1.1);
  cudaDeviceSynchronize();
  double cyc;
  cudaMemcpy(&cyc, d + 1024 * 1024, 8, cudaMemcpyDeviceToHost);
  double dp = 6.0 * E * R * threads;  // DFMA, DMUL, DFMA, DMUL(scale), DADD, DFMA
  printf("E=%2d ACC=%d threads=%4d (warps/SMSP=%2d): %.1f DP lane-ops/clk/SM (peak 64)\n", E, ACC, threads,
         threads / 128, dp / cyc);
  cudaFree(d);
}

int main() {
  for (int t : {128, 256, 384, 512, 768, 1024}) run<20, 2>(t);
  for (int t : {128, 256, 512}) run<38, 2>(t);
  for (int t : {128, 256, 512}) run<38, 4>(t);
  for (int t : {256, 512}) run<38, 8>(t);
  return 0;
}
