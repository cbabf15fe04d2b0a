// chain_bench.cu — latency of the ahead kernel's control-chain phase B in one
// warp (dev tool).  Dependent loop: each call's output feeds the next input.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2509_08383_b200/csrc/cutmax_ahead_kernel.cuh"
using namespace pam;

__global__ void chainb(const CutmaxArgs a, long long* cyc, double* out, int reps, int i, int T) {
  const int lane = threadIdx.x & 31;
  double Sl = lane < 9 ? 1.0 + 0.1 * lane : 0.0;
  AhCoefA ca{0.2, 0.9, 0, 0};
  double acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    double S[10];
    S[0] = 151936.0;
#pragma unroll
    for (int j = 1; j <= 9; ++j) S[j] = __shfl_sync(0xffffffffu, Sl, j - 1);
    const AhCoefB b = i == 0 ? ah_phase_b_t<6, true, false>(S, ca, 0, 1.0 / 151936.0, 1e-24, a.rp)
                             : ah_phase_b_t<9, true, true>(S, ca, 2, 1.0 / 151936.0, 1e-24, a.rp);
    acc += b.kb + b.rn;
    ca.aa = 0.9 + 1e-30 * b.bb;  // dependency
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}

int main() {
  CutmaxArgs a{};
  a.rp.T = 4;
  for (int t = 0; t < 4; ++t) { a.rp.inv_c[t] = 0.2; a.rp.kshift[t + 1] = 1.12; }
  a.rp.eps_var = 1e-24;
  long long* cyc; double* out;
  cudaMalloc(&cyc, 8); cudaMalloc(&out, 32 * 8);
  long long h;
  for (int reps : {100, 1}) {
    for (int i = 0; i < 2; ++i) {
      chainb<<<1, 32>>>(a, cyc, out, reps, i, 4);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("phase B stage %d (T=4) reps=%d: %lld cycles per call\n", i, reps, h);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
