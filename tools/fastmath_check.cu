// fastmath_check.cu — bit-for-bit check of the sampler's branch-free device
// forms (pam_div_nr, pam_log_fast, pam_exp_fast, beta_icdf_fast, gumbel_fast)
// against the portable functions the oracle mirrors (dev tool; exit 1 on any
// mismatch).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2509_08383_b200/csrc/pam_scalar.h"
using namespace pam;

__device__ unsigned long long g_bad[8];
__device__ double g_first[8][3];

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}
__device__ void report(int t, double in, double a, double b) {
  if (pam_double_to_bits(a) != pam_double_to_bits(b)) {
    if (atomicAdd(&g_bad[t], 1ULL) == 0) { g_first[t][0] = in; g_first[t][1] = a; g_first[t][2] = b; }
  }
}

__global__ void check(uint64_t seed, int per_thread) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (int i = 0; i < per_thread; ++i) {
    const uint64_t r = mix(seed ^ (tid * 0x9e3779b97f4a7c15ULL + i));
    const uint64_t r2 = mix(r + 0x1234567);
    // 0: division on the log's range: m in [sqrt(1/2), sqrt(2))
    const double m = 0x1.6a09e667f3bcdp-1 + (double)(r >> 11) * 0x1p-53 * (1.4142135623730951 - 0.7071067811865476);
    report(0, m, pam_div_nr(m - 1.0, m + 1.0), (m - 1.0) / (m + 1.0));
    // 1: log on the uniforms
    const double u = u01_from_bits((uint32_t)r, (uint32_t)(r >> 32));
    report(1, u, pam_log_fast(u), log_p(u));
    // 2: log on (1e-16, 40] (gumbel's outer log)
    const double w = -log_p(u);
    report(2, w, pam_log_fast(w), log_p(w));
    // 3: exp on [-700, 709]
    const double x = -700.0 + (double)(r2 >> 11) * 0x1p-53 * 1409.0;
    report(3, x, pam_exp_fast(x), exp_p(x));
    // 4: exp on [-2, 0] (beta noise, x - max near the top)
    const double x2 = -(double)(r2 >> 11) * 0x1p-52;
    report(4, x2, pam_exp_fast(x2), exp_p(x2));
    // 5: beta noise for alpha(0.9), alpha(0.95), 2, 1/19
    const double ia[4] = {1.0 / 21.854345326782836, 1.0 / 58.40397667459505, 0.5, 19.0};
    const double inv = ia[(r2 >> 3) & 3];
    report(5, u, beta_icdf_fast(u, inv), beta_icdf(u, inv));
    // 6: gumbel noise
    report(6, u, gumbel_fast(u), gumbel_from_u(u));
  }
}

int main() {
  const int blocks = 148 * 4, threads = 256, per = 512;
  unsigned long long zero[8] = {0};
  cudaMemcpyToSymbol(g_bad, zero, sizeof zero);
  for (int s = 0; s < 4; ++s) check<<<blocks, threads>>>(0x2509083830000ULL + s, per);
  cudaDeviceSynchronize();
  unsigned long long bad[8];
  double first[8][3];
  cudaMemcpyFromSymbol(bad, g_bad, sizeof bad);
  cudaMemcpyFromSymbol(first, g_first, sizeof first);
  const char* nm[7] = {"div (log range)", "log(uniform)", "log(-log u)", "exp[-700,709]", "exp[-2,0]", "beta_icdf", "gumbel"};
  const double n = 4.0 * blocks * threads * per;
  int fails = 0;
  for (int t = 0; t < 7; ++t) {
    printf("%-16s %.3g samples: %llu mismatches", nm[t], n, bad[t]);
    if (bad[t]) { printf("  (first: in %.17g fast %.17g ref %.17g)", first[t][0], first[t][1], first[t][2]); ++fails; }
    printf("\n");
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return fails ? 1 : 0;
}
