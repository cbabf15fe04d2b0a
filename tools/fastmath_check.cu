// fastmath_check.cu — bit-for-bit check of the sampler's branch-free device
// forms with the tables in shared memory (log_t_core, exp_t_core,
// beta_icdf_tab, gumbel_tab; pam_scalar.h) against the portable forms
// (log_t, exp_t, beta_icdf, gumbel_from_u) that the host library and the CPU
// oracle evaluate identically (dev tool; exit 1 on any mismatch).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o tools/fastmath_check tools/fastmath_check.cu
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

__global__ void check(uint64_t seed, int per_thread, double inv_alpha) {
  __shared__ double tabs[384];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) {
    tabs[i] = pam_d_logt_invc[i];
    tabs[128 + i] = pam_d_logt_logc[i];
    tabs[256 + i] = pam_d_expt_e2[i];
  }
  __syncthreads();
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (int i = 0; i < per_thread; ++i) {
    const uint64_t r = mix(seed ^ (tid * 0x9e3779b97f4a7c15ULL + i));
    const uint64_t r2 = mix(r + 0x1234567);
    // the sampler's uniforms: ((bits >> 12) + 0.5) 2^-52
    const double u = u01_from_bits((uint32_t)r, (uint32_t)(r >> 32));
    report(0, u, log_t_core(u, tabs, tabs + 128), log_t(u));
    // exp on the nucleus / Beta range [-700, 0]
    const double x = -700.0 * ((double)(r2 >> 11) * 0x1p-53);
    report(1, x, exp_t_core(x, tabs + 256), exp_t(x));
    report(2, u, beta_icdf_tab(u, inv_alpha, tabs), beta_icdf(u, inv_alpha));
    report(3, u, gumbel_tab(u, tabs), gumbel_from_u(u));
    // Gumbel's inner value -log u in [2^-53, 36.7]
    const double w = -log_t(u);
    report(4, w, log_t_core(w, tabs, tabs + 128), log_t(w));
  }
}

int main() {
  const char* names[5] = {"log_t_core(u)", "exp_t_core(x)", "beta_icdf_tab", "gumbel_tab", "log_t_core(-log u)"};
  const double inv_alphas[3] = {1.0 / 21.854345326782834, 1.0 / 3.0, 19.0};
  unsigned long long total = 0;
  int fail = 0;
  for (int a = 0; a < 3; ++a) {
    unsigned long long zero[8] = {0};
    cudaMemcpyToSymbol(g_bad, zero, sizeof zero);
    const int blocks = 148 * 8, threads = 256, per = 1024;
    check<<<blocks, threads>>>(0x5eed + a, per, inv_alphas[a]);
    if (cudaDeviceSynchronize() != cudaSuccess) { std::printf("kernel failed\n"); return 2; }
    unsigned long long bad[8];
    double first[8][3];
    cudaMemcpyFromSymbol(bad, g_bad, sizeof bad);
    cudaMemcpyFromSymbol(first, g_first, sizeof first);
    const unsigned long long n = (unsigned long long)blocks * threads * per;
    total += n;
    for (int t = 0; t < 5; ++t) {
      std::printf("inv_alpha %.6f %-20s %llu mismatches in %llu\n", inv_alphas[a], names[t], bad[t], n);
      if (bad[t]) {
        fail = 1;
        std::printf("   first: in %.17g fast %.17g portable %.17g\n", first[t][0], first[t][1], first[t][2]);
      }
    }
  }
  std::printf("%s (%llu samples per function)\n", fail ? "MISMATCH" : "all bit-identical", total);
  return fail;
}
