// Device-facts probe (first gpurun call): SM count, smem, cluster occupancy,
// fp64 pipe throughput, PCIe copy bandwidth.  Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

template<int OP>
__global__ void dp_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) { x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b); x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);}
      if (OP == 1) { x0 = x0 + b; x1 = x1 + b; x2 = x2 + b; x3 = x3 + b; x4 = x4 + b; x5 = x5 + b; x6 = x6 + b; x7 = x7 + b;}
      if (OP == 2) { x0 = x0 * a; x1 = x1 * a; x2 = x2 * a; x3 = x3 * a; x4 = x4 * a; x5 = x5 * a; x6 = x6 * a; x7 = x7 * a;}
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void __cluster_dims__(1,1,1) dummy_cluster(double* p) { if (p) p[0] = 1; }
__global__ void dummy(double* p) { extern __shared__ double s[]; if (p) { s[threadIdx.x] = 1; p[threadIdx.x] = s[threadIdx.x^1]; } }

int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  printf("name=%s sms=%d cc=%d.%d smemPerBlockOptin=%zu smemPerSM=%zu regsPerSM=%d l2=%d clock=%d memclk=%d busw=%d\n",
         pr.name, pr.multiProcessorCount, pr.major, pr.minor, pr.sharedMemPerBlockOptin,
         pr.sharedMemPerMultiprocessor, pr.regsPerMultiprocessor, pr.l2CacheSize, pr.clockRate, pr.memoryClockRate, pr.memoryBusWidth);
  double* out; CK(cudaMalloc(&out, 148 * 8 * 1024 * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[3] = {"DFMA", "DADD", "DMUL"};
  for (int op = 0; op < 3; ++op) {
    int iters = 4096; int blocks = 148 * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (op == 0) dp_kernel<0><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
      if (op == 1) dp_kernel<1><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
      if (op == 2) dp_kernel<2><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = double(blocks) * threads * iters * 64;
      if (rep) printf("%s: %.3f ms  %.2f Tinst/s  per-SM-per-clk(@%.0fMHz)=%.1f\n", names[op], ms, ops / ms / 1e9,
                      pr.clockRate / 1e3, ops / (ms * 1e-3) / 148 / (pr.clockRate * 1e3));
    }
  }
  // cluster occupancy for various (cluster size, threads, smem)
  int sizes[5] = {1, 2, 4, 8, 16};
  CK(cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  int smems[4] = {40 * 1024, 78 * 1024, 110 * 1024, 160 * 1024};
  int thr[3] = {256, 384, 512};
  for (int si = 0; si < 4; ++si) for (int ti = 0; ti < 3; ++ti) for (int c = 0; c < 5; ++c) {
    cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute at[1];
    cfg.gridDim = dim3(sizes[c] * 64); cfg.blockDim = dim3(thr[ti]); cfg.dynamicSmemBytes = smems[si];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = sizes[c]; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int ncl = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void*)dummy, &cfg);
    printf("cluster=%2d threads=%d smem=%3dKB -> maxActiveClusters=%d (%s) CTAs=%d\n", sizes[c], thr[ti], smems[si] / 1024, ncl,
           e == cudaSuccess ? "ok" : cudaGetErrorString(e), ncl * sizes[c]);
    cudaGetLastError();
  }
  // PCIe bandwidth
  size_t bytes = 1ull << 30; void *h, *d; CK(cudaMallocHost(&h, bytes)); CK(cudaMalloc(&d, bytes));
  void *h2, *d2; CK(cudaMallocHost(&h2, bytes)); CK(cudaMalloc(&d2, bytes));
  cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); printf("H2D %.1f GB/s\n", bytes / ms / 1e6);
    cudaEventRecord(e0); cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("D2H %.1f GB/s\n", bytes / ms / 1e6);
    cudaEventRecord(e0, 0);
    cudaEvent_t f; cudaEventCreate(&f); cudaEventRecord(f, 0); cudaStreamWaitEvent(s1, f); cudaStreamWaitEvent(s2, f);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s1); cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s2);
    cudaEvent_t g1, g2; cudaEventCreate(&g1); cudaEventCreate(&g2); cudaEventRecord(g1, s1); cudaEventRecord(g2, s2);
    cudaStreamWaitEvent(0, g1); cudaStreamWaitEvent(0, g2); cudaEventRecord(e1, 0); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("duplex H2D+D2H %.1f GB/s each\n", bytes / ms / 1e6);
  }
  printf("done\n");
  return 0;
}
