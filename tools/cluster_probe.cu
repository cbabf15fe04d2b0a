// cluster_probe.cu — max active clusters vs cluster size at 1 CTA/SM (dev tool).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dummy(double* p) { extern __shared__ double s[]; if (p) { s[threadIdx.x] = 1; p[threadIdx.x] = s[threadIdx.x ^ 1]; } }
int main() {
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int smem : {140 * 1024, 100 * 1024}) {
    for (int c = 1; c <= 16; ++c) {
      cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute at[1];
      cfg.gridDim = dim3(c * 32); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem;
      at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = c; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int ncl = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void*)dummy, &cfg);
      printf("smem=%3dKB cluster=%2d -> clusters=%3d CTAs=%3d %s\n", smem / 1024, c, ncl, ncl * c, e ? cudaGetErrorString(e) : "");
      cudaGetLastError();
    }
  }
  return 0;
}
