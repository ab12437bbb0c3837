// Diagnostics: how many thread-block clusters of size 1/2/4/8/16 can be co-resident
// with one 384-thread CTA per SM and ~225 KB of dynamic shared memory (K4's footprint).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe_kernel(int* x) {
  extern __shared__ int s[];
  if (x) x[0] = s[0];
}

int main() {
  const int smem = 225 * 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64, 1, 1);
    cfg.blockDim = dim3(384, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe_kernel, &cfg);
    printf("cluster %2d: max active clusters %d (%d CTAs) %s\n", cs, n, n * cs,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
