// How many clusters of a given size can be co-resident on this B200 for a
// 128-thread kernel with the given dynamic smem (cudaOccupancyMaxActiveClusters).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 cluster_occupancy.cu -o cluster_occupancy
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(int* p) {
  extern __shared__ int s[];
  if (p) p[0] = s[0];
}

int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int smems[] = {48, 84, 120, 180, 200};
  for (int sm : smems)
    for (int c = 1; c <= 16; ++c) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c * 64);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = sm * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("smem %3d KB cluster %2d: max active clusters %3d (%3d CTAs) %s\n", sm, c, n, n * c,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  return 0;
}
