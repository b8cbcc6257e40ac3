#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* o) { extern __shared__ int s[]; if (threadIdx.x == 0) o[blockIdx.x] = s[0]; }
int main() {
  int* o; cudaMalloc(&o, 4096 * 4);
  for (int smem : {200 * 1024, 100 * 1024}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 64); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int n = 0; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("smem %dKB cluster %2d: max active clusters %d -> %d CTAs (%s)\n", smem / 1024, cs, n, n * cs, cudaGetErrorString(e));
    }
  }
  return 0;
}
