// How many thread-block clusters of each size fit on this GPU at one CTA per SM (K1 design input).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void kern(int *p) { if (p) p[0] = 1; }
int main(int argc, char **argv) {
  const int smem = (argc > 1 ? atoi(argv[1]) : 200) * 1024;
  const int threads = argc > 2 ? atoi(argv[2]) : 640;
  printf("smem %d KB, %d threads\n", smem / 1024, threads);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
    printf("cluster %2d: max active clusters %d (%d SMs) %s\n", cs, n, n * cs, cudaGetErrorString(e));
  }
  return 0;
}
