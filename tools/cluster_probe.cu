// Largest number of co-resident thread-block clusters per cluster size (1..16) for a kernel of NT threads and SMEM
// bytes of dynamic shared memory (cudaOccupancyMaxActiveClusters): the GPC structure the term-split launches fit into.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/cluster_probe tools/cluster_probe.cu
//   tools/cluster_probe NT SMEM
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void k(double *p) {
  extern __shared__ double s[];
  if (p) p[threadIdx.x] = s[threadIdx.x];
}
int main(int argc, char **argv) {
  const int nt = argc > 1 ? atoi(argv[1]) : 256;
  const int smem = argc > 2 ? atoi(argv[2]) : 111744;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  printf("NT %d smem %d:", nt, smem);
  for (int S = 1; S <= 16; ++S) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(S);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = S;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, k, &cfg);
    printf(" %d:%d%s", S, nc, e == cudaSuccess ? "" : "(err)");
  }
  printf("\n");
  return 0;
}
