// Largest thread-block cluster the device co-schedules for a 1024- and a
// 512-thread kernel (diagnostic for the one-cluster solver path).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k1024() {}
__global__ void k512() {}
template <typename K>
int probe(K k, int threads) {
  cudaFuncSetAttribute((const void*)k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16);
  cfg.blockDim = dim3(threads);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 16;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = -1;
  cudaError_t e = cudaOccupancyMaxPotentialClusterSize(&n, (const void*)k, &cfg);
  int nc = -1;
  cudaOccupancyMaxActiveClusters(&nc, (const void*)k, &cfg);
  printf("threads %d: max cluster %d (%s), active 16-clusters %d\n", threads, n, cudaGetErrorString(e), nc);
  return n;
}
int main() {
  probe(k1024, 1024);
  probe(k512, 512);
  return 0;
}
