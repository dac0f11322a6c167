// How many clusters of size CS, each CTA with `smem` bytes of dynamic shared memory (1 CTA per
// SM), can be co-resident on this GPU (cudaOccupancyMaxActiveClusters)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 cluster_occ.cu -o cluster_occ
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { if (p) p[blockIdx.x] = 1; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int smem : {100 * 1024, 150 * 1024, 184 * 1024, 220 * 1024})
    for (int cs : {1, 2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 16);
      cfg.blockDim = dim3(320);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("{\"smem_kb\": %d, \"cluster\": %d, \"max_active_clusters\": %d, \"ctas\": %d, \"status\": \"%s\"}\n",
             smem / 1024, cs, n, n * cs, cudaGetErrorString(e));
    }
  return 0;
}
