// How many thread-block clusters of size C fit on this B200 when each CTA needs one SM
// (~226 KB dynamic shared memory): the feasibility of TMA multicast staging for k_sweep2.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_clusters tools/probe_clusters.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dummy(float* p) {
  extern __shared__ float s[];
  s[threadIdx.x] = 0.f;
  if (p) p[0] = s[0];
}
int main() {
  const int smem = 226 * 1024;
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int c : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148 / c * c);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
    printf("cluster %2d: max active clusters %d (CTAs %d) %s\n", c, n, n * c, cudaGetErrorString(e));
  }
  return 0;
}
