// Probe: how many clusters of a given shape can be co-resident with one 200 KB CTA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/cluster_occupancy tools/cluster_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k() { extern __shared__ char s[]; s[threadIdx.x] = 0; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int dims[][3] = {{1, 1, 2}, {1, 1, 4}, {1, 1, 8}, {1, 2, 8}, {1, 4, 4}, {1, 16, 1}, {1, 1, 16}, {1, 4, 1}};
  for (auto& d : dims) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(d[0], d[1], d[2]);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = d[0];
    at[0].val.clusterDim.y = d[1];
    at[0].val.clusterDim.z = d[2];
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int m = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&m, (void*)k, &cfg);
    printf("cluster (%d,%d,%d): max active %d (%s)\n", d[0], d[1], d[2], m, cudaGetErrorString(e));
  }
}
