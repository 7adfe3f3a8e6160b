// How many thread-block clusters of size 2 / 4 / 8 can be co-resident for a kernel shaped
// like assoc_i8_kernel (768 threads, ~217 KB dynamic shared memory, 1 CTA per SM)?
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cluster_probe tools/cluster_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe_kernel(int* x) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && x) x[blockIdx.x] = s[0];
}

int main() {
  const int smem = 216 * 1024 + 1536;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148 * 2 / cs * cs);
    cfg.blockDim = dim3(768);
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
    printf("cluster %2d: max active clusters %d -> %d CTAs (%s)\n", cs, n, n * cs, cudaGetErrorString(e));
  }
  return 0;
}
