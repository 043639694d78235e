// cluster_probe.cu -- how many clusters of 2/4/8/16 CTAs of the fused kernel's
// footprint (544 threads, ~210 KB dynamic shared memory, 1 CTA per SM) are
// co-resident on this device: a grid-barrier kernel launched in clusters of
// size CS needs G/CS <= that number.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_probe tools/cluster_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void dummy(int *p) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0];
}

int main() {
  int optin = 0, sms = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = optin - 4096;
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  printf("sms %d optin smem %d\n", sms, optin);
  for (int cs : {1, 2, 4, 6, 8, 10, 12, 14, 16}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((sms / cs) * cs);
    cfg.blockDim = dim3(544);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
    printf("cluster %2d: max active clusters %d -> %d CTAs (%s)\n", cs, n, n * cs,
           e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  }
  return 0;
}
