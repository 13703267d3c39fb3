// How many 2-, 4- and 8-CTA clusters of an attention-sized CTA (384 threads,
// ~231 KB dynamic shared memory, 1 CTA per SM) can be co-resident on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(384, 1) dummy(int* p) { if (p) p[threadIdx.x] = 0; }
int main() {
  const int smem = 231040;
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs * (sms / cs)); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
    printf("cluster %2d: max active clusters %d -> %d SMs of %d (%s)\n", cs, n, n * cs, sms, cudaGetErrorString(e));
  }
  return 0;
}
