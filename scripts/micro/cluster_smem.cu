// Which (dynamic smem, cluster size, grid) launches succeed on this GPU?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(320, 1) k(int* o) {
  extern __shared__ char sm[];
  sm[threadIdx.x] = 1;
  if (threadIdx.x == 0 && o) o[blockIdx.x] = sm[0];
}
int main() {
  int* o;
  cudaMalloc(&o, 4096);
  int smems[] = {150 * 1024, 190 * 1024, 200 * 1024, 210 * 1024, 216 * 1024, 220 * 1024, 222 * 1024, 226836, 227 * 1024};
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int sm : smems) {
    for (int cl : {1, 2}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(320);
      cfg.dynamicSmemBytes = sm;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cl;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = -1;
      cudaError_t oe = cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
      cudaError_t e = cudaLaunchKernelEx(&cfg, k, o);
      cudaError_t e2 = cudaDeviceSynchronize();
      printf("smem %6d cluster %d: occ %s %d launch %s sync %s\n", sm, cl, cudaGetErrorString(oe), ncl,
             cudaGetErrorString(e), cudaGetErrorString(e2));
      cudaGetLastError();
    }
  }
  return 0;
}
