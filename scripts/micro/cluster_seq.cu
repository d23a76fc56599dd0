// Which launches fail after a cluster-2 launch?  A, A2: functions with cluster instructions
// behind a runtime flag; B: plain.
#include <cstdio>
#include <cuda_runtime.h>
__device__ void cl_body(int* o, int use) {
  if (use) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0 && o) o[blockIdx.x] = 1;
}
__global__ void A(int* o, int use) { cl_body(o, use); }
__global__ void A2(int* o, int use) { cl_body(o, use); }
__global__ void B(int* o) { if (threadIdx.x == 0 && o) o[blockIdx.x] = 2; }
static void run(const char* what, cudaError_t e) {
  cudaError_t e2 = cudaDeviceSynchronize();
  printf("%-40s launch %s / sync %s\n", what, cudaGetErrorString(e), cudaGetErrorString(e2));
  cudaGetLastError();
}
int main() {
  int* o;
  cudaMalloc(&o, 4096);
  B<<<148, 128>>>(o); run("B plain", cudaGetLastError());
  A<<<148, 128>>>(o, 0); run("A plain (no cluster, flag 0)", cudaGetLastError());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(128);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  run("A cluster 2 (flag 1)", cudaLaunchKernelEx(&cfg, A, o, 1));
  B<<<148, 128>>>(o); run("B plain after", cudaGetLastError());
  A2<<<148, 128>>>(o, 0); run("A2 plain after (never clustered)", cudaGetLastError());
  A<<<148, 128>>>(o, 0); run("A plain after", cudaGetLastError());
  run("A2 cluster 2 (flag 1)", cudaLaunchKernelEx(&cfg, A2, o, 1));
  run("A cluster 2 again", cudaLaunchKernelEx(&cfg, A, o, 1));
  return 0;
}
