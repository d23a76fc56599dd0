// Does tcgen05.alloc.cta_group::2 work with a cluster of 2 given at launch time vs at compile time?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ void body(int* o, int variant) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    if (variant == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&holder)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&holder)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  if (threadIdx.x == 0) o[blockIdx.x] = holder * 10 + r;
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    if (variant == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(holder) : "memory");
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(holder) : "memory");
  }
}
__global__ void __launch_bounds__(128, 1) k_dyn(int* o, int v) { body(o, v); }
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_static(int* o, int v) { body(o, v); }
int main() {
  int* o;
  cudaMalloc(&o, 4096);
  for (int v : {1, 2, 1, 2}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(128);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_dyn, o, v);
    cudaError_t e2 = cudaDeviceSynchronize();
    printf("dyn cluster, cta_group::%d: launch %s sync %s\n", v, cudaGetErrorString(e), cudaGetErrorString(e2));
    cudaGetLastError();
    at[0].val.clusterDim.x = 1;
    e = cudaLaunchKernelEx(&cfg, k_dyn, o, 1);
    e2 = cudaDeviceSynchronize();
    printf("  then cluster dim 1, cta_group::1: launch %s sync %s\n", cudaGetErrorString(e), cudaGetErrorString(e2));
    cudaGetLastError();
    cfg.numAttrs = 0;
    e = cudaLaunchKernelEx(&cfg, k_dyn, o, 1);
    e2 = cudaDeviceSynchronize();
    printf("  then no attribute, cta_group::1: launch %s sync %s\n", cudaGetErrorString(e), cudaGetErrorString(e2));
    cudaGetLastError();
  }
  return 0;
}
