// HBM ceilings by access mix (context for the f2 scores kernel, which only writes):
// write-only with st.global.v4 (default / .cs), write-only with cp.async.bulk stores from
// shared memory (the scores kernel's store path), read-only, copy.  4 GiB, best of 10.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void wr_v4(uint4* p, size_t n) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void wr_cs(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(p + i), "r"((unsigned)i) : "memory");
}
__global__ void rd_v4(const uint4* p, size_t n, unsigned* o) {
  unsigned x = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i);
    x ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (x == 0x12345678u) o[0] = x;
}
__global__ void cp_v4(const uint4* a, uint4* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = __ldcs(a + i);
}
// bulk stores: one thread per CTA streams its contiguous slice out of a 16 KB box
template <int INFLIGHT>
__global__ void wr_bulk(char* p, size_t bytes) {
  extern __shared__ __align__(128) char sm[];
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<int*>(sm)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t boxes = bytes / 16384;
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  for (size_t b = blockIdx.x; b < boxes; b += gridDim.x) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 16384;" ::"l"(p + b * 16384), "r"(s) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(INFLIGHT) : "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class F>
static float best(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float m = 1e30f;
  for (int r = 0; r < 12; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float t; cudaEventElapsedTime(&t, a, b);
    if (r >= 2 && t < m) m = t;
  }
  return m;
}
int main() {
  const size_t bytes = 4ull << 30, n = bytes / 16;
  uint4 *a, *b; unsigned* o;
  cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMalloc(&o, 64);
  cudaMemset(a, 1, bytes);
  cudaFuncSetAttribute(wr_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  cudaFuncSetAttribute(wr_bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  auto gbs = [&](double by, float ms) { return by / (ms * 1e-3) / 1e9; };
  for (int g : {148, 296, 592, 1184}) {
    printf("{\"grid\": %d, \"wr_v4\": %.0f, \"wr_cs\": %.0f, \"rd_v4\": %.0f, \"copy_v4\": %.0f, \"wr_bulk8\": %.0f, \"wr_bulk2\": %.0f}\n", g,
           gbs(bytes, best([&] { wr_v4<<<g, 512>>>(a, n); })),
           gbs(bytes, best([&] { wr_cs<<<g, 512>>>(a, n); })),
           gbs(bytes, best([&] { rd_v4<<<g, 512>>>(a, n, o); })),
           gbs(2.0 * bytes, best([&] { cp_v4<<<g, 512>>>(a, b, n); })),
           gbs(bytes, best([&] { wr_bulk<8><<<g, 32, 16384>>>((char*)b, bytes); })),
           gbs(bytes, best([&] { wr_bulk<2><<<g, 32, 16384>>>((char*)b, bytes); })));
  }
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
