// MUFU ex2 throughput microbenchmark: f32, f16x2, bf16x2 (results per SM per clock)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

template <int V>
__global__ void k(float* out, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  uint32_t h0 = 0x3c003c00u ^ threadIdx.x, h1 = h0 + 1, h2 = h0 + 2, h3 = h0 + 3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (V == 0) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a1));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a3));
    } else if (V == 1) {
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h0)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h1));
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h2)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h3));
    } else {
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h0)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h1));
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h2)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h3));
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
  out[1 + blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + (float)(h0 ^ h1 ^ h2 ^ h3);
}

int main() {
  float* d;
  cudaMalloc(&d, 4 * (1 + 148 * 1024 * 4));
  const int iters = 4096;
  const char* names[3] = {"ex2.f32", "ex2.f16x2 (2 results)", "ex2.bf16x2 (2 results)"};
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      float clk;
      if (v == 0) k<0><<<148, 1024>>>(d, iters);
      if (v == 1) k<1><<<148, 1024>>>(d, iters);
      if (v == 2) k<2><<<148, 1024>>>(d, iters);
      cudaDeviceSynchronize();
      cudaMemcpy(&clk, d, 4, cudaMemcpyDeviceToHost);
      const double instrs = 1024.0 * iters * 4;  // per SM (one block per SM)
      if (rep) printf("%-24s %.2f instr/clk/SM\n", names[v], instrs / clk);
    }
  }
  return 0;
}
