// G3 row softmax and G5 LayerNorm (HBM-bound row kernels, sm_100a).
//
// Both keep a whole row in registers (16-byte vector loads/stores, coalesced
// across the warp), reduce with warp shuffles (+ shared memory across warps),
// and touch HBM exactly once per element in each direction.  Statistics are
// fp32.  softmax: m = max_j s_j, l = sum_j exp(s_j - m), p_j = exp(s_j - m) / l
// (stable form).  LayerNorm: biased variance, eps inside the
// square root.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "kernels.h"

namespace ac {
namespace {

template <typename T>
struct Vec;  // 16-byte vector of T
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  uint4 raw;
  __device__ __forceinline__ void to_float(float (&f)[8]) const {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 t = __bfloat1622float2(h[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
  __device__ __forceinline__ void from_float(const float (&f)[8]) {
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  }
};
template <>
struct Vec<float> {
  static constexpr int N = 4;
  uint4 raw;
  __device__ __forceinline__ void to_float(float (&f)[4]) const {
    f[0] = __uint_as_float(raw.x); f[1] = __uint_as_float(raw.y);
    f[2] = __uint_as_float(raw.z); f[3] = __uint_as_float(raw.w);
  }
  __device__ __forceinline__ void from_float(const float (&f)[4]) {
    raw = make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
  }
};

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ softmax
// THREADS threads per row (32 or 256), VPT 16-byte vectors per thread.
template <typename T, int THREADS, int VPT>
__global__ void __launch_bounds__(256) softmax_kernel(const T* __restrict__ s, T* __restrict__ p, int64_t rows,
                                                      int64_t ncols, int64_t ld, int causal, int64_t row_off) {
  constexpr int VN = Vec<T>::N;
  constexpr int RPB = 256 / THREADS;
  __shared__ float red[2][8][RPB > 0 ? RPB : 1];
  const int sub = threadIdx.x / THREADS;       // row within block
  const int tid = threadIdx.x % THREADS;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * RPB + sub;
  const bool live = r < rows;
  const T* srow = s + r * ld;
  T* prow = p + r * ld;
  int64_t valid = ncols, wend = ncols;
  if (causal) {
    const int64_t R = row_off + r;
    valid = R + 1 < ncols ? R + 1 : ncols;
    const int64_t k = ((R >> 7) + 1) << 7;
    wend = k < ncols ? k : ncols;
  }
  Vec<T> v[VPT];
  float mx = -CUDART_INF_F;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int64_t c = (static_cast<int64_t>(i) * THREADS + tid) * VN;
    if (live && c < valid) {
      v[i].raw = *reinterpret_cast<const uint4*>(srow + c);
      float f[VN];
      v[i].to_float(f);
#pragma unroll
      for (int e = 0; e < VN; ++e)
        if (c + e < valid) mx = fmaxf(mx, f[e]);
    }
  }
  mx = warp_max(mx);
  if (THREADS > 32) {
    const int w = tid >> 5;
    if ((tid & 31) == 0) red[0][w][sub] = mx;
    __syncthreads();
    mx = red[0][0][sub];
#pragma unroll
    for (int i = 1; i < THREADS / 32; ++i) mx = fmaxf(mx, red[0][i][sub]);
  }
  constexpr float L2E = 1.4426950408889634f;
  const float mxl = mx * L2E;
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int64_t c = (static_cast<int64_t>(i) * THREADS + tid) * VN;
    if (live && c < valid) {
      float f[VN];
      v[i].to_float(f);
#pragma unroll
      for (int e = 0; e < VN; ++e)
        if (c + e < valid) sum += exp2f(fmaf(f[e], L2E, -mxl));
    }
  }
  sum = warp_sum(sum);
  if (THREADS > 32) {
    const int w = tid >> 5;
    if ((tid & 31) == 0) red[1][w][sub] = sum;
    __syncthreads();
    sum = 0.f;
#pragma unroll
    for (int i = 0; i < THREADS / 32; ++i) sum += red[1][i][sub];
  }
  const float inv = 1.f / sum;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int64_t c = (static_cast<int64_t>(i) * THREADS + tid) * VN;
    if (live && c < wend) {
      float f[VN];
      v[i].to_float(f);
#pragma unroll
      for (int e = 0; e < VN; ++e) f[e] = (c + e < valid) ? exp2f(fmaf(f[e], L2E, -mxl)) * inv : 0.f;
      Vec<T> o;
      o.from_float(f);
      *reinterpret_cast<uint4*>(prow + c) = o.raw;
    }
  }
}

template <typename T, int THREADS, int VPT>
cudaError_t launch_softmax(const void* s, void* p, int64_t rows, int64_t ncols, int64_t ld, int causal,
                           int64_t row_off, cudaStream_t st) {
  constexpr int RPB = 256 / THREADS;
  const int64_t blocks = (rows + RPB - 1) / RPB;
  if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
  softmax_kernel<T, THREADS, VPT><<<static_cast<unsigned>(blocks), 256, 0, st>>>(
      static_cast<const T*>(s), static_cast<T*>(p), rows, ncols, ld, causal, row_off);
  return cudaGetLastError();
}

template <typename T>
cudaError_t softmax_dispatch(const void* s, void* p, int64_t rows, int64_t ncols, int64_t ld, int causal,
                             int64_t row_off, cudaStream_t st) {
  constexpr int VN = Vec<T>::N;
  const int64_t vecs = (ncols + VN - 1) / VN;
  if (vecs <= 32 * 1) return launch_softmax<T, 32, 1>(s, p, rows, ncols, ld, causal, row_off, st);
  if (vecs <= 32 * 2) return launch_softmax<T, 32, 2>(s, p, rows, ncols, ld, causal, row_off, st);
  if (vecs <= 32 * 4) return launch_softmax<T, 32, 4>(s, p, rows, ncols, ld, causal, row_off, st);
  if (vecs <= 32 * 8) return launch_softmax<T, 32, 8>(s, p, rows, ncols, ld, causal, row_off, st);
  if (vecs <= 256 * 2) return launch_softmax<T, 256, 2>(s, p, rows, ncols, ld, causal, row_off, st);
  if (vecs <= 256 * 4) return launch_softmax<T, 256, 4>(s, p, rows, ncols, ld, causal, row_off, st);
  if (vecs <= 256 * 8) return launch_softmax<T, 256, 8>(s, p, rows, ncols, ld, causal, row_off, st);
  if (vecs <= 256 * 16) return launch_softmax<T, 256, 16>(s, p, rows, ncols, ld, causal, row_off, st);
  if (vecs <= 256 * 32) return launch_softmax<T, 256, 32>(s, p, rows, ncols, ld, causal, row_off, st);
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------ layernorm
// one warp per row, VPT 16-byte vectors per lane
template <typename T, int VPT>
__global__ void __launch_bounds__(256) layernorm_kernel(const T* __restrict__ x, const T* __restrict__ g,
                                                        const T* __restrict__ b, T* __restrict__ y, int64_t rows,
                                                        int C, float eps) {
  constexpr int VN = Vec<T>::N;
  const int lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const T* xr = x + r * C;
  T* yr = y + r * C;
  const int nv = C / VN;
  float f[VPT][VN];
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int vi = i * 32 + lane;
    if (vi < nv) {
      Vec<T> v;
      v.raw = *reinterpret_cast<const uint4*>(xr + vi * VN);
      v.to_float(f[i]);
#pragma unroll
      for (int e = 0; e < VN; ++e) sum += f[i][e];
    }
  }
  const float mean = warp_sum(sum) / static_cast<float>(C);
  float sq = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int vi = i * 32 + lane;
    if (vi < nv) {
#pragma unroll
      for (int e = 0; e < VN; ++e) {
        const float d = f[i][e] - mean;
        sq += d * d;
      }
    }
  }
  const float var = warp_sum(sq) / static_cast<float>(C);
  const float inv = 1.f / sqrtf(var + eps);
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int vi = i * 32 + lane;
    if (vi < nv) {
      Vec<T> gv, bv, o;
      gv.raw = *reinterpret_cast<const uint4*>(g + vi * VN);
      bv.raw = *reinterpret_cast<const uint4*>(b + vi * VN);
      float gf[VN], bf[VN], of[VN];
      gv.to_float(gf);
      bv.to_float(bf);
#pragma unroll
      for (int e = 0; e < VN; ++e) of[e] = (f[i][e] - mean) * inv * gf[e] + bf[e];
      o.from_float(of);
      *reinterpret_cast<uint4*>(yr + vi * VN) = o.raw;
    }
  }
}

template <typename T>
cudaError_t layernorm_dispatch(const void* x, const void* g, const void* b, void* y, int64_t rows, int C,
                               float eps, cudaStream_t st) {
  constexpr int VN = Vec<T>::N;
  if (C % VN != 0) return cudaErrorInvalidValue;
  const int nv = C / VN;
  const int64_t blocks = (rows + 7) / 8;
  if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
  const unsigned gb = static_cast<unsigned>(blocks);
  auto X = static_cast<const T*>(x);
  auto G = static_cast<const T*>(g);
  auto B = static_cast<const T*>(b);
  auto Y = static_cast<T*>(y);
  if (nv <= 32) layernorm_kernel<T, 1><<<gb, 256, 0, st>>>(X, G, B, Y, rows, C, eps);
  else if (nv <= 64) layernorm_kernel<T, 2><<<gb, 256, 0, st>>>(X, G, B, Y, rows, C, eps);
  else if (nv <= 128) layernorm_kernel<T, 4><<<gb, 256, 0, st>>>(X, G, B, Y, rows, C, eps);
  else if (nv <= 256) layernorm_kernel<T, 8><<<gb, 256, 0, st>>>(X, G, B, Y, rows, C, eps);
  else if (nv <= 512) layernorm_kernel<T, 16><<<gb, 256, 0, st>>>(X, G, B, Y, rows, C, eps);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace

cudaError_t softmax_rows(const void* s_in, void* p_out, int64_t rows, int64_t ncols, int64_t ld, int causal,
                         int64_t row_off, int dtype, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  if (dtype == 1) {
    if (ld % 8 || ncols % 8) return cudaErrorInvalidValue;
    return softmax_dispatch<__nv_bfloat16>(s_in, p_out, rows, ncols, ld, causal, row_off, st);
  }
  if (ld % 4 || ncols % 4) return cudaErrorInvalidValue;
  return softmax_dispatch<float>(s_in, p_out, rows, ncols, ld, causal, row_off, st);
}

cudaError_t layernorm(const void* x, const void* gamma, const void* beta, void* y, int64_t rows, int C, float eps,
                      int dtype, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  if (dtype == 1) return layernorm_dispatch<__nv_bfloat16>(x, gamma, beta, y, rows, C, eps, st);
  return layernorm_dispatch<float>(x, gamma, beta, y, rows, C, eps, st);
}

}  // namespace ac
