// Shared GEMM epilogue (DESIGN.md §5 G1): applied per output element in fp32,
// rounded once at the store.  Used by the tcgen05 path (T = bf16) and the SIMT
// fp32 path (T = float).
#pragma once
#include <cuda_bf16.h>
#include <math_constants.h>

#include "kernels.h"

namespace ac {

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ float act_apply(int act, float v) {
  if (act == ACT_GELU) return 0.5f * v * (1.f + erff(v * 0.70710678118654752f));
  if (act == ACT_SIGMOID) return 1.f / (1.f + expf(-v));
  if (act == ACT_RELU) return fmaxf(v, 0.f);
  return v;
}

// Process 32 consecutive columns n0..n0+31 of row m (vals: fp32 accumulators).
// Columns >= N and rows >= M are not stored.
template <typename T>
__device__ __forceinline__ void epilogue_row32(const Epilogue& ep, int M, int N, int b1, int b2,
                                               int m, int n0, float (&v)[32]) {
  if (m >= M) return;
  const int64_t ob = static_cast<int64_t>(b1) * ep.out_sb1 + static_cast<int64_t>(b2) * ep.out_sb2 +
                     static_cast<int64_t>(m) * ep.out_sm;
  const bool full = (n0 + 32 <= N);
  const T* add = static_cast<const T*>(ep.add);
  const T* bias = static_cast<const T*>(ep.bias);
  const T* gate = static_cast<const T*>(ep.gate);
  const T* res = static_cast<const T*>(ep.res);
  T* out = static_cast<T*>(ep.out);
  const int64_t ab = add ? (static_cast<int64_t>(b1) * ep.add_sb1 +
                            static_cast<int64_t>(b2) * ep.add_sb2 + static_cast<int64_t>(m) * ep.add_sm)
                         : 0;
  const float bm = (bias && ep.bias_along_m) ? to_f<T>(bias[m]) : 0.f;
  const int64_t lim = static_cast<int64_t>(ep.row_off) + m - ep.col_off;  // causal: n > lim masked
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int n = n0 + j;
    if (!full && n >= N) break;
    float x = v[j] * ep.scale;
    if (add) x += to_f<T>(add[ab + static_cast<int64_t>(n) * ep.add_sn]);
    if (bias) x += ep.bias_along_m ? bm : to_f<T>(bias[n]);
    x = act_apply(ep.act, x);
    const int64_t o = ob + static_cast<int64_t>(n) * ep.out_sn;
    if (gate) x *= to_f<T>(gate[o]);
    if (res) x += to_f<T>(res[o]);
    if (ep.causal && n > lim) x = -CUDART_INF_F;
    v[j] = x;
  }
  if (full && ep.out_sn == 1 && sizeof(T) == 2 && ((ob + n0) % 8) == 0) {
    uint4* dst = reinterpret_cast<uint4*>(out + ob + n0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[q * 8 + 2 * e], v[q * 8 + 2 * e + 1]);
        w[e] = *reinterpret_cast<uint32_t*>(&h);
      }
      dst[q] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = n0 + j;
      if (!full && n >= N) break;
      out[ob + static_cast<int64_t>(n) * ep.out_sn] = from_f<T>(v[j]);
    }
  }
}

}  // namespace ac
