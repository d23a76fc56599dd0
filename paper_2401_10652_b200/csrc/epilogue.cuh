// Shared GEMM epilogue (DESIGN.md §5 G1): applied per output element in fp32,
// rounded once at the store.  Used by the tcgen05 path (T = bf16); the SIMT
// fp32 path applies the same order inline.
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

#ifndef SIGMOID_TANH
#define SIGMOID_TANH 1
#endif

// Branch-free erf for the GELU epilogue, Abramowitz & Stegun 7.1.26:
// erf(a) = 1 - t (a1 + t (a2 + t (a3 + t (a4 + t a5)))) exp(-a^2), t = 1 / (1 + p a),
// a = |z| (absolute error < 1.5e-7, below the fp32 / bf16 rounding of the GELU
// output; rcp.approx adds < 2 ulp).  One MUFU reciprocal + one MUFU exp and five
// FMAs, no branches (CUDA's erff has a data-dependent branch that serialises the
// epilogue).
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Sigmoid of a value stored in bf16: 0.5 + 0.5 tanh(x / 2) with MUFU tanh.approx (one MUFU
// op; |error| <= 2.5e-4 absolute, below the bf16 half-ulp of every sigmoid value >= 0.125)
// instead of ex2 + rcp, two dependent MUFU ops (reading R28).  fp32 outputs keep the
// precise form (their tolerance is 1e-4).
__device__ __forceinline__ float sigmoid_bf16(float x) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * x));
  return fmaf(0.5f, t, 0.5f);
}

__device__ __forceinline__ float erf_fast(float z) {
  const float a = fabsf(z);
  const float t = rcp_approx(fmaf(0.3275911f, a, 1.f));  // MUFU.RCP (the IEEE __frcp_rn is a slow sequence)
  float p = fmaf(t, 1.061405429f, -1.453152027f);
  p = fmaf(t, p, 1.421413741f);
  p = fmaf(t, p, -0.284496736f);
  p = fmaf(t, p, 0.254829592f);
  const float erfc = t * p * __expf(-a * a);
  return copysignf(1.f - erfc, z);
}

// packed fp32 pairs (FFMA2 / FMUL2: two lanes per instruction, each rounded as the
// scalar op) for the element-wise epilogue math
__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_splat(float v) { return f2_pack(v, v); }
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// x[j] = x[j] * s, x[j] = x[j] + y[j], x[j] = x[j] * y[j] over even-length arrays, two
// lanes per instruction (bitwise the scalar results)
template <int NE>
__device__ __forceinline__ void arr_scale(float (&x)[NE], float sc) {
  const uint64_t s2 = f2_splat(sc);
#pragma unroll
  for (int j = 0; j < NE; j += 2) f2_unpack(f2_mul(f2_pack(x[j], x[j + 1]), s2), x[j], x[j + 1]);
}
template <int NE>
__device__ __forceinline__ void arr_add(float (&x)[NE], const float (&y)[NE]) {
#pragma unroll
  for (int j = 0; j < NE; j += 2) f2_unpack(f2_add(f2_pack(x[j], x[j + 1]), f2_pack(y[j], y[j + 1])), x[j], x[j + 1]);
}
template <int NE>
__device__ __forceinline__ void arr_mul(float (&x)[NE], const float (&y)[NE]) {
#pragma unroll
  for (int j = 0; j < NE; j += 2) f2_unpack(f2_mul(f2_pack(x[j], x[j + 1]), f2_pack(y[j], y[j + 1])), x[j], x[j + 1]);
}

// GELU of a pair with erf_fast's arithmetic on packed pairs (the two reciprocals and
// exponentials stay scalar MUFU ops): half the FMA-pipe instructions of two gelu calls
__device__ __forceinline__ void gelu_pair(float& x0, float& x1) {
  const uint64_t x = f2_pack(x0, x1);
  const uint64_t z = f2_mul(x, f2_splat(0.70710678118654752f));
  float z0, z1;
  f2_unpack(z, z0, z1);
  const uint64_t av = f2_pack(fabsf(z0), fabsf(z1));
  float d0, d1;
  f2_unpack(f2_fma(f2_splat(0.3275911f), av, f2_splat(1.f)), d0, d1);
  const uint64_t t = f2_pack(rcp_approx(d0), rcp_approx(d1));
  uint64_t p = f2_fma(t, f2_splat(1.061405429f), f2_splat(-1.453152027f));
  p = f2_fma(t, p, f2_splat(1.421413741f));
  p = f2_fma(t, p, f2_splat(-0.284496736f));
  p = f2_fma(t, p, f2_splat(0.254829592f));
  float q0, q1;
  f2_unpack(f2_mul(f2_mul(av, av), f2_splat(-1.4426950408889634f)), q0, q1);
  float ex0, ex1;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ex0) : "f"(q0));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ex1) : "f"(q1));
  float e0, e1;
  f2_unpack(f2_mul(f2_mul(t, p), f2_pack(ex0, ex1)), e0, e1);
  const uint64_t erf = f2_pack(copysignf(1.f - e0, z0), copysignf(1.f - e1, z1));
  const uint64_t h = f2_mul(x, f2_splat(0.5f));
  f2_unpack(f2_fma(h, erf, h), x0, x1);  // 0.5 x (1 + erf)
}

// Activation over an array with the kind test hoisted out of the element loop: a
// per-element branch puts every element in its own reconvergence region and
// serialises the otherwise independent erf chains (measured 2x on FFN1).
template <int NE>
__device__ __forceinline__ void act_array(int act, float (&x)[NE]) {
  if (act == ACT_GELU) {
    if constexpr (NE % 2 == 0) {
#pragma unroll
      for (int j = 0; j < NE; j += 2) gelu_pair(x[j], x[j + 1]);
    } else {
#pragma unroll
      for (int j = 0; j < NE; ++j) x[j] = 0.5f * x[j] * (1.f + erf_fast(x[j] * 0.70710678118654752f));
    }
  } else if (act == ACT_SIGMOID) {
#pragma unroll
    for (int j = 0; j < NE; ++j) x[j] = SIGMOID_TANH ? sigmoid_bf16(x[j]) : rcp_approx(1.f + __expf(-x[j]));
  } else if (act == ACT_RELU) {
#pragma unroll
    for (int j = 0; j < NE; ++j) x[j] = fmaxf(x[j], 0.f);
  }
}

template <typename T = float>
__device__ __forceinline__ float act_apply(int act, float v) {
  if (act == ACT_GELU) return 0.5f * v * (1.f + erf_fast(v * 0.70710678118654752f));
  if (act == ACT_SIGMOID)
    return (SIGMOID_TANH && sizeof(T) == 2) ? sigmoid_bf16(v) : rcp_approx(1.f + __expf(-v));
  if (act == ACT_RELU) return fmaxf(v, 0.f);
  return v;
}

// v = acc*scale (+add) (+bias) -> act (*gate) (+res), causal -> -inf.  o = output offset.
template <typename T>
__device__ __forceinline__ float epi_value(const Epilogue& ep, int b1, int b2, int m, int n, float acc, int64_t o) {
  float x = acc * ep.scale;
  if (ep.add)
    x += to_f<T>(static_cast<const T*>(ep.add)[static_cast<int64_t>(b1) * ep.add_sb1 +
                                               static_cast<int64_t>(b2) * ep.add_sb2 +
                                               static_cast<int64_t>(m) * ep.add_sm + static_cast<int64_t>(n) * ep.add_sn]);
  if (ep.bias) x += to_f<T>(static_cast<const T*>(ep.bias)[ep.bias_along_m ? m : n]);
  x = act_apply<T>(ep.act, x);
  (void)o;
  if (ep.gate)
    x *= to_f<T>(static_cast<const T*>(ep.gate)[static_cast<int64_t>(b1) * ep.gate_sb1 +
                                                static_cast<int64_t>(b2) * ep.gate_sb2 +
                                                static_cast<int64_t>(m) * ep.gate_sm +
                                                static_cast<int64_t>(n) * ep.gate_sn]);
  if (ep.res)
    x += to_f<T>(static_cast<const T*>(ep.res)[static_cast<int64_t>(b1) * ep.res_sb1 +
                                               static_cast<int64_t>(b2) * ep.res_sb2 +
                                               static_cast<int64_t>(m) * ep.res_sm + static_cast<int64_t>(n) * ep.res_sn]);
  if (ep.causal && static_cast<int64_t>(n) + ep.col_off > ep.row_off + m) x = -CUDART_INF_F;
  return x;
}

// Two adjacent columns n, n+1 of row m (a lane's share of a coalesced row segment).
template <typename T>
__device__ __forceinline__ void epilogue_pair(const Epilogue& ep, int N, int b1, int b2, int m, int n, float a0,
                                              float a1) {
  if (n >= N) return;
  const int64_t o = static_cast<int64_t>(b1) * ep.out_sb1 + static_cast<int64_t>(b2) * ep.out_sb2 +
                    static_cast<int64_t>(m) * ep.out_sm + static_cast<int64_t>(n) * ep.out_sn;
  T* out = static_cast<T*>(ep.out);
  const float x0 = epi_value<T>(ep, b1, b2, m, n, a0, o);
  if (n + 1 >= N) {
    out[o] = from_f<T>(x0);
    return;
  }
  const float x1 = epi_value<T>(ep, b1, b2, m, n + 1, a1, o + ep.out_sn);
  if constexpr (sizeof(T) == 2) {
    if (ep.out_sn == 1 && (o & 1) == 0) {
      *reinterpret_cast<__nv_bfloat162*>(out + o) = __floats2bfloat162_rn(x0, x1);
      return;
    }
  }
  out[o] = from_f<T>(x0);
  out[o + ep.out_sn] = from_f<T>(x1);
}

__device__ __forceinline__ void bf16x8_to_f(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

// Eight consecutive columns n..n+7 of row m, bf16, all aux tensors n-contiguous
// and 16-byte aligned (checked on the host): one 16-byte load per aux tensor and
// one 16-byte store.  Same operation order as epi_value.
__device__ __forceinline__ void epilogue8(const Epilogue& ep, int b1, int b2, int m, int n, float (&x)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] *= ep.scale;
  float a[8];
  if (ep.add) {
    const int64_t o = static_cast<int64_t>(b1) * ep.add_sb1 + static_cast<int64_t>(b2) * ep.add_sb2 +
                      static_cast<int64_t>(m) * ep.add_sm + n;
    bf16x8_to_f(*reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(ep.add) + o), a);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] += a[i];
  }
  if (ep.bias) {
    const __nv_bfloat16* b = static_cast<const __nv_bfloat16*>(ep.bias);
    if (ep.bias_along_m) {
      const float bm = __bfloat162float(b[m]);
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] += bm;
    } else {
      bf16x8_to_f(*reinterpret_cast<const uint4*>(b + n), a);
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] += a[i];
    }
  }
  act_array(ep.act, x);
  if (ep.gate) {
    const int64_t o = static_cast<int64_t>(b1) * ep.gate_sb1 + static_cast<int64_t>(b2) * ep.gate_sb2 +
                      static_cast<int64_t>(m) * ep.gate_sm + n;
    bf16x8_to_f(*reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(ep.gate) + o), a);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] *= a[i];
  }
  if (ep.res) {
    const int64_t o = static_cast<int64_t>(b1) * ep.res_sb1 + static_cast<int64_t>(b2) * ep.res_sb2 +
                      static_cast<int64_t>(m) * ep.res_sm + n;
    bf16x8_to_f(*reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(ep.res) + o), a);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] += a[i];
  }
  if (ep.causal) {
    const int64_t lim = ep.row_off + m - ep.col_off - n;  // column n+i masked when i > lim
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i > lim) x[i] = -CUDART_INF_F;
  }
  uint4 w;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(x[2 * i], x[2 * i + 1]);
  const int64_t o = static_cast<int64_t>(b1) * ep.out_sb1 + static_cast<int64_t>(b2) * ep.out_sb2 +
                    static_cast<int64_t>(m) * ep.out_sm + n;
  *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.out) + o) = w;
}

// Operands of epilogue8p loaded ahead of time (several rows in flight).
struct Aux8 {
  uint4 add, gate, res;
  float bias_m;
};

__device__ __forceinline__ void load_aux8(const Epilogue& ep, int b1, int b2, int m, int n, Aux8& x) {
  if (ep.add)
    x.add = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(ep.add) + static_cast<int64_t>(b1) * ep.add_sb1 +
                                            static_cast<int64_t>(b2) * ep.add_sb2 + static_cast<int64_t>(m) * ep.add_sm + n);
  if (ep.gate)
    x.gate = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(ep.gate) +
                                             static_cast<int64_t>(b1) * ep.gate_sb1 + static_cast<int64_t>(b2) * ep.gate_sb2 +
                                             static_cast<int64_t>(m) * ep.gate_sm + n);
  if (ep.res)
    x.res = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(ep.res) + static_cast<int64_t>(b1) * ep.res_sb1 +
                                            static_cast<int64_t>(b2) * ep.res_sb2 + static_cast<int64_t>(m) * ep.res_sm + n);
  if (ep.bias && ep.bias_along_m) x.bias_m = __bfloat162float(static_cast<const __nv_bfloat16*>(ep.bias)[m]);
}

// epilogue8 with the aux operands preloaded; bias_n = the column bias of this
// lane's 8 columns (loaded once per slab).  Same operation order as epi_value.
__device__ __forceinline__ void epilogue8p(const Epilogue& ep, int b1, int b2, int m, int n, float (&x)[8],
                                           const Aux8& aux, const float (&bias_n)[8]) {
  float a[8];
  arr_scale(x, ep.scale);
  if (ep.add) {
    bf16x8_to_f(aux.add, a);
    arr_add(x, a);
  }
  if (ep.bias) {
    if (ep.bias_along_m) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = aux.bias_m;
      arr_add(x, a);
    } else {
      arr_add(x, bias_n);
    }
  }
  act_array(ep.act, x);
  if (ep.gate) {
    bf16x8_to_f(aux.gate, a);
    arr_mul(x, a);
  }
  if (ep.res) {
    bf16x8_to_f(aux.res, a);
    arr_add(x, a);
  }
  if (ep.causal) {
    const int64_t lim = ep.row_off + m - ep.col_off - n;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i > lim) x[i] = -CUDART_INF_F;
  }
  uint4 w;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(x[2 * i], x[2 * i + 1]);
  const int64_t o = static_cast<int64_t>(b1) * ep.out_sb1 + static_cast<int64_t>(b2) * ep.out_sb2 +
                    static_cast<int64_t>(m) * ep.out_sm + n;
  *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.out) + o) = w;
}

// 32 consecutive bf16 -> fp32; only the 8-element groups below `nvalid` are
// read (columns past N are never touched; the vec path guarantees N % 8 == 0)
__device__ __forceinline__ void load32_bf16(const __nv_bfloat16* p, float (&f)[32], int nvalid = 32) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  uint4 u[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) u[i] = 8 * i < nvalid ? q[i] : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float g[8];
    bf16x8_to_f(u[i], g);
#pragma unroll
    for (int e = 0; e < 8; ++e) f[8 * i + e] = g[e];
  }
}

// Thread-per-row epilogue of 32 consecutive accumulator columns n..n+31 of row m
// (all aux tensors n-contiguous and 16-byte aligned, checked on the host); the
// result is packed to 16 bf16x2 words.  Same operation order as epi_value.
__device__ __forceinline__ void epilogue_row32(const Epilogue& ep, int b1, int b2, int m, int n, bool mvalid,
                                               const uint32_t (&r)[32], uint32_t (&pk)[16], int nvalid) {
  float x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = __uint_as_float(r[j]);
  arr_scale(x, ep.scale);
  float a[32];
  if (ep.add && mvalid) {
    load32_bf16(static_cast<const __nv_bfloat16*>(ep.add) + static_cast<int64_t>(b1) * ep.add_sb1 +
                    static_cast<int64_t>(b2) * ep.add_sb2 + static_cast<int64_t>(m) * ep.add_sm + n,
                a, nvalid);
    arr_add(x, a);
  }
  if (ep.bias) {
    if (ep.bias_along_m) {
      const float bm = mvalid ? __bfloat162float(static_cast<const __nv_bfloat16*>(ep.bias)[m]) : 0.f;
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] += bm;
    } else {
      load32_bf16(static_cast<const __nv_bfloat16*>(ep.bias) + n, a, nvalid);
      arr_add(x, a);
    }
  }
  act_array(ep.act, x);
  if (ep.gate && mvalid) {
    load32_bf16(static_cast<const __nv_bfloat16*>(ep.gate) + static_cast<int64_t>(b1) * ep.gate_sb1 +
                    static_cast<int64_t>(b2) * ep.gate_sb2 + static_cast<int64_t>(m) * ep.gate_sm + n,
                a, nvalid);
    arr_mul(x, a);
  }
  if (ep.res && mvalid) {
    load32_bf16(static_cast<const __nv_bfloat16*>(ep.res) + static_cast<int64_t>(b1) * ep.res_sb1 +
                    static_cast<int64_t>(b2) * ep.res_sb2 + static_cast<int64_t>(m) * ep.res_sm + n,
                a, nvalid);
    arr_add(x, a);
  }
  if (ep.causal) {
    const int64_t lim = ep.row_off + m - ep.col_off - n;  // column n+j masked when j > lim
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j > lim) x[j] = -CUDART_INF_F;
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    __nv_bfloat162 h = __floats2bfloat162_rn(x[2 * j], x[2 * j + 1]);
    pk[j] = *reinterpret_cast<uint32_t*>(&h);
  }
}

template <typename T>
__device__ __forceinline__ void epilogue_one(const Epilogue& ep, int N, int b1, int b2, int m, int n, float a0) {
  if (n >= N) return;
  const int64_t o = static_cast<int64_t>(b1) * ep.out_sb1 + static_cast<int64_t>(b2) * ep.out_sb2 +
                    static_cast<int64_t>(m) * ep.out_sm + static_cast<int64_t>(n) * ep.out_sn;
  static_cast<T*>(ep.out)[o] = from_f<T>(epi_value<T>(ep, b1, b2, m, n, a0, o));
}

}  // namespace ac
