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
                                                      int64_t ncols, int64_t ld, int causal, int64_t row_off, int64_t group, int64_t gstride,
                                                      int64_t ldo, int64_t gstrideo) {
  constexpr int VN = Vec<T>::N;
  constexpr int RPB = 256 / THREADS;
  __shared__ float red[2][8][RPB > 0 ? RPB : 1];
  const int sub = threadIdx.x / THREADS;       // row within block
  const int tid = threadIdx.x % THREADS;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * RPB + sub;
  const bool live = r < rows;
  const int64_t roff = group > 0 ? (r / group) * gstride + (r % group) * ld : r * ld;
  const int64_t rofo = group > 0 ? (r / group) * gstrideo + (r % group) * ldo : r * ldo;
  const T* srow = s + roff;
  T* prow = p + rofo;
  int64_t valid = ncols, wend = ncols;
  if (causal) {
    const int64_t R = row_off + (group > 0 ? r % group : r);
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
                           int64_t row_off, int64_t group, int64_t gstride, int64_t ldo, int64_t gstrideo,
                           cudaStream_t st) {
  constexpr int RPB = 256 / THREADS;
  const int64_t blocks = (rows + RPB - 1) / RPB;
  if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
  softmax_kernel<T, THREADS, VPT><<<static_cast<unsigned>(blocks), 256, 0, st>>>(
      static_cast<const T*>(s), static_cast<T*>(p), rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- pipelined bf16 softmax
// Persistent CTAs; each row is brought into shared memory with ONE bulk TMA copy
// (cp.async.bulk, mbarrier completion) issued NBUF-1 rows ahead, so HBM reads of
// the next rows overlap the reductions / exponentials / stores of this one.
// Reads touch only the row's valid (causal) prefix; the output is written from
// registers with coalesced 16-byte stores.
constexpr int SMX_THREADS = 512;
constexpr int SMX_NBUF = 3;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(SMX_THREADS) softmax_bulk_kernel(
    const __nv_bfloat16* __restrict__ s, __nv_bfloat16* __restrict__ p, int64_t rows, int64_t ncols, int64_t ld,
    int causal, int64_t row_off, int64_t group, int64_t gstride, int64_t ldo, int64_t gstrideo, int64_t cap_bytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  __shared__ float red[2][SMX_THREADS / 32];
  uint8_t* buf0 = sm + 128;
  const int tid = threadIdx.x;
  auto row_geom = [&](int64_t r, int64_t& sof, int64_t& pof, int64_t& valid, int64_t& wend) {
    sof = group > 0 ? (r / group) * gstride + (r % group) * ld : r * ld;
    pof = group > 0 ? (r / group) * gstrideo + (r % group) * ldo : r * ldo;
    valid = ncols;
    wend = ncols;
    if (causal) {
      const int64_t R = row_off + (group > 0 ? r % group : r);
      valid = R + 1 < ncols ? R + 1 : ncols;
      const int64_t k = ((R >> 7) + 1) << 7;
      wend = k < ncols ? k : ncols;
    }
  };
  auto issue = [&](int64_t r, int b) {
    int64_t sof, pof, valid, wend;
    row_geom(r, sof, pof, valid, wend);
    const uint32_t bytes = static_cast<uint32_t>(((valid * 2 + 15) / 16) * 16);
    const uint32_t mb = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[b]));
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(buf0 + b * cap_bytes));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(s + sof), "r"(bytes), "r"(mb)
                 : "memory");
  };
  if (tid == 0) {
    for (int b = 0; b < SMX_NBUF; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&bar[b]))));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t first = blockIdx.x, stride = gridDim.x;
  if (tid == 0)
    for (int b = 0; b < SMX_NBUF - 1; ++b)
      if (first + b * stride < rows) issue(first + b * stride, b);
  constexpr float L2E = 1.4426950408889634f;
  int64_t j = 0;
  for (int64_t r = first; r < rows; r += stride, ++j) {
    const int b = static_cast<int>(j % SMX_NBUF);
    const uint32_t par = static_cast<uint32_t>((j / SMX_NBUF) & 1);
    if (tid == 0) {
      const int64_t rn = r + (SMX_NBUF - 1) * stride;
      // the buffer was read through the generic proxy last iteration; order those
      // reads before the async-proxy (TMA) write that refills it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (rn < rows) issue(rn, static_cast<int>((j + SMX_NBUF - 1) % SMX_NBUF));
    }
    int64_t sof, pof, valid, wend;
    row_geom(r, sof, pof, valid, wend);
    {
      const uint32_t mb = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[b]));
      asm volatile(
          "{\n\t.reg .pred q;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n\t@!q bra W_%=;\n}" ::"r"(mb),
          "r"(par)
          : "memory");
    }
    const uint4* row = reinterpret_cast<const uint4*>(buf0 + b * cap_bytes);
    const int64_t nv = (valid + 7) / 8;
    float mx = -CUDART_INF_F;
    for (int64_t v = tid; v < nv; v += SMX_THREADS) {
      float f[8];
      Vec<__nv_bfloat16> q;
      q.raw = row[v];
      q.to_float(f);
      if ((v + 1) * 8 <= valid) {
#pragma unroll
        for (int e = 0; e < 8; ++e) mx = fmaxf(mx, f[e]);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (v * 8 + e < valid) mx = fmaxf(mx, f[e]);
      }
    }
    mx = warp_max(mx);
    if ((tid & 31) == 0) red[0][tid >> 5] = mx;
    __syncthreads();
    mx = red[0][0];
#pragma unroll
    for (int i = 1; i < SMX_THREADS / 32; ++i) mx = fmaxf(mx, red[0][i]);
    const float mxl = mx * L2E;
    float sum = 0.f;
    for (int64_t v = tid; v < nv; v += SMX_THREADS) {
      float f[8];
      Vec<__nv_bfloat16> q;
      q.raw = row[v];
      q.to_float(f);
      if ((v + 1) * 8 <= valid) {
#pragma unroll
        for (int e = 0; e < 8; ++e) sum += ex2(fmaf(f[e], L2E, -mxl));
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (v * 8 + e < valid) sum += ex2(fmaf(f[e], L2E, -mxl));
      }
    }
    sum = warp_sum(sum);
    if ((tid & 31) == 0) red[1][tid >> 5] = sum;
    __syncthreads();
    sum = 0.f;
#pragma unroll
    for (int i = 0; i < SMX_THREADS / 32; ++i) sum += red[1][i];
    const float inv = 1.f / sum;
    uint4* out = reinterpret_cast<uint4*>(p + pof);
    const int64_t nw = (wend + 7) / 8;
    for (int64_t v = tid; v < nw; v += SMX_THREADS) {
      float f[8];
      if (v < nv) {
        Vec<__nv_bfloat16> q;
        q.raw = row[v];
        q.to_float(f);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = (v * 8 + e < valid) ? ex2(fmaf(f[e], L2E, -mxl)) * inv : 0.f;
      Vec<__nv_bfloat16> o;
      o.from_float(f);
      out[v] = o.raw;
    }
    __syncthreads();  // buffer b and red[] free for reuse
  }
}

cudaError_t launch_softmax_bulk(const void* s, void* p, int64_t rows, int64_t ncols, int64_t ld, int causal,
                                int64_t row_off, int64_t group, int64_t gstride, int64_t ldo, int64_t gstrideo,
                                cudaStream_t st) {
  const int64_t cap = ((ncols * 2 + 127) / 128) * 128;
  const int smem = static_cast<int>(128 + SMX_NBUF * cap);
  static int attr_set = 0;
  if (attr_set < smem) {
    cudaError_t e = cudaFuncSetAttribute(softmax_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = 200 * 1024;
  }
  int per_sm = (220 * 1024) / smem;
  if (per_sm > 4) per_sm = 4;
  if (per_sm < 1) return cudaErrorInvalidValue;
  int64_t grid = static_cast<int64_t>(num_sms()) * per_sm;
  if (grid > rows) grid = rows;
  softmax_bulk_kernel<<<static_cast<unsigned>(grid), SMX_THREADS, smem, st>>>(
      static_cast<const __nv_bfloat16*>(s), static_cast<__nv_bfloat16*>(p), rows, ncols, ld, causal, row_off, group,
      gstride, ldo, gstrideo, cap);
  return cudaGetLastError();
}

template <typename T>
cudaError_t softmax_dispatch(const void* s, void* p, int64_t rows, int64_t ncols, int64_t ld, int causal,
                             int64_t row_off, int64_t group, int64_t gstride, int64_t ldo, int64_t gstrideo,
                           cudaStream_t st) {
  constexpr int VN = Vec<T>::N;
  const int64_t vecs = (ncols + VN - 1) / VN;
  if (sizeof(T) == 2 && ncols > 2048 && ncols <= 32768 && (reinterpret_cast<uintptr_t>(s) & 15) == 0)
    return launch_softmax_bulk(s, p, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
  if (vecs <= 32 * 1) return launch_softmax<T, 32, 1>(s, p, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
  if (vecs <= 32 * 2) return launch_softmax<T, 32, 2>(s, p, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
  if (vecs <= 32 * 4) return launch_softmax<T, 32, 4>(s, p, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
  if (vecs <= 32 * 8) return launch_softmax<T, 32, 8>(s, p, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
  if (vecs <= 256 * 2) return launch_softmax<T, 256, 2>(s, p, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
  if (vecs <= 256 * 4) return launch_softmax<T, 256, 4>(s, p, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
  if (vecs <= 256 * 8) return launch_softmax<T, 256, 8>(s, p, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
  if (vecs <= 256 * 16) return launch_softmax<T, 256, 16>(s, p, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
  if (vecs <= 256 * 32) return launch_softmax<T, 256, 32>(s, p, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
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

cudaError_t softmax_rows(const void* s_in, void* p_out, int64_t rows, int64_t ncols, int64_t ld, int64_t gstride,
                         int64_t ldo, int64_t gstrideo, int causal, int64_t row_off, int64_t group, int dtype,
                         cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  if (dtype == 1) {
    if (ld % 8 || ldo % 8 || ncols % 8) return cudaErrorInvalidValue;
    return softmax_dispatch<__nv_bfloat16>(s_in, p_out, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
  }
  if (ld % 4 || ldo % 4 || ncols % 4) return cudaErrorInvalidValue;
  return softmax_dispatch<float>(s_in, p_out, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
}

cudaError_t layernorm(const void* x, const void* gamma, const void* beta, void* y, int64_t rows, int C, float eps,
                      int dtype, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  if (dtype == 1) return layernorm_dispatch<__nv_bfloat16>(x, gamma, beta, y, rows, C, eps, st);
  return layernorm_dispatch<float>(x, gamma, beta, y, rows, C, eps, st);
}

}  // namespace ac
