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

#ifndef LNC_JT
#define LNC_JT 128
#endif

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
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
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

__device__ __forceinline__ float sc_to_f(float v) { return v; }
__device__ __forceinline__ float sc_to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T sc_from_f(float v);
template <>
__device__ __forceinline__ float sc_from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 sc_from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// Scalar fallback for rows the vector kernels cannot take (row length or stride
// not a multiple of the 16-byte vector, e.g. a 9-token sequence): one warp per row,
// three strided passes (max, sum, normalise); same masking and rounding as above.
template <typename T>
__global__ void __launch_bounds__(256) softmax_scalar_kernel(const T* __restrict__ s, T* __restrict__ p, int64_t rows,
                                                             int64_t ncols, int64_t ld, int causal, int64_t row_off,
                                                             int64_t group, int64_t gstride, int64_t ldo,
                                                             int64_t gstrideo) {
  const int lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int64_t roff = group > 0 ? (r / group) * gstride + (r % group) * ld : r * ld;
  const int64_t rofo = group > 0 ? (r / group) * gstrideo + (r % group) * ldo : r * ldo;
  const T* srow = s + roff;
  T* prow = p + rofo;
  int64_t valid = ncols;
  if (causal) {
    const int64_t R = row_off + (group > 0 ? r % group : r);
    valid = R + 1 < ncols ? R + 1 : ncols;
  }
  constexpr float L2E = 1.4426950408889634f;
  float mx = -CUDART_INF_F;
  for (int64_t c = lane; c < valid; c += 32) mx = fmaxf(mx, sc_to_f(srow[c]));
  mx = warp_max(mx);
  const float mxl = mx * L2E;
  float sum = 0.f;
  for (int64_t c = lane; c < valid; c += 32) sum += exp2f(fmaf(sc_to_f(srow[c]), L2E, -mxl));
  sum = warp_sum(sum);
  const float inv = 1.f / sum;
  for (int64_t c = lane; c < ncols; c += 32)
    prow[c] = sc_from_f<T>(c < valid ? exp2f(fmaf(sc_to_f(srow[c]), L2E, -mxl)) * inv : 0.f);
}

template <typename T>
cudaError_t launch_softmax_scalar(const void* s, void* p, int64_t rows, int64_t ncols, int64_t ld, int causal,
                                  int64_t row_off, int64_t group, int64_t gstride, int64_t ldo, int64_t gstrideo,
                                  cudaStream_t st) {
  const int64_t blocks = (rows + 7) / 8;
  if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
  softmax_scalar_kernel<T><<<static_cast<unsigned>(blocks), 256, 0, st>>>(
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

template <int TH>
__global__ void __launch_bounds__(TH) softmax_bulk_kernel(
    const __nv_bfloat16* __restrict__ s, __nv_bfloat16* __restrict__ p, int64_t rows, int64_t ncols, int64_t ld,
    int causal, int64_t row_off, int64_t group, int64_t gstride, int64_t ldo, int64_t gstrideo, int64_t cap_bytes) {
  constexpr int SMX_THREADS = TH;  // threads per row (CTA), sized to the launch's longest valid row
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  __shared__ float red[2][SMX_THREADS / 32];
  uint8_t* buf0 = sm + 128;
  const int tid = threadIdx.x;
  if (group <= 0) group = rows;
  // row r = gq * group + gr, tracked incrementally (no 64-bit division per row)
  struct Pos {
    int64_t gq, gr;
  };
  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int64_t sq = stride / group, sr = stride % group;
  auto advance = [&](Pos& p, int64_t times) {
    for (int64_t t = 0; t < times; ++t) {
      p.gq += sq;
      p.gr += sr;
      if (p.gr >= group) {
        p.gr -= group;
        p.gq += 1;
      }
    }
  };
  auto row_geom = [&](const Pos& p, int64_t& sof, int64_t& pof, int& valid, int& wend) {
    sof = p.gq * gstride + p.gr * ld;
    pof = p.gq * gstrideo + p.gr * ldo;
    valid = static_cast<int>(ncols);
    wend = static_cast<int>(ncols);
    if (causal) {
      const int64_t R = row_off + p.gr;
      valid = static_cast<int>(R + 1 < ncols ? R + 1 : ncols);
      const int64_t k = ((R >> 7) + 1) << 7;
      wend = static_cast<int>(k < ncols ? k : ncols);
    }
  };
  auto issue = [&](const Pos& pr, int b) {
    int64_t sof, pof;
    int valid, wend;
    row_geom(pr, sof, pof, valid, wend);
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
  Pos cur{first / group, first % group};
  Pos ahead = cur;  // thread 0: the row NBUF-1 iterations ahead
  if (tid == 0) {
    Pos q = cur;
    for (int b = 0; b < SMX_NBUF - 1; ++b) {
      if (first + b * stride < rows) issue(q, b);
      advance(q, 1);
    }
    ahead = q;
  }
  constexpr float L2E = 1.4426950408889634f;
  int64_t j = 0;
  for (int64_t r = first; r < rows; r += stride, ++j, advance(cur, 1)) {
    const int b = static_cast<int>(j % SMX_NBUF);
    const uint32_t par = static_cast<uint32_t>((j / SMX_NBUF) & 1);
    if (tid == 0) {
      const int64_t rn = r + (SMX_NBUF - 1) * stride;
      // the buffer was read through the generic proxy last iteration; order those
      // reads before the async-proxy (TMA) write that refills it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (rn < rows) issue(ahead, static_cast<int>((j + SMX_NBUF - 1) % SMX_NBUF));
      advance(ahead, 1);
    }
    int64_t sof, pof;
    int valid, wend;
    row_geom(cur, sof, pof, valid, wend);
    {
      const uint32_t mb = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[b]));
      asm volatile(
          "{\n\t.reg .pred q;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n\t@!q bra W_%=;\n}" ::"r"(mb),
          "r"(par)
          : "memory");
    }
    const uint4* row = reinterpret_cast<const uint4*>(buf0 + b * cap_bytes);
    const int nfull = valid >> 3, tail = valid & 7, nv = nfull + (tail ? 1 : 0);
    float mx = -CUDART_INF_F;
    {
      __nv_bfloat162 m2 = __float2bfloat162_rn(-CUDART_INF_F);
      for (int v = tid; v < nfull; v += SMX_THREADS) {
        const uint4 u = row[v];
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
        m2 = __hmax2(m2, __hmax2(__hmax2(h[0], h[1]), __hmax2(h[2], h[3])));
      }
      const float2 mf = __bfloat1622float2(m2);
      mx = fmaxf(mf.x, mf.y);
      if (tail && tid == (nfull % SMX_THREADS)) {
        float f[8];
        Vec<__nv_bfloat16> q;
        q.raw = row[nfull];
        q.to_float(f);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (e < tail) mx = fmaxf(mx, f[e]);
      }
    }
    mx = warp_max(mx);
    if ((tid & 31) == 0) red[0][tid >> 5] = mx;
    __syncthreads();
    mx = red[0][0];
#pragma unroll
    for (int i = 1; i < SMX_THREADS / 32; ++i) mx = fmaxf(mx, red[0][i]);
    const float mxl = mx * L2E;
    // pass 2: e = exp(s - m) once per element; the sum uses the fp32 e, the row
    // buffer is overwritten in place with bf16(e) for the normalising pass
    float sum = 0.f;
    uint4* rowm = const_cast<uint4*>(row);
    for (int v = tid; v < nfull; v += SMX_THREADS) {
      float f[8];
      Vec<__nv_bfloat16> q;
      q.raw = row[v];
      q.to_float(f);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        f[e] = ex2(fmaf(f[e], L2E, -mxl));
        sum += f[e];
      }
      q.from_float(f);
      rowm[v] = q.raw;
    }
    if (tail && tid == (nfull % SMX_THREADS)) {
      float f[8];
      Vec<__nv_bfloat16> q;
      q.raw = row[nfull];
      q.to_float(f);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        f[e] = e < tail ? ex2(fmaf(f[e], L2E, -mxl)) : 0.f;
        sum += f[e];
      }
      q.from_float(f);
      rowm[nfull] = q.raw;
    }
    sum = warp_sum(sum);
    if ((tid & 31) == 0) red[1][tid >> 5] = sum;
    __syncthreads();
    sum = 0.f;
#pragma unroll
    for (int i = 0; i < SMX_THREADS / 32; ++i) sum += red[1][i];
    const float inv = 1.f / sum;
    uint4* out = reinterpret_cast<uint4*>(p + pof);
    const int nw = (wend + 7) >> 3;
    for (int v = tid; v < nw; v += SMX_THREADS) {
      uint4 w = make_uint4(0, 0, 0, 0);
      if (v < nv) {  // e (bf16, zero beyond the valid prefix) * 1/l
        float f[8];
        Vec<__nv_bfloat16> q;
        q.raw = row[v];
        q.to_float(f);
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] *= inv;
        q.from_float(f);
        w = q.raw;
      }
      out[v] = w;
    }
    __syncthreads();  // buffer b and red[] free for reuse
  }
}

// ---------------------------------------------------------------- long rows (> 32768 columns)
// Streaming two-read softmax: pass 1 keeps a per-thread online (max, sum) while
// streaming the row with several 16-byte loads in flight, the block combines
// them; pass 2 re-reads the row (mostly L2 hits: the rows in flight fit in L2)
// and writes p.  Rows stay out of registers and shared memory, so any length works.
constexpr int STR_THREADS = 512;
constexpr int STR_UNROLL = 4;

__global__ void __launch_bounds__(STR_THREADS) softmax_stream_kernel(
    const __nv_bfloat16* __restrict__ s, __nv_bfloat16* __restrict__ p, int64_t rows, int64_t ncols, int64_t ld,
    int causal, int64_t row_off, int64_t group, int64_t gstride, int64_t ldo, int64_t gstrideo) {
  __shared__ float red_m[STR_THREADS / 32], red_l[STR_THREADS / 32];
  const int tid = threadIdx.x;
  if (group <= 0) group = rows;
  constexpr float L2E = 1.4426950408889634f;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t gq = r / group, gr = r % group;
    const uint4* row = reinterpret_cast<const uint4*>(s + gq * gstride + gr * ld);
    uint4* out = reinterpret_cast<uint4*>(p + gq * gstrideo + gr * ldo);
    int64_t valid = ncols, wend = ncols;
    if (causal) {
      const int64_t R = row_off + gr;
      valid = R + 1 < ncols ? R + 1 : ncols;
      const int64_t k = ((R >> 7) + 1) << 7;
      wend = k < ncols ? k : ncols;
    }
    const int nv = static_cast<int>((valid + 7) >> 3);
    float m = -CUDART_INF_F, l = 0.f;
    for (int v0 = tid; v0 < nv; v0 += STR_THREADS * STR_UNROLL) {
      uint4 u[STR_UNROLL];
#pragma unroll
      for (int k = 0; k < STR_UNROLL; ++k) {
        const int v = v0 + k * STR_THREADS;
        if (v < nv) u[k] = row[v];
      }
#pragma unroll
      for (int k = 0; k < STR_UNROLL; ++k) {
        const int v = v0 + k * STR_THREADS;
        if (v >= nv) break;
        float f[8];
        Vec<__nv_bfloat16> q;
        q.raw = u[k];
        q.to_float(f);
        float vm = -CUDART_INF_F;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (static_cast<int64_t>(v) * 8 + e >= valid) f[e] = -CUDART_INF_F;
          vm = fmaxf(vm, f[e]);
        }
        if (vm > m) {
          l *= ex2((m - vm) * L2E);
          m = vm;
        }
        const float ml = m * L2E;
#pragma unroll
        for (int e = 0; e < 8; ++e) l += ex2(fmaf(f[e], L2E, -ml));
      }
    }
    // combine (m, l) across the block
    float mw = warp_max(m);
    float lw = l * (m == -CUDART_INF_F ? 0.f : ex2((m - mw) * L2E));
    lw = warp_sum(lw);
    if ((tid & 31) == 0) {
      red_m[tid >> 5] = mw;
      red_l[tid >> 5] = lw;
    }
    __syncthreads();
    float M = red_m[0];
#pragma unroll
    for (int i = 1; i < STR_THREADS / 32; ++i) M = fmaxf(M, red_m[i]);
    float Lsum = 0.f;
#pragma unroll
    for (int i = 0; i < STR_THREADS / 32; ++i)
      Lsum += red_m[i] == -CUDART_INF_F ? 0.f : red_l[i] * ex2((red_m[i] - M) * L2E);
    const float inv = 1.f / Lsum, ML = M * L2E;
    const int nw = static_cast<int>((wend + 7) >> 3);
    for (int v0 = tid; v0 < nw; v0 += STR_THREADS * STR_UNROLL) {
      uint4 u[STR_UNROLL];
#pragma unroll
      for (int k = 0; k < STR_UNROLL; ++k) {
        const int v = v0 + k * STR_THREADS;
        if (v < nv) u[k] = row[v];
      }
#pragma unroll
      for (int k = 0; k < STR_UNROLL; ++k) {
        const int v = v0 + k * STR_THREADS;
        if (v >= nw) break;
        uint4 w = make_uint4(0, 0, 0, 0);
        if (v < nv) {
          float f[8];
          Vec<__nv_bfloat16> q;
          q.raw = u[k];
          q.to_float(f);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            f[e] = static_cast<int64_t>(v) * 8 + e < valid ? ex2(fmaf(f[e], L2E, -ML)) * inv : 0.f;
          q.from_float(f);
          w = q.raw;
        }
        out[v] = w;
      }
    }
    __syncthreads();  // red_* reused by the next row
  }
}

cudaError_t launch_softmax_stream(const void* s, void* p, int64_t rows, int64_t ncols, int64_t ld, int causal,
                                  int64_t row_off, int64_t group, int64_t gstride, int64_t ldo, int64_t gstrideo,
                                  cudaStream_t st) {
  int64_t grid = static_cast<int64_t>(num_sms()) * 4;
  if (grid > rows) grid = rows;
  softmax_stream_kernel<<<static_cast<unsigned>(grid), STR_THREADS, 0, st>>>(
      static_cast<const __nv_bfloat16*>(s), static_cast<__nv_bfloat16*>(p), rows, ncols, ld, causal, row_off, group,
      gstride, ldo, gstrideo);
  return cudaGetLastError();
}

cudaError_t launch_softmax_bulk(const void* s, void* p, int64_t rows, int64_t ncols, int64_t ld, int causal,
                                int64_t row_off, int64_t group, int64_t gstride, int64_t ldo, int64_t gstrideo,
                                cudaStream_t st) {
  // a causal launch never reads beyond its last row's diagonal: size the row
  // buffers (and the CTA) by the longest valid prefix, so early chunks get many
  // small CTAs per SM (more rows in flight) instead of a few half-empty ones
  int64_t maxv = ncols;
  if (causal) {
    const int64_t last = row_off + (group > 0 ? group : rows);
    if (last < maxv) maxv = last;
  }
  const int64_t cap = ((maxv * 2 + 127) / 128) * 128;
  const int smem = static_cast<int>(128 + SMX_NBUF * cap);
  static bool attr_set = false;
  if (!attr_set) {
    for (auto fn : {softmax_bulk_kernel<128>, softmax_bulk_kernel<256>, softmax_bulk_kernel<512>}) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (e != cudaSuccess) return e;
    }
    attr_set = true;
  }
  const int th = maxv >= 8192 ? 512 : (maxv >= 2048 ? 256 : 128);
  int per_sm = (220 * 1024) / smem;
  if (per_sm > 2048 / th) per_sm = 2048 / th;
  if (per_sm < 1) return cudaErrorInvalidValue;
  int64_t grid = static_cast<int64_t>(num_sms()) * per_sm;
  if (grid > rows) grid = rows;
  auto S = static_cast<const __nv_bfloat16*>(s);
  auto P = static_cast<__nv_bfloat16*>(p);
  const unsigned g = static_cast<unsigned>(grid);
  if (th == 512)
    softmax_bulk_kernel<512><<<g, 512, smem, st>>>(S, P, rows, ncols, ld, causal, row_off, group, gstride, ldo,
                                                    gstrideo, cap);
  else if (th == 256)
    softmax_bulk_kernel<256><<<g, 256, smem, st>>>(S, P, rows, ncols, ld, causal, row_off, group, gstride, ldo,
                                                    gstrideo, cap);
  else
    softmax_bulk_kernel<128><<<g, 128, smem, st>>>(S, P, rows, ncols, ld, causal, row_off, group, gstride, ldo,
                                                    gstrideo, cap);
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
  if (sizeof(T) == 2 && ncols > 32768)
    return launch_softmax_stream(s, p, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
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
// GS lanes per row (32: a warp per row; 8 lanes for rows of <= 16 vectors, e.g. the
// AlphaFold pair channels c_z = 128: four rows per warp, two 16-byte loads per lane in
// flight, instead of a warp per row with half its lanes idle).  The sums are xor
// butterflies over the GS lanes.
template <int GS>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = GS / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T, int VPT, int GS = 32>
__global__ void __launch_bounds__(256) layernorm_kernel(const T* __restrict__ x, const T* __restrict__ g,
                                                        const T* __restrict__ b, T* __restrict__ y, int64_t rows,
                                                        int C, float eps, int pdl, int64_t group, int64_t gx,
                                                        int64_t gy) {
  if (pdl) {  // chunk loop: launched early (programmatic dependent launch); wait for the input
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  constexpr int VN = Vec<T>::N;
  constexpr int RPW = 32 / GS;  // rows per warp
  const int lane = threadIdx.x & (GS - 1);
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 8 * RPW + (threadIdx.x >> 5) * RPW + ((threadIdx.x & 31) / GS);
  if (RPW == 1 && r0 >= rows) return;
  const bool rvalid = r0 < rows;  // (groups of a warp share its shuffles: no early exit)
  const int64_t r = rvalid ? r0 : rows - 1;
  // rows in groups of `group` contiguous rows, groups gx / gy elements apart (a view
  // cut along a middle dim, e.g. a column chunk of the pair representation)
  const int64_t gi = r / group, ri = r - gi * group;
  const T* xr = x + gi * gx + ri * C;
  T* yr = y + gi * gy + ri * C;
  const int nv = C / VN;
  float f[VPT][VN];
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int vi = i * GS + lane;
    if (vi < nv) {
      Vec<T> v;
      v.raw = *reinterpret_cast<const uint4*>(xr + vi * VN);
      v.to_float(f[i]);
#pragma unroll
      for (int e = 0; e < VN; ++e) sum += f[i][e];
    }
  }
  const float mean = group_sum<GS>(sum) / static_cast<float>(C);
  float sq = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int vi = i * GS + lane;
    if (vi < nv) {
#pragma unroll
      for (int e = 0; e < VN; ++e) {
        const float d = f[i][e] - mean;
        sq += d * d;
      }
    }
  }
  const float var = group_sum<GS>(sq) / static_cast<float>(C);
  const float inv = 1.f / sqrtf(var + eps);
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int vi = i * GS + lane;
    if (vi < nv && rvalid) {
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
                               float eps, cudaStream_t st, int pdl, int64_t group, int64_t gx, int64_t gy) {
  constexpr int VN = Vec<T>::N;
  if (C % VN != 0) return cudaErrorInvalidValue;
  const int nv = C / VN;
  const int rpb = 8 * (nv <= 16 ? 4 : 1);  // rows per 256-thread block
  const int64_t blocks = (rows + rpb - 1) / rpb;
  if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
  const unsigned gb = static_cast<unsigned>(blocks);
  auto X = static_cast<const T*>(x);
  auto G = static_cast<const T*>(g);
  auto B = static_cast<const T*>(b);
  auto Y = static_cast<T*>(y);
  if (group <= 0 || gx % VN || gy % VN) return cudaErrorInvalidValue;
  void (*kern)(const T*, const T*, const T*, T*, int64_t, int, float, int, int64_t, int64_t, int64_t) =
      nv <= 8 ? layernorm_kernel<T, 1, 8> : nv <= 16 ? layernorm_kernel<T, 2, 8>
      : nv <= 32 ? layernorm_kernel<T, 1> : nv <= 64 ? layernorm_kernel<T, 2> : nv <= 128 ? layernorm_kernel<T, 4>
      : nv <= 256 ? layernorm_kernel<T, 8> : nv <= 512 ? layernorm_kernel<T, 16> : nullptr;
  if (!kern) return cudaErrorInvalidValue;
  if (pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(gb);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, X, G, B, Y, rows, C, eps, 1, group, gx, gy);
  }
  kern<<<gb, 256, 0, st>>>(X, G, B, Y, rows, C, eps, 0, group, gx, gy);
  return cudaGetLastError();
}

// LayerNorm over the leading (channel) dim of x [C, I, J] written channel-last,
// y[i, j, :] = gamma * (x[:, i, j] - mu) / sqrt(var + eps) + beta (ln_cfirst, AF2
// Alg. 11 line 4: the LN of the triangle product, whose GEMM leaves it channel-major).
// One CTA per (i, JT j): the [C x JT] tile is read coalesced along j into shared
// memory (fp32, pitch JT + 1), 256 / JT threads per column fold its mean and then its
// variance (two passes, fp32), and the normalised tile leaves coalesced along c in
// 16-byte vectors.  HBM-bound: one read and one write of x.
template <typename T, int JT>
__global__ void __launch_bounds__(256) ln_cfirst_kernel(const T* __restrict__ x, int64_t xs_c, int64_t xs_i,
                                                         const T* __restrict__ g, const T* __restrict__ b,
                                                         T* __restrict__ y, int64_t ys_i, int64_t ys_j, int C,
                                                         int64_t J, float eps, int pdl) {
  constexpr int PT = JT + 1;     // smem pitch (odd: column reads conflict-free)
  constexpr int TPC = 256 / JT;  // threads per column in the statistics pass
  extern __shared__ float lsm[];  // [C][JT + 1] values, then mu[JT], rstd[JT]
  float* mu = lsm + C * PT;
  float* rs = mu + JT;
  if (pdl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  const int64_t i = blockIdx.y;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * JT;
  const int jn = static_cast<int>(J - j0 < JT ? J - j0 : JT);
  constexpr int VL = 16 / sizeof(T);  // elements per 16-byte load
  if (jn == JT && (xs_c % VL) == 0 && (xs_i % VL) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    // full tile: 16-byte loads along j (a c-row of the tile is 64 / VL vectors)
    for (int idx = threadIdx.x; idx < C * (JT / VL); idx += 256) {
      const int c = idx / (JT / VL), jv = (idx - c * (JT / VL)) * VL;
      Vec<T> v;
      v.raw = *reinterpret_cast<const uint4*>(x + c * xs_c + i * xs_i + j0 + jv);
      float f[VL];
      v.to_float(f);
#pragma unroll
      for (int e = 0; e < VL; ++e) lsm[c * PT + jv + e] = f[e];
    }
  } else {
    for (int idx = threadIdx.x; idx < C * JT; idx += 256) {
      const int c = idx / JT, jj = idx % JT;
      lsm[c * PT + jj] = jj < jn ? static_cast<float>(x[c * xs_c + i * xs_i + j0 + jj]) : 0.f;
    }
  }
  __syncthreads();
  {
    const int col = threadIdx.x / TPC, part = threadIdx.x % TPC;
    float s = 0.f;
    for (int c = part; c < C; c += TPC) s += lsm[c * PT + col];
#pragma unroll
    for (int o = 1; o < TPC; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float m = s / static_cast<float>(C);
    float q = 0.f;
    for (int c = part; c < C; c += TPC) {
      const float d = lsm[c * PT + col] - m;
      q += d * d;
    }
#pragma unroll
    for (int o = 1; o < TPC; o <<= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    if (part == 0) {
      mu[col] = m;
      rs[col] = 1.f / sqrtf(q / static_cast<float>(C) + eps);
    }
  }
  __syncthreads();
  constexpr int VN = Vec<T>::N;
  const int cv = C / VN;
  for (int idx = threadIdx.x; idx < jn * cv; idx += 256) {
    const int jj = idx / cv, c0 = (idx - jj * cv) * VN;
    Vec<T> gv, bv, o;
    gv.raw = *reinterpret_cast<const uint4*>(g + c0);
    bv.raw = *reinterpret_cast<const uint4*>(b + c0);
    float gf[VN], bf[VN], of[VN];
    gv.to_float(gf);
    bv.to_float(bf);
#pragma unroll
    for (int e = 0; e < VN; ++e) of[e] = (lsm[(c0 + e) * PT + jj] - mu[jj]) * rs[jj] * gf[e] + bf[e];
    o.from_float(of);
    *reinterpret_cast<uint4*>(y + i * ys_i + (j0 + jj) * ys_j + c0) = o.raw;
  }
}

}  // namespace

cudaError_t layernorm_cfirst(const void* x, int64_t xs_c, int64_t xs_i, const void* gamma, const void* beta, void* y,
                             int64_t ys_i, int64_t ys_j, int C, int64_t I, int64_t J, float eps, int dtype,
                             cudaStream_t st, int pdl) {
  if (I <= 0 || J <= 0) return cudaSuccess;
  const int VN = dtype == 1 ? 8 : 4;
  auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (C % VN || C > 1024 || ys_j % VN || ys_i % VN || !al(y) || !al(gamma) || !al(beta)) return cudaErrorInvalidValue;
  // bf16: 128-column j tiles (each block reads 256 contiguous bytes of every channel row,
  // the rows being a 2 MB page apart for the AlphaFold pair tensor); fp32: 64
  constexpr int JTB = LNC_JT;
  const bool wide = dtype == 1 && (static_cast<size_t>(C) * (JTB + 1) + 2 * JTB) * 4 <= 200 * 1024;
  const int JT = wide ? JTB : 64;
  const size_t smem = (static_cast<size_t>(C) * (JT + 1) + 2 * JT) * 4;
  dim3 grid(static_cast<unsigned>((J + JT - 1) / JT), static_cast<unsigned>(I));
  auto launch = [&](auto kern, auto* X, auto* G, auto* B, auto* Y) -> cudaError_t {
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      if (e != cudaSuccess) return e;
    }
    if (pdl) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = grid;
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute la[1];
      la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      la[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = la;
      cfg.numAttrs = 1;
      return cudaLaunchKernelEx(&cfg, kern, X, xs_c, xs_i, G, B, Y, ys_i, ys_j, C, J, eps, 1);
    }
    kern<<<grid, 256, smem, st>>>(X, xs_c, xs_i, G, B, Y, ys_i, ys_j, C, J, eps, 0);
    return cudaGetLastError();
  };
  if (dtype == 1) {
    using T = __nv_bfloat16;
    if (wide)
      return launch(ln_cfirst_kernel<T, JTB>, static_cast<const T*>(x), static_cast<const T*>(gamma),
                    static_cast<const T*>(beta), static_cast<T*>(y));
    return launch(ln_cfirst_kernel<T, 64>, static_cast<const T*>(x), static_cast<const T*>(gamma),
                  static_cast<const T*>(beta), static_cast<T*>(y));
  }
  return launch(ln_cfirst_kernel<float, 64>, static_cast<const float*>(x), static_cast<const float*>(gamma),
                static_cast<const float*>(beta), static_cast<float*>(y));
}

cudaError_t softmax_rows(const void* s_in, void* p_out, int64_t rows, int64_t ncols, int64_t ld, int64_t gstride,
                         int64_t ldo, int64_t gstrideo, int causal, int64_t row_off, int64_t group, int dtype,
                         cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (dtype == 1) {
    if (ld % 8 || ldo % 8 || ncols % 8 || gstride % 8 || gstrideo % 8 || !al(s_in) || !al(p_out))
      return launch_softmax_scalar<__nv_bfloat16>(s_in, p_out, rows, ncols, ld, causal, row_off, group, gstride, ldo,
                                                  gstrideo, st);
    return softmax_dispatch<__nv_bfloat16>(s_in, p_out, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
  }
  if (ld % 4 || ldo % 4 || ncols % 4 || gstride % 4 || gstrideo % 4 || !al(s_in) || !al(p_out))
    return launch_softmax_scalar<float>(s_in, p_out, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
  return softmax_dispatch<float>(s_in, p_out, rows, ncols, ld, causal, row_off, group, gstride, ldo, gstrideo, st);
}

cudaError_t layernorm(const void* x, const void* gamma, const void* beta, void* y, int64_t rows, int C, float eps,
                      int dtype, cudaStream_t st, int pdl, int64_t group, int64_t gx, int64_t gy) {
  if (rows <= 0) return cudaSuccess;
  if (group <= 0) {  // contiguous rows
    group = rows;
    gx = gy = 0;
  }
  if (dtype == 1) return layernorm_dispatch<__nv_bfloat16>(x, gamma, beta, y, rows, C, eps, st, pdl, group, gx, gy);
  return layernorm_dispatch<float>(x, gamma, beta, y, rows, C, eps, st, pdl, group, gx, gy);
}

}  // namespace ac
