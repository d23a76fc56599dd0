// NEXT f1: fused (memory-efficient) attention for sm_100a, o = softmax(q k^T * scale) v
// with no N x N tensor in HBM (the "fused attention kernel" regime of the paper,
// P:350-351; the graph node kind attn_fused).  One CTA per SM, persistent over
// (head, 128-row query tile) work tiles, causal tiles heaviest first.
//
//   warp 0     : TMA producer - Q tile once per work tile, K / V^T blocks of 128
//                keys through a 3-stage ring (128B swizzle)
//   warp 1     : TMEM allocator + MMA issuer: S_j = Q K_j^T into one of two TMEM
//                S buffers (M=128, N=128, K=64), O += P_j V_j (M=128, N=64, K=128)
//                into the TMEM O accumulator; order S_0, S_1, PV_0, S_2, PV_1, ...
//   warps 2..5 : softmax, thread = query row: online max / sum in the log2 domain
//                (x = s * scale * log2 e), P_j = 2^(x - m) rounded to bf16 into a
//                shared-memory A operand (128B-swizzled, two 64-key k-blocks), the
//                O accumulator rescaled by 2^(m_old - m_new) in TMEM before PV_j,
//                and at the end o = O / l stored as bf16.
// Same arithmetic whatever chunk a query row falls in (the key loop and its order
// depend only on the global row), so chunked == unchunked bitwise.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "kernels.h"
#include "ptx.cuh"

namespace ac {

namespace {

constexpr int FA_BM = 128;   // query rows per tile
// Key block BNK = 128 (one CTA per SM) or 64 (two CTAs per SM, whose softmax and
// MMA phases interleave; chosen when the launch has at least two tiles per SM)
template <int BNK>
struct FaCfg {
  static constexpr int BN = BNK;        // keys per block
  static constexpr int HK = BNK / 2;    // keys per softmax half-row
  static constexpr int MINB = BNK == 64 ? 2 : 1;
  static constexpr int OCOL = 2 * BNK;  // TMEM column of the O accumulator (after two S buffers)
  static constexpr int TMEM = OCOL + 64 <= 256 ? 256 : 512;
  static constexpr int K_BYTES = BNK * 64 * 2;
  static constexpr int V_BYTES = 64 * BNK * 2;   // 64-key boxes of 8 KB
  static constexpr int P_BYTES = 128 * BNK * 2;  // 64-key k-blocks of 16 KB
  static constexpr int SMEM = 1024 + 128 * 64 * 2 + 3 * (K_BYTES + V_BYTES) + 2 * P_BYTES + 256 + 2 * 2 * 128 * 4 +
                              128 * 4 * 2;
};
constexpr int FA_DH = 64;    // head dim (one 128-byte swizzle row)
constexpr int FA_STG = 3;    // K/V ring depth
constexpr int FA_THREADS = 320;  // producer, MMA, 8 softmax warps
constexpr int Q_BYTES = FA_BM * FA_DH * 2;        // 16 KB

struct alignas(64) FaArgs {
  CUtensorMap tq, tk, tv;
  __nv_bfloat16* out;
  long long o_srow, o_sh;
  int M, Nk, H;
  int MT;
  int causal;
  long long row_off;
  float cl;  // scale * log2(e)
  int pdl;
};

// 2^x on the FMA / ALU pipes (x <= 0, the softmax exponent): x = j + f with j the
// nearest integer, f in [-0.5, 0.5]; 2^f by a degree-3 polynomial (relative error
// 2.1e-4, below half a bf16 ulp of P); 2^j added to the exponent field.  x < -126
// (masked keys: -inf) gives 0.  Opt-in (AC_FA_POLY=1) for a fixed quarter of the
// columns, so that the MUFU unit carries three quarters of the exponentials.
__device__ __forceinline__ float ex2_poly(float x) {
  const float xc = fmaxf(x, -126.f);
  const float t = xc + 12582912.f;  // 1.5 * 2^23: round to nearest integer in the low bits
  const int j = __float_as_int(t) - 0x4B400000;
  const float f = xc - (t - 12582912.f);
  float p = fmaf(f, 0.05484806f, 0.24180646f);
  p = fmaf(f, p, 0.69324815f);
  p = fmaf(f, p, 0.99998868f);
  const float r = __int_as_float(__float_as_int(p) + (j << 23));
  return x < -126.f ? 0.f : r;
}

template <int BNK, bool POLY>
__global__ void __launch_bounds__(FA_THREADS, FaCfg<BNK>::MINB) attn_fused_kernel(const __grid_constant__ FaArgs a) {
  using CF = FaCfg<BNK>;
  constexpr int FA_BN = CF::BN, HK = CF::HK, OCOL = CF::OCOL, FA_TMEM = CF::TMEM;
  constexpr int K_BYTES = CF::K_BYTES, V_BYTES = CF::V_BYTES, P_BYTES = CF::P_BYTES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Q_BYTES;
  uint8_t* sV = sK + FA_STG * K_BYTES;
  uint8_t* sP = sV + FA_STG * V_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + 2 * P_BYTES);
  uint64_t* q_full = bar;
  uint64_t* q_empty = bar + 1;
  uint64_t* kv_full = bar + 2;              // [FA_STG]
  uint64_t* kv_empty = bar + 2 + FA_STG;    // [FA_STG]
  uint64_t* s_full = bar + 2 + 2 * FA_STG;  // [2]
  uint64_t* s_free = s_full + 2;            // [2]
  uint64_t* p_full = s_full + 4;            // [2]
  uint64_t* pv_done = s_full + 6;           // [2]: PV of block q commits to pv_done[q & 1]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_full + 8);
  // softmax row halves exchange their block maxima ([block parity][half][row]) and,
  // at the end, their partial sums ([half][row])
  float* xmax = reinterpret_cast<float*>(bar + 32);
  float* xsum = xmax + 2 * 2 * 128;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = a.H * a.MT;
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&a.tq);
    ptx::prefetch_tmap(&a.tk);
    ptx::prefetch_tmap(&a.tv);
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int s = 0; s < FA_STG; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&s_full[b], 1);
      ptx::mbar_init(&s_free[b], 8);
      ptx::mbar_init(&p_full[b], 8);
    }
    ptx::mbar_init(&pv_done[0], 1);
    ptx::mbar_init(&pv_done[1], 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<FA_TMEM>(tmem_holder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;  // S buffers at columns 0 / 128, O at 256
  if (a.pdl) {  // chunk loop: the prologue overlapped the previous kernel; now wait for its results
    ptx::griddep_wait();
    ptx::griddep_launch();
  }

  // work tile t -> (head, m-tile, key blocks); causal: heaviest (last) m-tiles first
  auto tile = [&](int t, int& head, int& mt, int& nkb) {
    const int r = t / a.H;
    head = t - r * a.H;
    mt = a.causal ? a.MT - 1 - r : r;
    long long kend = a.Nk;
    if (a.causal) {
      const long long e = a.row_off + static_cast<long long>(mt + 1) * FA_BM;
      if (e < kend) kend = e;
    }
    nkb = static_cast<int>((kend + FA_BN - 1) / FA_BN);
  };

  if (warp == 0) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0, qph = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int head, mt, nkb;
        tile(t, head, mt, nkb);
        ptx::mbar_wait(q_empty, qph ^ 1);
        qph ^= 1;
        ptx::mbar_expect_tx(q_full, Q_BYTES);
        ptx::tma_load_4d(sQ, &a.tq, q_full, 0, mt * FA_BM, head, 0);
        for (int j = 0; j < nkb; ++j) {
          ptx::mbar_wait(&kv_empty[st], ph ^ 1);
          ptx::mbar_expect_tx(&kv_full[st], K_BYTES + V_BYTES);
          ptx::tma_load_4d(sK + st * K_BYTES, &a.tk, &kv_full[st], 0, j * FA_BN, head, 0);
          for (int vb = 0; vb < FA_BN / 64; ++vb)
            ptx::tma_load_4d(sV + st * V_BYTES + vb * 8192, &a.tv, &kv_full[st], j * FA_BN + vb * 64, 0, head, 0);
          if (++st == FA_STG) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t IDS = ptx::idesc_bf16(FA_BM, FA_BN);
    constexpr uint32_t IDO = ptx::idesc_bf16(FA_BM, FA_DH);
    int st = 0;
    uint32_t ph = 0, qph = 0;
    int sidx = 0;  // S blocks issued by this CTA
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int head, mt, nkb;
      tile(t, head, mt, nkb);
      ptx::mbar_wait(q_full, qph);
      qph ^= 1;
      ptx::tc_fence_after();
      int pst = st;          // stage of the pending PV
      int pidx = sidx;       // block index of the pending PV
      for (int j = 0; j <= nkb; ++j) {
        if (j < nkb) {
          const int b = sidx & 1;
          ptx::mbar_wait(&kv_full[st], ph);
          ptx::mbar_wait(&s_free[b], ((sidx >> 1) & 1) ^ 1);
          ptx::tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = ptx::smem_u32(sQ), sb = ptx::smem_u32(sK + st * K_BYTES);
#pragma unroll
            for (int k = 0; k < FA_DH / 16; ++k)
              ptx::mma_bf16(tmem + b * FA_BN, ptx::sdesc_sw128(sa + k * 32), ptx::sdesc_sw128(sb + k * 32), IDS,
                            k ? 1u : 0u);
            ptx::mma_commit(&s_full[b]);
            if (j == nkb - 1) ptx::mma_commit(q_empty);  // Q no longer read in this tile
          }
          __syncwarp();
        }
        if (j >= 1) {
          // PV of block j - 1 (stage pst, P buffer pidx & 1)
          const int b = pidx & 1;
          ptx::mbar_wait(&p_full[b], (pidx >> 1) & 1);
          ptx::tc_fence_after();
          if (lane == 0) {
            const uint32_t pa = ptx::smem_u32(sP + b * P_BYTES), vb = ptx::smem_u32(sV + pst * V_BYTES);
#pragma unroll
            for (int k = 0; k < FA_BN / 16; ++k) {
              const int kb = k >> 2, kk = k & 3;
              ptx::mma_bf16(tmem + OCOL, ptx::sdesc_sw128(pa + kb * 16384 + kk * 32),
                            ptx::sdesc_sw128(vb + kb * 8192 + kk * 32), IDO, (j > 1 || k) ? 1u : 0u);
            }
            ptx::mma_commit(&kv_empty[pst]);
            ptx::mma_commit(&pv_done[pidx & 1]);
          }
          __syncwarp();
          pidx = sidx;
          pst = st;
        }
        if (j < nkb) {
          if (j == 0) { pidx = sidx; pst = st; }
          ++sidx;
          if (++st == FA_STG) { st = 0; ph ^= 1; }
        }
      }
    }
  } else {
    // softmax warps: thread = (query row r of the tile, half of the 128-key block);
    // warps w and w + 4 share TMEM lane quarter w % 4 and split each row's keys
    const int sw = warp - 2;
    const int quarter = warp & 3;
    const int hf = sw >> 2;  // keys hf*64 .. hf*64+63 of every block; O columns hf*32..
    const int r = quarter * 32 + lane;
    const uint32_t lrow = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t nbar = 1 + quarter;  // named barrier of the two warps of a quarter
    int sidx = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int head, mt, nkb;
      tile(t, head, mt, nkb);
      const long long qg = a.row_off + static_cast<long long>(mt) * FA_BM + r;  // global query row
      float m = -CUDART_INF_F, l = 0.f;  // l: this half's partial sum (same rescales as the other)
      for (int j = 0; j < nkb; ++j) {
        const int b = sidx & 1;
        ptx::mbar_wait(&s_full[b], (sidx >> 1) & 1);
        ptx::tc_fence_after();
        uint32_t s[HK];
#pragma unroll
        for (int c = 0; c < HK / 32; ++c)
          ptx::tmem_ld32(tmem + lrow + b * FA_BN + hf * HK + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[c * 32]));
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&s_free[b]);
        // mask: causal keys past the row, keys past Nk
        const long long k0 = static_cast<long long>(j) * FA_BN + hf * HK;
        long long lim = a.Nk - 1 - k0;  // last valid column of this half-block
        if (a.causal && qg - k0 < lim) lim = qg - k0;
        float mb = -CUDART_INF_F;
        if (lim >= HK - 1) {
#pragma unroll
          for (int c = 0; c < HK; ++c) mb = fmaxf(mb, __uint_as_float(s[c]));
        } else {
#pragma unroll
          for (int c = 0; c < HK; ++c) {
            if (c > lim) s[c] = __float_as_uint(-CUDART_INF_F);
            mb = fmaxf(mb, __uint_as_float(s[c]));
          }
        }
        // row max over both halves (slots double-buffered by block parity)
        xmax[((j & 1) * 2 + hf) * 128 + r] = mb;
        asm volatile("bar.sync %0, 64;" ::"r"(nbar) : "memory");
        mb = fmaxf(mb, xmax[((j & 1) * 2 + (hf ^ 1)) * 128 + r]);
        const float m_new = fmaxf(m, mb * a.cl);
        const float mref = m_new == -CUDART_INF_F ? 0.f : m_new;
        const float alpha = m == -CUDART_INF_F ? 0.f : ptx::ex2(m - mref);
        float ls = 0.f;
        uint32_t pk[HK / 2];
#pragma unroll
        for (int c = 0; c < HK / 2; ++c) {
          const float x0 = fmaf(__uint_as_float(s[2 * c]), a.cl, -mref);
          const float x1 = fmaf(__uint_as_float(s[2 * c + 1]), a.cl, -mref);
          // (columns 8q+6, 8q+7 of every 8 on the FMA pipe: the choice depends on the
          // column only, so chunked == unchunked stays bitwise)
          const bool pc = POLY && (c & 3) == 3;
          const float e0 = pc ? ex2_poly(x0) : ptx::ex2(x0);
          const float e1 = pc ? ex2_poly(x1) : ptx::ex2(x1);
          ls += e0 + e1;
          __nv_bfloat162 h = __floats2bfloat162_rn(e0, e1);
          pk[c] = *reinterpret_cast<uint32_t*>(&h);
        }
        l = l * alpha + ls;
        m = m_new;
        // O needs rescaling only when some row's max moved (alpha != 1; skipping a
        // multiply by 1.0 is exact): then PV_{j-1} must be complete; otherwise only
        // PV_{j-2} (the last reader of P buffer b) is awaited, so the exponentials of
        // block j overlap PV_{j-1}
        const bool resc = j >= 1 && __any_sync(0xffffffffu, alpha != 1.f);
        if (resc) {
          ptx::mbar_wait(&pv_done[(sidx - 1) & 1], ((sidx - 1) >> 1) & 1);
        } else if (sidx >= 2) {
          ptx::mbar_wait(&pv_done[sidx & 1], ((sidx - 2) >> 1) & 1);
        }
        if (resc) {
          ptx::tc_fence_after();
          uint32_t o[32];
          ptx::tmem_ld32(tmem + lrow + OCOL + hf * 32, o);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
          ptx::tmem_st32(tmem + lrow + OCOL + hf * 32, o);
          ptx::tmem_st_wait();
        }
        // this half's keys: k-block (hf*HK)/64 of P_j, 16-byte chunks from ((hf*HK)%64)/8
        uint8_t* pb = sP + b * P_BYTES + ((hf * HK) / 64) * 16384 + r * 128;
        constexpr int CH0 = 0;
        const int ch0 = ((hf * HK) % 64) / 8 + CH0;
#pragma unroll
        for (int c = 0; c < HK / 8; ++c) {
          const uint32_t addr = ptx::smem_u32(pb + (((ch0 + c) ^ (r & 7)) * 16));
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pk[4 * c]), "r"(pk[4 * c + 1]),
                       "r"(pk[4 * c + 2]), "r"(pk[4 * c + 3])
                       : "memory");
        }
        ptx::fence_proxy_async_smem();  // generic-proxy P writes -> visible to the tensor core
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&p_full[b]);
        ++sidx;
      }
      // epilogue: wait for the last PV; l = sum of both halves; o = O / l
      xsum[hf * 128 + r] = l;
      ptx::mbar_wait(&pv_done[(sidx - 1) & 1], ((sidx - 1) >> 1) & 1);
      ptx::tc_fence_after();
      uint32_t o[32];
      ptx::tmem_ld32(tmem + lrow + OCOL + hf * 32, o);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      asm volatile("bar.sync %0, 64;" ::"r"(nbar) : "memory");
      const float lt = l + xsum[(hf ^ 1) * 128 + r];
      asm volatile("bar.sync %0, 64;" ::"r"(nbar) : "memory");  // xsum reusable by the next tile
      const int mrow = mt * FA_BM + r;
      if (mrow < a.M) {
        const float inv = lt > 0.f ? 1.f / lt : 0.f;
        uint4* dst = reinterpret_cast<uint4*>(a.out + static_cast<long long>(mrow) * a.o_srow +
                                              static_cast<long long>(head) * a.o_sh + hf * 32);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 2 * e]) * inv,
                                                     __uint_as_float(o[8 * c + 2 * e + 1]) * inv);
            w[e] = *reinterpret_cast<uint32_t*>(&h);
          }
          dst[c] = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<FA_TMEM>(tmem);
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// bf16 map {inner (contiguous), rows, heads, 1} with element strides, box {64, box_rows, 1, 1}
// (rank 4 to match the 4-D TMA instruction the kernel issues)
bool map3(CUtensorMap* m, const void* p, long long inner, long long rows, long long heads, long long srow,
          long long sh, int box_rows) {
  EncodeFn enc = encode_fn();
  if (!enc || (reinterpret_cast<uintptr_t>(p) & 15)) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(heads), 1};
  const long long big = ((sh * heads + srow * rows) * 2 + 15) / 16 * 16;
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(srow * 2), static_cast<cuuint64_t>(sh * 2),
                           static_cast<cuuint64_t>(big)};
  if (strides[0] % 16 || strides[1] % 16 || !strides[0] || !strides[1]) return false;
  cuuint32_t box[4] = {64, static_cast<cuuint32_t>(box_rows), 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BNK, bool POLY>
cudaError_t attn_fused_launch(const AttnFusedProblem& p, cudaStream_t s, FaArgs& a, long long tiles) {
  using CF = FaCfg<BNK>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_fused_kernel<BNK, POLY>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (!map3(&a.tk, p.k, FA_DH, p.Nk, p.H, p.k_srow, p.k_sh, BNK)) return cudaErrorInvalidValue;
  const int grid = static_cast<int>(tiles < CF::MINB * num_sms() ? tiles : CF::MINB * num_sms());
  if (p.pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(FA_THREADS);
    cfg.dynamicSmemBytes = CF::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, attn_fused_kernel<BNK, POLY>, a);
  }
  attn_fused_kernel<BNK, POLY><<<grid, FA_THREADS, CF::SMEM, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t attn_fused(const AttnFusedProblem& p, cudaStream_t s) {
  if (p.M <= 0 || p.Nk <= 0 || p.H <= 0) return cudaSuccess;
  if (p.dh != FA_DH) return cudaErrorInvalidValue;
  FaArgs a;
  memset(&a, 0, sizeof(a));
  // q [M, H, dh] / k [Nk, H, dh]: inner dh; vt [H, dh, Nk]: inner keys, rows dh
  if (!map3(&a.tq, p.q, FA_DH, p.M, p.H, p.q_srow, p.q_sh, FA_BM) ||
      !map3(&a.tv, p.vt, p.Nk, FA_DH, p.H, p.v_sdh, p.v_sh, FA_DH))
    return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(p.out) & 15) || p.o_srow % 8 || p.o_sh % 8) return cudaErrorInvalidValue;
  a.out = static_cast<__nv_bfloat16*>(p.out);
  a.o_srow = p.o_srow;
  a.o_sh = p.o_sh;
  a.M = static_cast<int>(p.M);
  a.Nk = static_cast<int>(p.Nk);
  a.H = static_cast<int>(p.H);
  a.MT = static_cast<int>((p.M + FA_BM - 1) / FA_BM);
  a.causal = p.causal;
  a.row_off = p.row_off;
  a.cl = p.scale * 1.4426950408889634f;
  a.pdl = p.pdl;
  const long long tiles = static_cast<long long>(a.H) * a.MT;
  // two CTAs per SM (64-key blocks) only when the launch can fill them
  static const int force = getenv("AC_FA_BN") ? atoi(getenv("AC_FA_BN")) : 0;  // experiments
  const bool dual = force ? force == 64 : tiles >= 2 * num_sms();
  // AC_FA_POLY=1: a quarter of the exponentials on the FMA pipe (measured slower: the
  // kernel is not MUFU-bound — unchunked GPT attention 0.98 -> 1.11 ms, chunked equal)
  static const bool poly = getenv("AC_FA_POLY") && getenv("AC_FA_POLY")[0] == '1';
  if (poly) return dual ? attn_fused_launch<64, true>(p, s, a, tiles) : attn_fused_launch<128, true>(p, s, a, tiles);
  return dual ? attn_fused_launch<64, false>(p, s, a, tiles) : attn_fused_launch<128, false>(p, s, a, tiles);
}

}  // namespace ac
