// NEXT f1: fused (memory-efficient) attention for sm_100a, o = softmax(q k^T * scale) v
// with no N x N tensor in HBM (the "fused attention kernel" regime of the paper,
// P:350-351; the graph node kind attn_fused).  One CTA per SM, persistent over work
// units of NT query tiles (128 rows each, the same head, adjacent rows), causal units
// heaviest first.
//
//   warp 0       : TMA producer - the unit's Q tiles once, K / V^T blocks of 128 keys
//                  through a 3-stage ring shared by the NT tiles (128B swizzle)
//   warp 1       : TMEM allocator + MMA issuer.  Jobs (tile t, key block j) in the
//                  order j-major, t-minor; job k: S = Q_t K_j^T (M=128, N=128, K=64) into
//                  TMEM slot k % 3, so the tensor core runs up to two jobs ahead of the
//                  softmax warpgroups (NT = 2: the two tiles' softmax phases overlap each
//                  other and the MMAs); O_t += P V_j (M=128, N=64, K=128) with P read from
//                  TMEM (the slot's first 64 columns, bf16 pairs) - issued right before
//                  the slot's next S, so the tensor core's in-order execution keeps the
//                  slot's WAR order
//   warp 3       : idle (NT = 2: registers handed to the softmax warpgroups)
//   warpgroup 1+t: softmax of tile t, thread = query row over all 128 keys of a block:
//                  max, lazy online reference (moves only when the block max exceeds
//                  it by FA_LAZY log2 units, so most blocks need no O rescale),
//                  P = bf16(2^(x - m)) stored to TMEM, l += sum; O rescaled in TMEM when
//                  the reference moved; at the end o = O / l stored as bf16.
// Same arithmetic whatever chunk a query row falls in (the key loop, its order and the
// reference sequence depend only on the global row), so chunked == unchunked bitwise.
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

constexpr int FA_BM = 128;       // query rows per tile
constexpr int FA_BN = 128;       // keys per block
constexpr int FA_DH = 64;        // head dim (one 128-byte swizzle row)
constexpr int FA_STG = 4;        // K ring and V ring depth (separate rings: K is released by the
                                 // block's last S, V by its last PV, which runs three jobs later)
constexpr float FA_LAZY = 8.f;   // reference-update threshold of the online softmax (log2 units)
constexpr int Q_BYTES = FA_BM * FA_DH * 2;   // 16 KB
constexpr int K_BYTES = FA_BN * FA_DH * 2;   // 16 KB
// V^T per stage: two 64-key boxes, each 64 rows (head dim) of 128 B from TMA plus 16 rows
// of bf16 ones written once at kernel start, so the PV MMA (N = 80) also accumulates the
// row sums of P in the output's column 64: l = sum of exactly the bf16 P the MMA used,
// no per-element additions in the softmax
constexpr int V_BOX = 64 * 128 + 16 * 128;   // 10 KB
constexpr int V_BYTES = 2 * V_BOX;
constexpr int FA_OW = 80;                    // O columns per tile: 64 head dims + 16 (column 64 = l)
constexpr int FA_OSTR = 96;                  // TMEM column stride between the tiles' O (32-aligned)
constexpr int FA_SLOTS = 3;                  // barrier slots allocated (NT = 2 uses 2 TMEM S slots)

template <int NT>
struct FaCfg {
  static constexpr int THREADS = 128 * (1 + NT);
  static constexpr int SMEM = 1024 + NT * Q_BYTES + FA_STG * (K_BYTES + V_BYTES) + 256;
};

struct alignas(64) FaArgs {
  CUtensorMap tq, tk, tv;
  __nv_bfloat16* out;
  long long o_srow, o_sh;
  int M, Nk, H;
  int MT;        // 128-row tiles
  int NP;        // units per head (ceil(MT / NT))
  int causal;
  long long row_off;
  float cl;      // scale * log2(e)
  int pdl;
};

// key blocks of query tile mt (0 for a tile past the rows)
__device__ __forceinline__ int fa_nkb(const FaArgs& a, int mt) {
  if (mt >= a.MT) return 0;
  long long kend = a.Nk;
  if (a.causal) {
    const long long e = a.row_off + static_cast<long long>(mt + 1) * FA_BM;
    if (e < kend) kend = e;
  }
  return static_cast<int>((kend + FA_BN - 1) / FA_BN);
}

// 16 consecutive 32-bit columns per thread (tcgen05.ld 32x32b.x16)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// 16 packed 32-bit columns per thread (tcgen05.st 32x32b.x16)
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// D(tmem) (+)= A(tmem) * B(smem)^T, kind::f16: A = 128 lanes x K/2 packed bf16 pairs
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int NT>
__global__ void __launch_bounds__(FaCfg<NT>::THREADS, 1) attn_fused_kernel(const __grid_constant__ FaArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + NT * Q_BYTES;
  uint8_t* sV = sK + FA_STG * K_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + FA_STG * V_BYTES);
  uint64_t* q_full = bar;
  uint64_t* q_empty = bar + 1;
  uint64_t* k_full = bar + 2;               // [FA_STG]
  uint64_t* k_empty = k_full + FA_STG;      // [FA_STG]
  uint64_t* v_full = k_empty + FA_STG;      // [FA_STG]
  uint64_t* v_empty = v_full + FA_STG;      // [FA_STG]
  uint64_t* s_full = v_empty + FA_STG;      // [3] per slot: S written (MMA commit)
  uint64_t* p_full = s_full + FA_SLOTS;     // [3] per slot: P stored, O rescaled (4 softmax warps)
  uint64_t* pv_done = p_full + FA_SLOTS;    // [2] per tile: a PV of the tile completed (MMA commit)
  uint64_t* o_free = pv_done + 2;           // [2] per tile: the epilogue read O (4 softmax warps)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_free + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = a.H * a.NP;
  // TMEM: SLOTS S slots of 128 columns, then O_t (80 columns) per tile: NT = 2 -> 2 slots
  // (the two tiles' softmax phases alternate), NT = 1 -> 3 (the tensor core runs ahead)
  constexpr int SLOTS = NT == 2 ? 2 : 3;
  constexpr int O_COL = SLOTS * 128;
  static_assert(O_COL + NT * FA_OSTR <= 512, "TMEM columns");
  // the ones rows of every V stage (constant; their swizzle is irrelevant)
  for (int i = threadIdx.x; i < FA_STG * 2 * 512; i += blockDim.x) {
    const int box = i / 512, w = i % 512;
    reinterpret_cast<uint32_t*>(sV + box * V_BOX + 8192)[w] = 0x3F803F80u;
  }
  ptx::fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&a.tq);
    ptx::prefetch_tmap(&a.tk);
    ptx::prefetch_tmap(&a.tv);
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int s = 0; s < FA_STG; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 1);
      ptx::mbar_init(&v_full[s], 1);
      ptx::mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < FA_SLOTS; ++b) {
      ptx::mbar_init(&s_full[b], 1);
      ptx::mbar_init(&p_full[b], 4);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&pv_done[b], 1);
      ptx::mbar_init(&o_free[b], 4);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_holder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  if (a.pdl) {  // chunk loop: the prologue overlapped the previous kernel; now wait for its results
    ptx::griddep_wait();
    ptx::griddep_launch();
  }
  // work unit u -> (head, first tile); causal: heaviest (last) units first
  auto unit = [&](int u, int& head, int& mt0) {
    const int r = u / a.H;
    head = u - r * a.H;
    mt0 = (a.causal ? a.NP - 1 - r : r) * NT;
  };

  if (warp < 4) {
    // NT = 2: 384 threads x 168 registers at launch; the softmax warpgroups take the
    // producer / MMA warpgroup's spare registers (168 -> 96 there, 168 -> 200 here)
    if constexpr (NT == 2) ptx::setmaxnreg_dec<96>();
    if (warp == 0 && lane == 0) {
      int st = 0;
      uint32_t ph = 0, qph = 0;
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        int head, mt0;
        unit(u, head, mt0);
        int nkb = 0, nq = 0;
        for (int t = 0; t < NT; ++t) {
          const int k = fa_nkb(a, mt0 + t);
          nkb = k > nkb ? k : nkb;
          nq += k > 0;
        }
        ptx::mbar_wait(q_empty, qph ^ 1);
        qph ^= 1;
        ptx::mbar_expect_tx(q_full, nq * Q_BYTES);
        for (int t = 0; t < nq; ++t) ptx::tma_load_4d(sQ + t * Q_BYTES, &a.tq, q_full, 0, (mt0 + t) * FA_BM, head, 0);
        for (int j = 0; j < nkb; ++j) {
          ptx::mbar_wait(&k_empty[st], ph ^ 1);
          ptx::mbar_expect_tx(&k_full[st], K_BYTES);
          ptx::tma_load_4d(sK + st * K_BYTES, &a.tk, &k_full[st], 0, j * FA_BN, head, 0);
          if (++st == FA_STG) { st = 0; ph ^= 1; }
        }
      }
    } else if (warp == 2 && lane == 0) {   // V^T blocks, on their own ring
      int st = 0;
      uint32_t ph = 0;
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        int head, mt0;
        unit(u, head, mt0);
        int nkb = 0;
        for (int t = 0; t < NT; ++t) {
          const int k = fa_nkb(a, mt0 + t);
          nkb = k > nkb ? k : nkb;
        }
        for (int j = 0; j < nkb; ++j) {
          ptx::mbar_wait(&v_empty[st], ph ^ 1);
          ptx::mbar_expect_tx(&v_full[st], 2 * 8192);
          ptx::tma_load_4d(sV + st * V_BYTES, &a.tv, &v_full[st], j * FA_BN, 0, head, 0);
          ptx::tma_load_4d(sV + st * V_BYTES + V_BOX, &a.tv, &v_full[st], j * FA_BN + 64, 0, head, 0);
          if (++st == FA_STG) { st = 0; ph ^= 1; }
        }
      }
    } else if (warp == 1) {
      constexpr uint32_t IDS = ptx::idesc_bf16(FA_BM, FA_BN);
      constexpr uint32_t IDO = ptx::idesc_bf16(FA_BM, FA_OW);
      // job k (this CTA's k-th (tile, block)) uses S slot k % 3; its PV is issued right
      // before S of job k + 3 overwrites the slot (in-order MMAs keep the WAR order), so
      // the tensor core runs up to two jobs ahead of the softmax warpgroups.  The three
      // pending PVs (jobs k-3, k-2, k-1) are a register FIFO: no dynamically indexed
      // arrays (local memory) on this warp's critical path.
      struct Pend {
        int t = -1, j = 0, st = 0, rel = 0, x = 0;
        uint32_t ph = 0, pph = 0;  // V stage phase, P phase of the slot
      };
      Pend q0, q1, q2;                    // oldest .. newest
      uint32_t o_units0 = 0, o_units1 = 0;  // units of tile 0 / 1 whose first PV was issued
      int st = 0, slot = 0;
      uint32_t ph = 0, qph = 0, pcnt = 0;  // pcnt: jobs issued (slot use = pcnt / 3)
      auto flush = [&](const Pend& e) {    // issue a pending PV
        if (e.t < 0) return;
        ptx::mbar_wait(&p_full[e.x], e.pph);
        if (e.j == 0) {
          uint32_t& ou = e.t ? o_units1 : o_units0;
          if (ou++ > 0) ptx::mbar_wait(&o_free[e.t], (ou - 2) & 1);
        }
        ptx::mbar_wait(&v_full[e.st], e.ph);
        ptx::tc_fence_after();
        if (lane == 0) {
          const uint32_t vb = ptx::smem_u32(sV + e.st * V_BYTES);
          const uint32_t ot = tmem + O_COL + e.t * FA_OSTR, pt = tmem + e.x * 128;
#pragma unroll
          for (int k = 0; k < FA_BN / 16; ++k)
            mma_bf16_ts(ot, pt + k * 8, ptx::sdesc_sw128(vb + (k >> 2) * V_BOX + (k & 3) * 32), IDO,
                        (e.j > 0 || k) ? 1u : 0u);
          ptx::mma_commit(&pv_done[e.t]);
          if (e.rel) ptx::mma_commit(&v_empty[e.st]);
        }
        __syncwarp();
      };
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        int head, mt0;
        unit(u, head, mt0);
        int nk0 = fa_nkb(a, mt0), nk1 = NT == 2 ? fa_nkb(a, mt0 + 1) : 0;
        const int nkb = nk0 > nk1 ? nk0 : nk1;
        ptx::mbar_wait(q_full, qph);
        qph ^= 1;
        for (int j = 0; j < nkb; ++j) {
          const int last_t = (NT == 2 && j < nk1) ? 1 : 0;
          bool loaded = false;
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (j >= (t ? nk1 : nk0)) continue;
            // the slot's previous P is consumed before S overwrites it; flushed before
            // waiting for block j's K (in-order issue keeps every ring moving)
            // the oldest pending PV is job k - SLOTS (SLOTS = 2: q1, q2 hold the pending jobs)
            if constexpr (SLOTS == 3) flush(q0);
            else flush(q1);
            if (!loaded) {
              ptx::mbar_wait(&k_full[st], ph);
              loaded = true;
            }
            ptx::tc_fence_after();
            if (lane == 0) {
              const uint32_t sa = ptx::smem_u32(sQ + t * Q_BYTES), sb = ptx::smem_u32(sK + st * K_BYTES);
              const uint32_t dt = tmem + slot * 128;
#pragma unroll
              for (int k = 0; k < FA_DH / 16; ++k)
                ptx::mma_bf16(dt, ptx::sdesc_sw128(sa + k * 32), ptx::sdesc_sw128(sb + k * 32), IDS, k ? 1u : 0u);
              ptx::mma_commit(&s_full[slot]);
              if (t == last_t) ptx::mma_commit(&k_empty[st]);              // block j's K no longer read
              if (j == nkb - 1 && t == last_t) ptx::mma_commit(q_empty);  // Q no longer read in this unit
            }
            __syncwarp();
            if constexpr (SLOTS == 3) q0 = q1;
            q1 = q2;
            q2.t = t;
            q2.j = j;
            q2.st = st;
            q2.ph = ph;
            q2.rel = t == last_t;
            q2.x = slot;
            q2.pph = (pcnt / SLOTS) & 1;
            ++pcnt;
            if (++slot == SLOTS) slot = 0;
          }
          if (++st == FA_STG) { st = 0; ph ^= 1; }
        }
      }
      // drain, oldest job first
      flush(q0);
      flush(q1);
      flush(q2);
    }
  } else {
    if constexpr (NT == 2) ptx::setmaxnreg_inc<200>();
    const int t = (warp - 4) >> 2;          // this warpgroup's tile of the unit
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lrow = static_cast<uint32_t>(quarter * 32) << 16;
    uint32_t pv_cnt = 0;                    // PVs of this tile awaited so far
    int gjob = 0;                           // jobs of this CTA so far (all tiles): slot = job % 3
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      int head, mt0;
      unit(u, head, mt0);
      int nk[NT];
      for (int tt = 0; tt < NT; ++tt) nk[tt] = fa_nkb(a, mt0 + tt);
      const int mt = mt0 + t;
      const int nkb = nk[t];
      if (nkb == 0) {
        for (int tt = 0; tt < NT; ++tt) gjob += nk[tt];
        continue;
      }
      const long long qg = a.row_off + static_cast<long long>(mt) * FA_BM + r;  // global query row
      float m = -CUDART_INF_F;
      for (int j = 0; j < nkb; ++j) {
        for (int tt = 0; tt < t; ++tt) gjob += j < nk[tt];       // the other tiles' jobs of block j first
        const int job = gjob++;
        for (int tt = t + 1; tt < NT; ++tt) gjob += j < nk[tt];
        const int x = job % SLOTS;
        ptx::mbar_wait(&s_full[x], (job / SLOTS) & 1);
        ptx::tc_fence_after();
        uint32_t sv[128];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          ptx::tmem_ld32(tmem + lrow + x * 128 + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[c * 32]));
        ptx::tmem_ld_wait();
        // mask: keys past the row (causal) or past Nk
        const long long k0 = static_cast<long long>(j) * FA_BN;
        long long lim = a.Nk - 1 - k0;
        if (a.causal && qg - k0 < lim) lim = qg - k0;
        if (lim < FA_BN - 1) {
#pragma unroll
          for (int c = 0; c < FA_BN; ++c)
            if (c > lim) sv[c] = __float_as_uint(-CUDART_INF_F);
        }
        float m8[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) m8[c] = __uint_as_float(sv[c]);
#pragma unroll
        for (int c = 8; c < FA_BN; ++c) m8[c & 7] = fmaxf(m8[c & 7], __uint_as_float(sv[c]));
        const float mb = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        const float mx = mb * a.cl;
        const float m_new = (m == -CUDART_INF_F || mx > m + FA_LAZY) ? fmaxf(m, mx) : m;
        const float mref = m_new == -CUDART_INF_F ? 0.f : m_new;
        const float alpha = m == -CUDART_INF_F ? 0.f : (m_new == m ? 1.f : ptx::ex2(m - mref));
        const uint64_t cl2 = ptx::f32x2_splat(a.cl), nm2 = ptx::f32x2_splat(-mref);
#pragma unroll
        for (int h = 0; h < 4; ++h) {   // 32 keys -> 16 packed columns of P per pass
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            float x0, x1;  // x = s * cl - m for a key pair in one FFMA2 (same rounding as fmaf)
            ptx::fma2(sv[h * 32 + 2 * c], sv[h * 32 + 2 * c + 1], cl2, nm2, x0, x1);
            const float e0 = ptx::ex2(x0);
            const float e1 = ptx::ex2(x1);
            __nv_bfloat162 hh = __floats2bfloat162_rn(e0, e1);
            pk[c] = *reinterpret_cast<uint32_t*>(&hh);
          }
          tmem_st16(tmem + lrow + x * 128 + h * 16, pk);
        }
        m = m_new;
        if (j >= 1) {
          // PV_{j-1} of this tile complete (NT = 2: it preceded this S on the tensor core)
          ptx::mbar_wait(&pv_done[t], pv_cnt & 1);
          ++pv_cnt;
          if (__any_sync(0xffffffffu, alpha != 1.f)) {
            // rescale O and its row-sum column (columns 64..79) by 2^(m_old - m_new)
            ptx::tc_fence_after();
            const uint32_t ob = tmem + lrow + O_COL + t * FA_OSTR;
            uint32_t o[32];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              ptx::tmem_ld32(ob + hh * 32, o);
              ptx::tmem_ld_wait();
#pragma unroll
              for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
              ptx::tmem_st32(ob + hh * 32, o);
            }
            tmem_ld16(ob + 64, o);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 16; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
            tmem_st16(ob + 64, o);
          }
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&p_full[x]);
      }
      // the other tiles' jobs past this tile's last block
      int nmax = 0;
      for (int tt = 0; tt < NT; ++tt) nmax = nk[tt] > nmax ? nk[tt] : nmax;
      for (int j = nkb; j < nmax; ++j)
        for (int tt = 0; tt < NT; ++tt) gjob += j < nk[tt];
      // epilogue: the tile's last PV, o = O / l
      ptx::mbar_wait(&pv_done[t], pv_cnt & 1);
      ++pv_cnt;
      ptx::tc_fence_after();
      uint32_t o[64], ls[16];
      const uint32_t ob = tmem + lrow + O_COL + t * FA_OSTR;
      ptx::tmem_ld32(ob, *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
      ptx::tmem_ld32(ob + 32, *reinterpret_cast<uint32_t(*)[32]>(&o[32]));
      tmem_ld16(ob + 64, ls);
      ptx::tmem_ld_wait();
      const float l = __uint_as_float(ls[0]);  // row sum of P (the ones column)
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&o_free[t]);
      const int mrow = mt * FA_BM + r;
      if (mrow < a.M) {
        const float inv = l > 0.f ? 1.f / l : 0.f;
        uint4* dst = reinterpret_cast<uint4*>(a.out + static_cast<long long>(mrow) * a.o_srow +
                                              static_cast<long long>(head) * a.o_sh);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
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
    ptx::tmem_dealloc<512>(tmem);
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

template <int NT>
cudaError_t attn_fused_launch(cudaStream_t s, FaArgs& a, long long units) {
  using CF = FaCfg<NT>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_fused_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = static_cast<int>(units < num_sms() ? units : num_sms());
  if (a.pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(CF::THREADS);
    cfg.dynamicSmemBytes = CF::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, attn_fused_kernel<NT>, a);
  }
  attn_fused_kernel<NT><<<grid, CF::THREADS, CF::SMEM, s>>>(a);
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
      !map3(&a.tk, p.k, FA_DH, p.Nk, p.H, p.k_srow, p.k_sh, FA_BN) ||
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
  // two query tiles per CTA (ping-pong) when the launch still fills every SM with
  // such pairs; otherwise one tile per CTA (short row chunks)
  if (tiles >= 2LL * num_sms()) {
    a.NP = (a.MT + 1) / 2;
    return attn_fused_launch<2>(s, a, static_cast<long long>(a.H) * a.NP);
  }
  a.NP = a.MT;
  return attn_fused_launch<1>(s, a, tiles);
}

}  // namespace ac
