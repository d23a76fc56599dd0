// NEXT f1: fused (memory-efficient) attention for sm_100a, o = softmax(q k^T * scale) v
// with no N x N tensor in HBM (the "fused attention kernel" regime of the paper,
// P:350-351; the graph node kind attn_fused).  One CTA per SM, persistent over work units
// = (head, 128-row query tile), causal units heaviest first.  Each tile's key blocks are
// split into two halves at a position fixed by the tile's own key range (first ceil(n/2)
// blocks, the rest), one softmax warpgroup per half, merged at the end: a short row chunk
// (128 tiles < 148 SMs) keeps both warpgroups of every CTA busy, and the arithmetic of a
// row never depends on the launch, so chunked == unchunked bitwise.
//
//   warp 0       : TMA producer - the unit's Q tile once, K blocks of 128 keys through a
//                  4-stage ring (128B swizzle), one block per job
//   warp 2       : TMA producer of the V^T blocks (their own 4-stage ring)
//   warp 1       : TMEM allocator + MMA issuer.  Jobs (half t, block j) in the order
//                  j-major, t-minor; job k: S = Q K^T (M=128, N=128, K=64) into TMEM slot
//                  k % 2; O_t += P V (M=128, N=80, K=128) with P read from TMEM (the slot's
//                  first 64 columns, bf16 pairs), issued right before the slot's next S (the
//                  tensor core's in-order execution keeps the slot's WAR order); V^T carries
//                  16 rows of ones, so O_t's column 64 accumulates the row sum of P
//   warp 3       : idle (its registers go to the softmax warpgroups)
//   warpgroup 1+t: softmax of half t, thread = query row over all 128 keys of a block:
//                  max, lazy online reference (moves only when the block max exceeds it by
//                  FA_LAZY log2 units), P = bf16(2^(x - m)) stored to TMEM, O_t rescaled in
//                  TMEM when the reference moved.  At the end half 1 hands its reference
//                  over (shared memory + mbarrier) and half 0 merges:
//                  o = (a0 O_0 + a1 O_1) / (a0 l_0 + a1 l_1), a_t = 2^(m_t - max(m_0, m_1)).
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
constexpr int FA_STG = 4;        // K ring and V ring depth (separate rings: K is released by its
                                 // S, V by its PV, which runs two jobs later)
constexpr float FA_LAZY = 8.f;   // reference-update threshold of the online softmax (log2 units)
constexpr int Q_BYTES = FA_BM * FA_DH * 2;   // 16 KB
constexpr int K_BYTES = FA_BN * FA_DH * 2;   // 16 KB
// V^T per stage: two 64-key boxes, each 64 rows (head dim) of 128 B from TMA plus 16 rows
// of bf16 ones written once at kernel start, so the PV MMA (N = 80) also accumulates the
// row sums of P in the output's column 64: l = sum of exactly the bf16 P the MMA used,
// no per-element additions in the softmax
constexpr int V_BOX = 64 * 128 + 16 * 128;   // 10 KB
constexpr int V_BYTES = 2 * V_BOX;
constexpr int FA_OW = 80;                    // O columns per half: 64 head dims + 16 (column 64 = l)
constexpr int FA_OSTR = 96;                  // TMEM column stride between the halves' O (32-aligned)
constexpr int SLOTS = 2;                     // TMEM S slots (job k -> slot k % 2)
constexpr int O_COL = SLOTS * 128;           // O_0 at 256, O_1 at 352
constexpr int THREADS = 384;
constexpr int SMEM = 1024 + Q_BYTES + FA_STG * (K_BYTES + V_BYTES) + 512 + 128 * 4;

struct alignas(64) FaArgs {
  CUtensorMap tq, tk, tv;
  __nv_bfloat16* out;
  long long o_srow, o_sh;
  int M, Nk, H;
  int MT;        // 128-row tiles
  int causal;
  long long row_off;
  float cl;      // scale * log2(e)
  int pdl;
};

// key blocks of query tile mt
__device__ __forceinline__ int fa_nkb(const FaArgs& a, int mt) {
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

__global__ void __launch_bounds__(THREADS, 1) attn_fused_kernel(const __grid_constant__ FaArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // aligned by pointer arithmetic on the shared array (an integer round trip would
  // turn every later access into a generic LD / ST)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Q_BYTES;
  uint8_t* sV = sK + FA_STG * K_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + FA_STG * V_BYTES);
  uint64_t* q_full = bar;
  uint64_t* q_empty = bar + 1;
  uint64_t* k_full = bar + 2;               // [FA_STG]
  uint64_t* k_empty = k_full + FA_STG;      // [FA_STG]
  uint64_t* v_full = k_empty + FA_STG;      // [FA_STG]
  uint64_t* v_empty = v_full + FA_STG;      // [FA_STG]
  uint64_t* s_full = v_empty + FA_STG;      // [2] per slot: S written (MMA commit)
  uint64_t* p_full = s_full + SLOTS;        // [2] per slot: P stored, O rescaled (4 softmax warps)
  uint64_t* pv_done = p_full + SLOTS;       // [2] per half: a PV of the half completed (MMA commit)
  uint64_t* o_free = pv_done + 2;           // [2] per half: the merge read O_t (4 warps of half 0)
  uint64_t* merge_full = o_free + 2;        // half 1's reference is in sm1 (4 warps of half 1)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(merge_full + 1);
  float* sm1 = reinterpret_cast<float*>(bar + 64);  // [128] half 1's final reference per row

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = a.H * a.MT;
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
    for (int b = 0; b < SLOTS; ++b) {
      ptx::mbar_init(&s_full[b], 1);
      ptx::mbar_init(&p_full[b], 4);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&pv_done[b], 1);
      ptx::mbar_init(&o_free[b], 4);
    }
    ptx::mbar_init(merge_full, 4);
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
  // work unit u -> (head, tile); causal: heaviest (last) tiles first
  auto unit = [&](int u, int& head, int& mt) {
    const int r = u / a.H;
    head = u - r * a.H;
    mt = a.causal ? a.MT - 1 - r : r;
  };

  if (warp < 4) {
    // 384 threads x 168 registers at launch; the softmax warpgroups take this
    // warpgroup's spare registers (168 -> 96 here, 168 -> 200 there)
    ptx::setmaxnreg_dec<96>();
    if ((warp == 0 || warp == 2) && lane == 0) {
      // warp 0: Q + K blocks, warp 2: V^T blocks, one block per job in job order
      const bool isk = warp == 0;
      int st = 0;
      uint32_t ph = 0, qph = 0;
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        int head, mt;
        unit(u, head, mt);
        const int nkb = fa_nkb(a, mt), h0 = (nkb + 1) / 2;
        if (isk) {
          ptx::mbar_wait(q_empty, qph ^ 1);
          qph ^= 1;
          ptx::mbar_expect_tx(q_full, Q_BYTES);
          ptx::tma_load_4d(sQ, &a.tq, q_full, 0, mt * FA_BM, head, 0);
        }
        for (int j = 0; j < h0; ++j) {
          for (int t = 0; t < 2; ++t) {
            const int blk = 2 * j + t;
            if (blk >= nkb) continue;
            if (isk) {
              ptx::mbar_wait(&k_empty[st], ph ^ 1);
              ptx::mbar_expect_tx(&k_full[st], K_BYTES);
              ptx::tma_load_4d(sK + st * K_BYTES, &a.tk, &k_full[st], 0, blk * FA_BN, head, 0);
            } else {
              ptx::mbar_wait(&v_empty[st], ph ^ 1);
              ptx::mbar_expect_tx(&v_full[st], 2 * 8192);
              ptx::tma_load_4d(sV + st * V_BYTES, &a.tv, &v_full[st], blk * FA_BN, 0, head, 0);
              ptx::tma_load_4d(sV + st * V_BYTES + V_BOX, &a.tv, &v_full[st], blk * FA_BN + 64, 0, head, 0);
            }
            if (++st == FA_STG) { st = 0; ph ^= 1; }
          }
        }
      }
    } else if (warp == 1) {
      constexpr uint32_t IDS = ptx::idesc_bf16(FA_BM, FA_BN);
      constexpr uint32_t IDO = ptx::idesc_bf16(FA_BM, FA_OW);
      // job k uses S slot k % 2; its PV is issued right before S of job k + 2 overwrites the
      // slot.  The two pending PVs (jobs k-2, k-1) are a register FIFO (no local memory).
      struct Pend {
        int t = -1, j = 0, st = 0, x = 0;
        uint32_t ph = 0, pph = 0;  // V stage phase, P phase of the slot
      };
      Pend q1, q2;                        // older, newer
      uint32_t o_units0 = 0, o_units1 = 0;  // units of half 0 / 1 whose first PV was issued
      int st = 0, slot = 0;
      uint32_t ph = 0, qph = 0, pcnt = 0;
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
          ptx::mma_commit(&v_empty[e.st]);
        }
        __syncwarp();
      };
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        int head, mt;
        unit(u, head, mt);
        const int nkb = fa_nkb(a, mt), h0 = (nkb + 1) / 2;
        ptx::mbar_wait(q_full, qph);
        qph ^= 1;
        for (int j = 0; j < h0; ++j) {
          for (int t = 0; t < 2; ++t) {
            const int blk = 2 * j + t;
            if (blk >= nkb) continue;
            flush(q1);  // the slot's previous P is consumed before S overwrites it
            ptx::mbar_wait(&k_full[st], ph);
            ptx::tc_fence_after();
            if (lane == 0) {
              const uint32_t sa = ptx::smem_u32(sQ), sb = ptx::smem_u32(sK + st * K_BYTES);
              const uint32_t dt = tmem + slot * 128;
#pragma unroll
              for (int k = 0; k < FA_DH / 16; ++k)
                ptx::mma_bf16(dt, ptx::sdesc_sw128(sa + k * 32), ptx::sdesc_sw128(sb + k * 32), IDS, k ? 1u : 0u);
              ptx::mma_commit(&s_full[slot]);
              ptx::mma_commit(&k_empty[st]);                  // K read by this S only
              if (blk == nkb - 1) ptx::mma_commit(q_empty);  // the unit's last S (jobs run in block order)
            }
            __syncwarp();
            q1 = q2;
            q2.t = t;
            q2.j = j;
            q2.st = st;
            q2.ph = ph;
            q2.x = slot;
            q2.pph = (pcnt / SLOTS) & 1;
            ++pcnt;
            if (++slot == SLOTS) slot = 0;
            if (++st == FA_STG) { st = 0; ph ^= 1; }
          }
        }
      }
      flush(q1);
      flush(q2);
    }
  } else {
    ptx::setmaxnreg_inc<200>();
    const int t = (warp - 4) >> 2;          // this warpgroup's half of each tile's key blocks
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lrow = static_cast<uint32_t>(quarter * 32) << 16;
    uint32_t pv_cnt = 0;                    // PVs of this half awaited so far
    uint32_t merges = 0;                    // units merged (merge_full phase)
    int gjob = 0;                           // jobs of this CTA so far (both halves): slot = job % 2
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      int head, mt;
      unit(u, head, mt);
      const int nkb = fa_nkb(a, mt), h0 = (nkb + 1) / 2;
      const int nk0 = h0, nk1 = nkb - h0;   // even / odd key blocks
      const int nk = t ? nk1 : nk0;
      if (nk == 0) {                        // (half 1 of a one-block tile)
        gjob += nkb;
        continue;
      }
      const long long qg = a.row_off + static_cast<long long>(mt) * FA_BM + r;  // global query row
      float m = -CUDART_INF_F;
      for (int j = 0; j < nk; ++j) {
        if (t == 1) gjob += 1;                         // half 0's job of block pair j first
        const int job = gjob++;
        if (t == 0 && j < nk1) gjob += 1;              // then half 1's
        const int x = job % SLOTS;
        ptx::mbar_wait(&s_full[x], (job / SLOTS) & 1);
        ptx::tc_fence_after();
        uint32_t sv[128];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          ptx::tmem_ld32(tmem + lrow + x * 128 + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[c * 32]));
        ptx::tmem_ld_wait();
        // mask: keys past the row (causal) or past Nk
        const long long k0 = static_cast<long long>(2 * j + t) * FA_BN;
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
        // lazy reference: the running reference m moves only when the block max exceeds
        // it by more than FA_LAZY (log2 units), so P = 2^(x - m) <= 2^FA_LAZY; O and l
        // share the reference, so o = O / l is the same softmax.  The sequence of
        // references depends only on the row's keys, so chunked == unchunked bitwise.
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
          // this half's previous PV complete (it preceded this S on the tensor core)
          ptx::mbar_wait(&pv_done[t], pv_cnt & 1);
          ++pv_cnt;
          if (__any_sync(0xffffffffu, alpha != 1.f)) {
            // rescale O_t and its row-sum column (columns 64..79) by 2^(m_old - m_new)
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
      if (t == 1) gjob += nk0 - nk1;                   // half 0's jobs past half 1's last block
      // this half's last PV
      ptx::mbar_wait(&pv_done[t], pv_cnt & 1);
      ++pv_cnt;
      if (t == 1) {
        // hand the reference to half 0 (its O_1 stays in TMEM until half 0 read it)
        // racecheck: mbarrier handoff (released by merge_full; the next tile's write
        // waits on pv_done, which needs the o_free half 0 gives after reading it)
        sm1[r] = m;
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(merge_full);
        continue;
      }
      ptx::tc_fence_after();
      const uint32_t ob0 = tmem + lrow + O_COL, ob1 = ob0 + FA_OSTR;
      float a0 = 1.f, a1 = 0.f;
      const bool two = nk1 > 0;
      if (two) {
        ptx::mbar_wait(merge_full, merges & 1);
        ++merges;
        ptx::tc_fence_after();
        // racecheck: mbarrier handoff (acquired by the merge_full wait)
        const float m1 = sm1[r];
        const float mm = fmaxf(m, m1);
        a0 = ptx::ex2(m - mm);
        a1 = ptx::ex2(m1 - mm);
      }
      uint32_t l0[16], l1[16];
      tmem_ld16(ob0 + 64, l0);
      if (two) tmem_ld16(ob1 + 64, l1);
      ptx::tmem_ld_wait();
      const float lt = two ? fmaf(a1, __uint_as_float(l1[0]), a0 * __uint_as_float(l0[0])) : __uint_as_float(l0[0]);
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      const float w0 = a0 * inv, w1 = a1 * inv;
      const int mrow = mt * FA_BM + r;
      uint4* dst = reinterpret_cast<uint4*>(a.out + static_cast<long long>(mrow) * a.o_srow +
                                            static_cast<long long>(head) * a.o_sh);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t o0[32], o1[32];
        ptx::tmem_ld32(ob0 + hh * 32, o0);
        if (two) ptx::tmem_ld32(ob1 + hh * 32, o1);
        ptx::tmem_ld_wait();
        if (mrow < a.M) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int k = 8 * c + 2 * e;
              float y0 = __uint_as_float(o0[k]) * w0, y1 = __uint_as_float(o0[k + 1]) * w0;
              if (two) {
                y0 = fmaf(__uint_as_float(o1[k]), w1, y0);
                y1 = fmaf(__uint_as_float(o1[k + 1]), w1, y1);
              }
              __nv_bfloat162 h = __floats2bfloat162_rn(y0, y1);
              w[e] = *reinterpret_cast<uint32_t*>(&h);
            }
            dst[hh * 4 + c] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(&o_free[0]);
        if (two) ptx::mbar_arrive(&o_free[1]);
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

cudaError_t attn_fused_launch(cudaStream_t s, FaArgs& a, long long units) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = static_cast<int>(units < num_sms() ? units : num_sms());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = la;
  cfg.numAttrs = a.pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, attn_fused_kernel, a);
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
  return attn_fused_launch(s, a, static_cast<long long>(a.H) * a.MT);
}

}  // namespace ac
