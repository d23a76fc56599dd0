// G1 / G2 / G4: persistent, warp-specialised tcgen05 GEMM for sm_100a.
//
//   warp 0     : TMA producer (one elected lane) - 4-D tiled loads, 128B swizzle
//   warp 1     : TMEM allocator + MMA issuer (one elected lane), tcgen05.mma kind::f16
//   warps 2..5 : epilogue - tcgen05.ld 32x32b -> fp32 epilogue -> 16-byte stores
//
// Pipelines: a STAGES-deep smem ring (full/empty mbarriers, tcgen05.commit frees
// a slot) and a double-buffered TMEM accumulator (tmem_full / tmem_empty), so
// the epilogue of tile i overlaps the MMAs of tile i+1.  Tiles are 128 x BN,
// K step 64 (one 128-byte swizzle row of bf16).  One CTA per SM, grid =
// min(#tiles, #SMs), static round-robin tile order.
//
// Causal QK^T (P:336 GPT prefill): tiles entirely above the diagonal are not
// enumerated.  Causal PV: the K loop of an M tile stops at the tile's last row
// and tiles are issued heaviest-first.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstring>
#include <mutex>

#include "epilogue.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace ac {

namespace {

// f2 scores: exponentials as packed bf16x2 ex2 (one instruction per pair) instead
// of fp32 ex2 + pack.  Measured slower on B200 (GPT scores 0.94 -> 1.04 ms), so off.
#ifndef AC_EX2_PACKED
#define AC_EX2_PACKED 0
#endif

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int EPI_WARPS = 8;  // two per TMEM lane quarter, alternating 64-column slabs
constexpr int MAX_MT = 2048;
// f2 scores (unbiased chains; the triangle chains' paired short-chunk kernel has no such
// split, so they stay on MUFU for chunk invariance): every F2_POLY_EVERY-th column pair of a
// full 32-column group takes 2^x from a polynomial on the FMA pipe instead of MUFU (0 = all
// MUFU; 4 measured faster alone, slower under the chunk-loop overlap on GPT)
#ifndef F2_STAGES
#define F2_STAGES 3
#endif
#ifndef F2_POLY_EVERY
#define F2_POLY_EVERY 0
#endif

struct alignas(64) GemmArgs {
  CUtensorMap ta;
  CUtensorMap tb;
  CUtensorMap tout;  // output map for the TMA-store epilogue (tma_store = 1)
  CUtensorMap tadd;  // MODE 1: map over the added bias tensor (add_tma = 1), box {64, 32}
  int add_tma;
  int tma_store;
  Epilogue ep;
  int M, N, K, B1, B2;
  int a_b1, a_b2, b_b1, b_b2;
  int causal_tiles, causal_k;
  long long k_row_off;
  int MT, NT;
  int tiles_per_batch_dense;
  int total_tiles_dense;
  int vec;  // 1: 8-wide vectorised epilogue (16-byte aux loads / stores) is legal
  int pair2;  // MODE 0, BN = 256: CTA pair (cta_group::2): a cluster of 2 CTAs runs M = 256 MMAs
  int lean; // TMA-store epilogue without aux tensors / activation (scale and causal only)
  int fuse; // fused softmax-normalised A operand (PV of the f2 path)
  const float2* fstats;
  int stats_smem;  // MODE 2: slab statistics staged into shared memory by the producer (16-slab ring)
  long long fst_sb1, fst_ss;
  // MODE 2 fixed split-K: K cut into granules of skgk k-blocks at fixed key
  // positions; one work unit per (tile, granule); multi-granule tiles leave fp32
  // partials in skpart and the last unit to finish sums them in granule order
  int skgk, skng;
  float* skpart;
  int* skcnt;
  float2* skml;  // split-K: per (unit, row) the granule's running (max, sum)
  int* sched;  // MODE 2: zero-initialised work counter for dynamic unit scheduling (null = round-robin)
  unsigned long long* trace;  // debug (AC_TRACE): per unit {cta, t_load0, t_tfull, t_done}
  char* etile;  // f2 pre-swizzled e tiles (GemmProblem::etile), null = tensor path
  int e_nkb;    // k-blocks per e-tile row
  // chunk-loop overlap (GemmProblem::pdl ...)
  int pdl_wait;
  int* done_cnt;
  int* done_epoch;
  int epoch, dep_epoch;
  int* tsched;  // MODE 1 / 3 dynamic tile counter
  int pair;     // MODE 2, BN = 32, M <= 64: work units are pairs of batches (two M = 64 MMAs)
  int* zero_word;   // MODE 1 / 3 / 4: zero_n words zeroed at kernel start (the PV's counters)
  int zero_n;
};

// epilogue staging: per epilogue warp a [32 rows][PITCH] fp32 slab; PITCH = 68
// keeps rows 16-byte aligned (float4 row writes are conflict-free per phase)
constexpr int PITCH = 68;

template <int BN, int MODE>
struct Cfg {
  // f2 scores (MODE 1): 16 epilogue warps (one 64-column slab each at BN = 256,
  // <= 112 registers) with a single 4 KB bf16 staging box per warp; K = head dim
  // is one or two k-blocks, so two smem stages suffice
  // f2 scores at BN = 128: 8 epilogue warps (one 64-column slab each) and two CTAs
  // per SM, whose tiles run out of phase (one CTA's max pass beside the other's
  // exponentials)
  static constexpr bool DUAL = MODE == 1 && BN == 128;
  static constexpr int EPI = DUAL ? 8 : (MODE == 1 || MODE == 3 || MODE == 4) ? 16 : MODE == 2 ? 4 : EPI_WARPS;
  static constexpr int MINB = DUAL ? 2 : 1;
  // f2 PV (MODE 2): producer, MMA, EPI = 4 scale warps (one per TMEM lane quarter)
  // and XEPI = 4 finish warps that take each unit's end (output epilogue, split-K
  // partials and merge) off them: 320 threads, <= 204 registers each
  static constexpr int XEPI = MODE == 2 ? 4 : 0;
  static constexpr int THREADS = 64 + 32 * (EPI + XEPI);
  // MODE 2: KBUF per-k-block TMEM accumulators of BN columns + one BN-column staging
  // buffer for the hand-over to the finish warps
  static constexpr int KBUF = MODE == 2 && BN == 64 ? 7 : 8;
  // f2 PV (MODE 2) stages no output in smem: its ring is 8 deep (one CTA must keep
  // ~8 x 24 KB of A/B tiles in flight to stream at full speed when few CTAs remain)
  // MODE 2: the statistics ring (SRING slots of 128 rows x (m2, l), 1 KB each)
  static constexpr int SRING = 16;
  static constexpr int EPI_BYTES = (MODE == 1 || MODE == 3 || MODE == 4) ? EPI * 4096 : MODE == 2 ? SRING * 1024 : EPI_WARPS * 32 * PITCH * 4;
  // f2 scores: one stage = one tile's Q and K blocks (K = head dim <= 64); a third stage
  // lets the producer run two tiles ahead of the MMA
  static constexpr int STAGES = (MODE == 1 && BN == 256) ? F2_STAGES
                                : (MODE == 1 || MODE == 3 || MODE == 4) ? 2 : MODE == 2 ? 8 : (BN >= 256 ? 3 : (BN >= 128 ? 4 : 5));
  static constexpr int A_BYTES = BM * BK * 2;
  // MODE 4 (paired 64-row tiles): each stage holds the B tiles of both tiles of a pair
  // MODE 4 (paired 64-row tiles) and the BN = 32 PV (pairs when M <= 64): each stage
  // holds the B tiles of both tiles of a pair
  static constexpr int B_TILE = BN * BK * 2;
  static constexpr int B_BYTES = (MODE == 4 || (MODE == 2 && BN == 32) ? 2 : 1) * B_TILE;
  static constexpr int SW = BN >= 64 ? 64 : 32;  // epilogue slab width (columns)
  static constexpr int TMEM_COLS = MODE == 2 ? 512
                                             : (2 * BN) <= 32 ? 32 : (2 * BN) <= 64 ? 64 : (2 * BN) <= 128 ? 128 : (2 * BN) <= 256 ? 256 : 512;
  static constexpr int SMEM = 1024 /*align slack*/ + STAGES * (A_BYTES + B_BYTES) + EPI_BYTES + 512 /*barriers*/ +
                              (MODE == 4 ? 0 : (MAX_MT + 1) * 4 + 16 + (MODE == 3 ? 16 * 8 + 8 : MODE == 2 ? 18 * 8 + 8 + 128 * 8 + 2 * SRING * 8 : 0));
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

__device__ __forceinline__ void decode_tile(const GemmArgs& a, const int* prefix, int tpb, int t,
                                            int& b1, int& b2, int& mt, int& nt, int& kb) {
  const int b = t / tpb;
  const int r = t - b * tpb;
  b1 = b / a.B2;
  b2 = b - b1 * a.B2;
  if (a.causal_tiles) {
    int lo = 0, hi = a.MT;  // find mt with prefix[mt] <= r < prefix[mt+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (prefix[mid] <= r) lo = mid; else hi = mid;
    }
    mt = lo;
    nt = r - prefix[lo];
  } else {
    mt = r / a.NT;
    nt = r - mt * a.NT;
  }
  int kend = a.K;
  if (a.causal_k) {
    mt = a.MT - 1 - mt;  // heaviest tiles first
    const long long e = a.k_row_off + static_cast<long long>(mt + 1) * BM;
    if (e < kend) kend = static_cast<int>(e);
  }
  kb = (kend + BK - 1) / BK;
}

// Incremental form of decode_tile for a CTA's static tile sequence t = cid,
// cid + ncl, ...: no integer division or binary search per tile (both showed up
// as ~20 % of the issue slots of the short-K f2 scores epilogue).
struct TileWalk {
  int b = 0, r = 0, mt = 0, lo = 0, hi = 0;
  bool started = false;
  __device__ __forceinline__ int row_end(const GemmArgs& a, const int* prefix, int m, int start) const {
    return a.causal_tiles ? prefix[m + 1] : start + a.NT;
  }
  __device__ __forceinline__ void next(const GemmArgs& a, const int* prefix, int tpb, int t, int ncl) {
    if (a.tsched) started = false;  // dynamic tiles: no fixed stride, decode afresh
    if (!a.causal_tiles) {
      // dense tiles: direct decode (stepping m-tile by m-tile costs ncl / NT
      // iterations per tile, 148 for a one-n-tile GEMM)
      b = t / tpb;
      r = t - b * tpb;
      mt = r / a.NT;
      lo = mt * a.NT;
      hi = lo + a.NT;
      return;
    }
    if (!started) {
      started = true;
      b = t / tpb;
      r = t - b * tpb;
      if (a.causal_tiles) {
        int l = 0, h = a.MT;
        while (h - l > 1) {
          const int mid = (l + h) >> 1;
          if (prefix[mid] <= r) l = mid; else h = mid;
        }
        mt = l;
        lo = prefix[l];
        hi = prefix[l + 1];
      } else {
        mt = r / a.NT;
        lo = mt * a.NT;
        hi = lo + a.NT;
      }
      return;
    }
    r += ncl;
    while (r >= tpb) {
      r -= tpb;
      ++b;
      mt = 0;
      lo = 0;
      hi = row_end(a, prefix, 0, 0);
    }
    while (r >= hi) {
      ++mt;
      lo = hi;
      hi = row_end(a, prefix, mt, lo);
    }
  }
  __device__ __forceinline__ void get(const GemmArgs& a, int& b1, int& b2, int& m, int& nt, int& kb) const {
    b1 = a.B2 == 1 ? b : b / a.B2;
    b2 = b - b1 * a.B2;
    nt = r - lo;
    m = mt;
    int kend = a.K;
    if (a.causal_k) {
      m = a.MT - 1 - m;  // heaviest tiles first
      const long long e = a.k_row_off + static_cast<long long>(m + 1) * BM;
      if (e < kend) kend = static_cast<int>(e);
    }
    kb = (kend + BK - 1) / BK;
  }
};

// MODE 2 work units: (tile, granule) pairs, tile order as decode_tile (one n-tile,
// heaviest m-tiles first under causal_k).  prefix[r] = first unit of the r-th
// tile of a batch (causal_k), else ng = skng units per tile.
__device__ __forceinline__ void decode_unit(const GemmArgs& a, const int* prefix, int upb, int u, int& b1, int& b2,
                                            int& mt, int& kbn, int& klo, int& khi, int& g, int& ng, int& tile,
                                            int& unit0) {
  const int pu = u / upb;
  const int v = u - pu * upb;
  const int b = a.pair ? 2 * pu : pu;  // pairs: the pair's first batch
  b1 = b / a.B2;
  b2 = b - b1 * a.B2;
  int r;
  if (a.causal_k) {
    int lo = 0, hi = a.MT;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (prefix[mid] <= v) lo = mid; else hi = mid;
    }
    r = lo;
    g = v - prefix[r];
    ng = prefix[r + 1] - prefix[r];
    mt = a.MT - 1 - r;
  } else {
    r = v / a.skng;
    g = v - r * a.skng;
    ng = a.skng;
    mt = r;
  }
  int kend = a.K;
  if (a.causal_k) {
    const long long e = a.k_row_off + static_cast<long long>(mt + 1) * BM;
    if (e < kend) kend = static_cast<int>(e);
  }
  kbn = (kend + BK - 1) / BK;
  klo = g * a.skgk;
  khi = klo + a.skgk < kbn ? klo + a.skgk : kbn;
  tile = b * a.MT + r;
  unit0 = u - g;
}

// one MODE 2 work unit as seen by the thread owning TMEM lane (quarter, lane): its
// output row m (pairs: lanes 0-15 the pair's first batch, 16-31 its second) and batch
struct PvUnit {
  int b1, b2, mt, kbn, klo, khi, g, ng, tile, unit0, m;
  bool mv;
  long long bb;
};
__device__ __forceinline__ void pv_unit(const GemmArgs& a, const int* prefix, int upb, int t, int quarter, int lane,
                                        PvUnit& u) {
  decode_unit(a, prefix, upb, t, u.b1, u.b2, u.mt, u.kbn, u.klo, u.khi, u.g, u.ng, u.tile, u.unit0);
  u.m = a.pair ? quarter * 16 + (lane & 15) : u.mt * BM + quarter * 32 + lane;
  if (a.pair && lane >= 16) {
    const int nb = u.b1 * a.B2 + u.b2 + 1;
    u.b1 = nb / a.B2;
    u.b2 = nb - u.b1 * a.B2;
  }
  u.mv = u.m < a.M && u.b1 < a.B1;
  u.bb = static_cast<long long>(u.b1) * a.B2 + u.b2;
}

// MODE: 0 generic; 1 f2 scores (QK^T -> e = exp(s - m_slab) + slab statistics,
// lean TMA-store epilogue only); 2 f2 PV (A tile e rescaled to P in shared
// memory by all epilogue warps, which also run the output epilogue)
template <int BN, int MODE, bool PAIR>
__device__ __forceinline__ void gemm_tc_body(const GemmArgs& a) {
  using C = Cfg<BN, MODE>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // aligned by pointer arithmetic on the shared array (an integer round trip would
  // turn every later access into a generic LD / ST)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  float* sEpi = reinterpret_cast<float*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES + C::EPI_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* ready = tempty + 11;      // fused softmax: A tile transformed S -> P (<= 8 stages)
  // MODE 2 unit queue: the producer picks the next work unit (dynamically from the
  // sched counter when given, else round-robin) and hands it to the other roles
  // through a 4-deep ring (uq_full: 1 arrival, uq_empty: one per consuming warp)
  uint64_t* uq_full = tempty + 19;
  uint64_t* uq_empty = tempty + 23;
  // slot = 8 ints: the unit, and for MODE 1 / 3 its decoded tile (TileWalk b, r, mt, lo, hi),
  // so the consuming warps do not each decode it (integer division + binary search)
  int* uq_slot = reinterpret_cast<int*>(tempty + 27);
  int* prefix = reinterpret_cast<int*>(tempty + 43);  // 2 * STAGES + 47 words, MODE 2: + 18 + 1 + 128
  // MODE 1 bias boxes: one mbarrier per epilogue warp, after the prefix table
  uint64_t* bbar = MODE == 4 ? reinterpret_cast<uint64_t*>(prefix)
                             : reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(prefix + MAX_MT + 2) +
                                                         ((8u - (ptx::smem_u32(prefix + MAX_MT + 2) & 7u)) & 7u));
  static_assert(C::STAGES <= 8, "barrier block layout");

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // CTA pair (MODE 0, BN = 256): both CTAs of a cluster walk the same tiles (tile rows in
  // 256-row units); rank r holds rows r * 128 .. +127 of A and of the accumulator and
  // B rows r * 128 .. +127 of the 256-wide n-tile; the leader (rank 0) issues the MMAs
  // (a compile-time false outside gemm_tc_pair_kernel: kernels that contain cta_group::2
  // instructions may only be launched as clusters once any such launch has run)
  const bool P2 = PAIR && MODE == 0 && BN == 256 && a.pair2 != 0;
  const uint32_t crank = P2 ? ptx::cluster_rank() : 0;
  const int cid = P2 ? blockIdx.x / 2 : blockIdx.x, ncl = P2 ? gridDim.x / 2 : gridDim.x;

  // --- tile table for causal QK^T: live n-tiles per m-tile, prefix-summed
  int tpb = a.tiles_per_batch_dense;
  if (a.causal_tiles) {
    for (int mt = threadIdx.x; mt < a.MT; mt += C::THREADS) {
      long long maxrow = static_cast<long long>(mt) * BM + BM - 1;
      if (maxrow > a.M - 1) maxrow = a.M - 1;
      const long long lastcol = a.ep.row_off + maxrow - a.ep.col_off;
      long long cnt = lastcol < 0 ? 0 : lastcol / BN + 1;
      if (cnt > a.NT) cnt = a.NT;
      prefix[mt + 1] = static_cast<int>(cnt);
    }
    __syncthreads();
    if (warp == 0) {
      int carry = 0;
      if (lane == 0) prefix[0] = 0;
      for (int base = 0; base < a.MT; base += 32) {
        const int i = base + lane;
        int v = i < a.MT ? prefix[i + 1] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += u;
        }
        if (i < a.MT) prefix[i + 1] = v + carry;
        carry += __shfl_sync(0xffffffffu, v, 31);
      }
    }
    __syncthreads();
    tpb = prefix[a.MT];
  }
  if constexpr (MODE == 2) {
    // units per batch: granules of every m-tile (prefix over the heaviest-first order)
    if (a.causal_k) {
      for (int r = threadIdx.x; r < a.MT; r += C::THREADS) {
        const int mt = a.MT - 1 - r;
        long long kend = a.k_row_off + static_cast<long long>(mt + 1) * BM;
        if (kend > a.K) kend = a.K;
        const int kbn = static_cast<int>((kend + BK - 1) / BK);
        prefix[r + 1] = (kbn + a.skgk - 1) / a.skgk;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        prefix[0] = 0;
        for (int r = 0; r < a.MT; ++r) prefix[r + 1] += prefix[r];
      }
      __syncthreads();
      tpb = prefix[a.MT];
    } else {
      tpb = a.MT * a.skng;
    }
  }
  // MODE 4 work unit = (pair of flattened batches 2p, 2p+1; n-tile)
  const int total = MODE == 4 ? ((a.B1 * a.B2 + 1) / 2) * a.NT
                                : (MODE == 2 && a.pair ? tpb * ((a.B1 * a.B2 + 1) / 2) : tpb * a.B1 * a.B2);
#ifdef AC_DEBUG_HANG
  if (blockIdx.x == 0 && threadIdx.x == 0)
    printf("gemm_tc<%d,%d> enter grid %d M %d N %d K %d B1 %d B2 %d total %d tpb %d etile %p\n", BN, MODE, gridDim.x, a.M,
           a.N, a.K, a.B1, a.B2, total, tpb, a.etile);
#endif

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&a.ta);
    ptx::prefetch_tmap(&a.tb);
    if (MODE == 3 || MODE == 4) ptx::prefetch_tmap(&a.tadd);
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], MODE == 2 ? (C::XEPI ? C::XEPI : 1) : (P2 ? 2 : 1) * C::EPI);
    }
    for (int s = 0; s < C::STAGES; ++s) ptx::mbar_init(&ready[s], 32 * C::EPI);
    if (MODE == 3 || MODE == 4)
      for (int w = 0; w < C::EPI; ++w) ptx::mbar_init(&bbar[w], 1);
    if (MODE == 2) {  // PV: kfull[8] (MMA commit), kempty[8] (4 scale warps), sfull, sempty (4 warps each)
      for (int w = 0; w < 18; ++w) ptx::mbar_init(&bbar[w], w < 8 ? 1 : 4);
      // statistics ring: stfull (producer's bulk load), stempty (4 scale warps)
      for (int w = 0; w < 2 * C::SRING; ++w) ptx::mbar_init(&bbar[18 + 128 + w], w < C::SRING ? 1 : 4);
    }
    for (int s = 0; s < 4; ++s) {
      ptx::mbar_init(&uq_full[s], 1);
      ptx::mbar_init(&uq_empty[s], 1 + C::EPI + C::XEPI);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    if (P2) ptx::tmem_alloc2<C::TMEM_COLS>(tmem_holder);
    else ptx::tmem_alloc<C::TMEM_COLS>(tmem_holder);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (P2) ptx::cluster_sync();  // the peer's barriers initialised before any remote arrive / commit
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // an epilogue warp is done with accumulator buffer `acc` (pair: tell the leader's MMA)
  auto acc_free = [&](int acc_) {
    if (P2) ptx::mbar_arrive_remote(ptx::map_remote(ptx::smem_u32(&tempty[acc_]), 0));
    else ptx::mbar_arrive(&tempty[acc_]);
  };
  // programmatic dependent launch: the prologue above overlapped the previous
  // kernel; wait for its results only when this kernel reads them, and let the
  // next kernel of the chunk loop be scheduled as SMs free up
  if (a.pdl_wait) ptx::griddep_wait();
  ptx::griddep_launch();

  if ((MODE == 1 || MODE == 3 || MODE == 4) && a.zero_word && blockIdx.x == 0)
    for (int z = threadIdx.x; z < a.zero_n; z += C::THREADS) a.zero_word[z] = 0;
  // unit sequence of this CTA: i-th unit (static round-robin, or the MODE 2 queue)
  // unit queue in use: MODE 2 always, MODE 1 / 3 with dynamic tiles
  const bool uq = MODE == 2 || (MODE != 0 && a.tsched != nullptr);
  auto produce = [&](int i) -> int {  // producer lane only
    if (uq) {
      const int sl = i & 3;
      int* sc = MODE == 2 ? a.sched : a.tsched;
      // dynamic: the first unit of every CTA is its own index (no atomic round trip at
      // the start of a launch), later ones come from the counter offset by the grid
      int u = !sc || i == 0 ? cid + i * ncl : ncl + atomicAdd(sc, 1);
      if (u > total) u = total;
      TileWalk w;
      if ((MODE == 1 || MODE == 3) && u < total) w.next(a, prefix, tpb, u, ncl);
      ptx::mbar_wait(&uq_empty[sl], ((i >> 2) & 1) ^ 1);
      volatile int* q = uq_slot + 8 * sl;
      q[0] = u;
      if (MODE == 1 || MODE == 3) {
        q[1] = w.b; q[2] = w.r; q[3] = w.mt; q[4] = w.lo; q[5] = w.hi;
      }
      ptx::mbar_arrive(&uq_full[sl]);
      return u;
    } else {
      return cid + i * ncl;
    }
  };
  auto take = [&](int i) -> int {  // whole consuming warp
    if (uq) {
      const int sl = i & 3;
      ptx::mbar_wait(&uq_full[sl], (i >> 2) & 1);
      const int u = uq_slot[8 * sl];
      __syncwarp();
      if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(&uq_empty[sl]);
      return u;
    } else {
      return cid + i * ncl;
    }
  };
  // MODE 1 / 3 consumers: the next tile, decoded (from the queue slot when tiles are
  // dynamic, else by the incremental walk)
  auto take_walk = [&](int i, TileWalk& w) -> int {
    if ((MODE == 1 || MODE == 3) && uq) {
      const int sl = i & 3;
      ptx::mbar_wait(&uq_full[sl], (i >> 2) & 1);
      const volatile int* q = uq_slot + 8 * sl;
      const int u = q[0];
      w.b = q[1]; w.r = q[2]; w.mt = q[3]; w.lo = q[4]; w.hi = q[5];
      __syncwarp();
      if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(&uq_empty[sl]);
      return u;
    }
    const int t = take(i);
    if (t < total) w.next(a, prefix, tpb, t, ncl);
    return t;
  };

  if (MODE == 4 && warp == 0) {
    // ------------------------------------------------------------ TMA producer, MODE 4:
    // two 64-row A tiles (box rows 64) and their two B tiles per stage
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const int Bt = a.B1 * a.B2;
      for (int i = 0, t = produce(0); t < total; t = produce(++i)) {
        const int pb = t / a.NT, nt = t - pb * a.NT;
        const int nb = 2 * pb + 1 < Bt ? 2 : 1;
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        ptx::mbar_expect_tx(&full[stage], nb * (C::A_BYTES / 2 + C::B_BYTES / 2));
        for (int q = 0; q < nb; ++q) {
          const int bb = 2 * pb + q, b1 = bb / a.B2, b2 = bb - (bb / a.B2) * a.B2;
          ptx::tma_load_4d(sA + stage * C::A_BYTES + q * (C::A_BYTES / 2), &a.ta, &full[stage], 0, 0,
                           a.a_b1 ? b1 : 0, a.a_b2 ? b2 : 0);
          ptx::tma_load_4d(sB + stage * C::B_BYTES + q * (C::B_BYTES / 2), &a.tb, &full[stage], 0, nt * BN,
                           a.b_b1 ? b1 : 0, a.b_b2 ? b2 : 0);
        }
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      TileWalk walk;
      const uint64_t epol = ptx::policy_evict_first();
      int ss = 0;          // MODE 2 statistics ring slot / phase
      uint32_t sph = 0;
      for (int i = 0, t = produce(0); t < total; t = produce(++i)) {
        int b1, b2, mt, nt = 0, kbn, klo, khi;
        if constexpr (MODE == 2) {
          int g, ng, tile, unit0;
          decode_unit(a, prefix, tpb, t, b1, b2, mt, kbn, klo, khi, g, ng, tile, unit0);
        } else {
          walk.next(a, prefix, tpb, t, ncl);
          walk.get(a, b1, b2, mt, nt, kbn);
          klo = 0;
          khi = kbn;
        }
        const int ac2 = a.a_b1 ? b1 : 0, ac3 = a.a_b2 ? b2 : 0;
        const int bc2 = a.b_b1 ? b1 : 0, bc3 = a.b_b2 ? b2 : 0;
        if (MODE == 2 && a.trace) {
          unsigned long long tnow;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
          a.trace[4 * t] = blockIdx.x;
          a.trace[4 * t + 1] = tnow;
        }
        const char* esrc = MODE == 2 && a.etile
                               ? a.etile + (static_cast<long long>(b1 * a.B2 + b2) * a.MT + mt) * a.e_nkb * 16384
                               : nullptr;
        // e-tile rows past M were never stored (short chunks, ragged tails): load only
        // the 32-row quarters that hold rows < M (the rest of the stage is stale and
        // feeds only accumulator rows that are never written out)
        int ebytes = C::A_BYTES;
        if (MODE == 2 && esrc) {
          const int rows = a.M - mt * BM;
          if (rows < BM) ebytes = ((rows + 31) / 32) * 4096;
        }
        // pairs: rows 0..63 of the second batch's e-tile go to the stage's upper half,
        // its V^T tile to the second B slot
        const bool two = MODE == 2 && a.pair && b1 * a.B2 + b2 + 1 < a.B1 * a.B2;
        const int pb1 = two ? (b1 * a.B2 + b2 + 1) / a.B2 : 0, pb2 = two ? (b1 * a.B2 + b2 + 1) - pb1 * a.B2 : 0;
        if (P2) {
          // pair: this CTA's 128 rows of A and 128 rows of B; both halves' bytes are
          // counted on the leader's full barrier (its expect_tx covers the pair)
          // the leader's barrier: this CTA's shared address with the pair's peer bit (bit 24 of
          // the shared window) cleared - the form the 2-SM TMA expects
          const uint32_t lead_full = ptx::smem_u32(full) & 0xFEFFFFFFu;
          for (int kb = klo; kb < khi; ++kb) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            if (crank == 0) ptx::mbar_expect_tx(&full[stage], 2 * (C::A_BYTES + C::B_TILE / 2));
            ptx::tma_load_4d_2sm(sA + stage * C::A_BYTES, &a.ta, lead_full + stage * 8, kb * BK,
                                 (2 * mt + static_cast<int>(crank)) * BM, ac2, ac3);
            ptx::tma_load_4d_2sm(sB + stage * C::B_BYTES, &a.tb, lead_full + stage * 8, kb * BK,
                                 nt * BN + static_cast<int>(crank) * (BN / 2), bc2, bc3);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
          continue;
        }
        for (int kb = klo; kb < khi; ++kb) {
          if (MODE == 2 && a.stats_smem) {
            // the slab's statistics of the tile's rows (< M, an even count) into the ring
            uint64_t* stfull = bbar + 18 + 128;
            const int rows = a.M - mt * BM < BM ? a.M - mt * BM : BM;
            ptx::mbar_wait(&stfull[C::SRING + ss], sph ^ 1);
            ptx::mbar_expect_tx(&stfull[ss], rows * 8);
            ptx::bulk_load(reinterpret_cast<uint8_t*>(sEpi) + ss * 1024,
                           a.fstats + static_cast<long long>(b1 * a.B2 + b2) * a.fst_sb1 +
                               static_cast<long long>(kb) * a.fst_ss + static_cast<long long>(mt) * BM,
                           rows * 8, &stfull[ss]);
            if (++ss == C::SRING) { ss = 0; sph ^= 1; }
          }
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_expect_tx(&full[stage], (two ? 2 : 1) * (ebytes + C::B_TILE));
          if (MODE == 2 && esrc) {
            // e-tiles are read once: L2 evict-first
            ptx::bulk_load_hint(sA + stage * C::A_BYTES, esrc + static_cast<long long>(kb) * 16384, ebytes,
                                &full[stage], epol);
          }
          else
            ptx::tma_load_4d(sA + stage * C::A_BYTES, &a.ta, &full[stage], kb * BK, mt * BM, ac2, ac3);
          ptx::tma_load_4d(sB + stage * C::B_BYTES, &a.tb, &full[stage], kb * BK, nt * BN, bc2, bc3);
          if (two) {
            ptx::bulk_load(sA + stage * C::A_BYTES + 8192,
                           esrc + (static_cast<long long>(a.MT) * a.e_nkb + kb) * 16384, ebytes, &full[stage]);
            ptx::tma_load_4d(sB + stage * C::B_BYTES + C::B_TILE, &a.tb, &full[stage], kb * BK, nt * BN,
                             a.b_b1 ? pb1 : 0, a.b_b2 ? pb2 : 0);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (MODE == 4 && warp == 1) {
    // ------------------------------------------------------------ MMA issuer, MODE 4: two
    // M = 64 MMAs per k-step; their accumulators interleave in TMEM (lanes 0-15 and
    // 16-31 of every 32-lane subpartition), so all four epilogue quarters get rows
    constexpr uint32_t IDESC64 = ptx::idesc_bf16(64, BN);
    const int Bt = a.B1 * a.B2;
    int stage = 0, acc = 0;
    uint32_t phase = 0, aphase = 0;
    for (int i = 0, t = take(0); t < total; t = take(++i)) {
      const int pb = t / a.NT;
      const int nb = 2 * pb + 1 < Bt ? 2 : 1;
      ptx::mbar_wait(&tempty[acc], aphase ^ 1);
      ptx::tc_fence_after();
      ptx::mbar_wait(&full[stage], phase);
      ptx::tc_fence_after();
      if (lane == 0) {
        const uint32_t d = tmem_base + acc * BN;
        for (int q = 0; q < nb; ++q) {
          const uint32_t sa = ptx::smem_u32(sA + stage * C::A_BYTES + q * (C::A_BYTES / 2));
          const uint32_t sb = ptx::smem_u32(sB + stage * C::B_BYTES + q * (C::B_BYTES / 2));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            ptx::mma_bf16(d + (static_cast<uint32_t>(16 * q) << 16), ptx::sdesc_sw128(sa + k * 32),
                          ptx::sdesc_sw128(sb + k * 32), IDESC64, k ? 1u : 0u);
        }
        ptx::mma_commit(&empty[stage]);
        ptx::mma_commit(&tfull[acc]);
      }
      __syncwarp();
      if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  } else if (warp == 1 && P2 && crank != 0) {
    // the pair's peer issues no MMAs (the leader's cta_group::2 MMAs use its smem halves)
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t IDESC = ptx::idesc_bf16(BM, BN);
    constexpr uint32_t IDESC2 = ptx::idesc_bf16(2 * BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t aphase = 0;
    int kbuf = 0;          // MODE 2 post-scale: next per-k-block TMEM buffer
    uint32_t kphase = 0;
    TileWalk walk;
    for (int i = 0, t = MODE == 2 ? take(0) : take_walk(0, walk); t < total;
         t = MODE == 2 ? take(++i) : take_walk(++i, walk)) {
      int b1, b2, mt, nt = 0, kbn, klo, khi;
      if constexpr (MODE == 2) {
        int g, ng, tile, unit0;
        decode_unit(a, prefix, tpb, t, b1, b2, mt, kbn, klo, khi, g, ng, tile, unit0);
      } else {
        walk.get(a, b1, b2, mt, nt, kbn);
        klo = 0;
        khi = kbn;
      }
      if constexpr (MODE == 2) {
        // post-scale PV: every k-block gets its own TMEM buffer (kb-th of 8, round
        // robin), accumulate = 0; the scale warps fold f_slab * (e V) into registers
        uint64_t* kfull = bbar;
        uint64_t* kempty = bbar + 8;
        const int np = a.pair && b1 * a.B2 + b2 + 1 < a.B1 * a.B2 ? 2 : 1;
        for (int kb = klo; kb < khi; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::mbar_wait(&kempty[kbuf], kphase ^ 1);
          ptx::tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = ptx::smem_u32(sA + stage * C::A_BYTES);
            const uint32_t sb = ptx::smem_u32(sB + stage * C::B_BYTES);
            const uint32_t dk = tmem_base + kbuf * BN;
            if (a.pair) {
              constexpr uint32_t IDESC64 = ptx::idesc_bf16(64, BN);
              for (int q = 0; q < np; ++q)
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                  ptx::mma_bf16(dk + (static_cast<uint32_t>(16 * q) << 16), ptx::sdesc_sw128(sa + q * 8192 + k * 32),
                                ptx::sdesc_sw128(sb + q * C::B_TILE + k * 32), IDESC64, k ? 1u : 0u);
            } else {
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                ptx::mma_bf16(dk, ptx::sdesc_sw128(sa + k * 32), ptx::sdesc_sw128(sb + k * 32), IDESC, k ? 1u : 0u);
            }
            ptx::mma_commit(&empty[stage]);
            ptx::mma_commit(&kfull[kbuf]);
          }
          __syncwarp();
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          if (++kbuf == C::KBUF) { kbuf = 0; kphase ^= 1; }
        }
        continue;
      }
      ptx::mbar_wait(&tempty[acc], aphase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d = tmem_base + acc * BN;
      for (int kb = klo; kb < khi; ++kb) {
        ptx::mbar_wait(MODE == 2 ? &ready[stage] : &full[stage], phase);
        ptx::tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = ptx::smem_u32(sA + stage * C::A_BYTES);
          const uint32_t sb = ptx::smem_u32(sB + stage * C::B_BYTES);
          if (MODE == 2 && a.pair) {
            // two M = 64 MMAs; their accumulators interleave in TMEM (lanes 0-15 / 16-31
            // of every subpartition)
            constexpr uint32_t IDESC64 = ptx::idesc_bf16(64, BN);
            const int np = b1 * a.B2 + b2 + 1 < a.B1 * a.B2 ? 2 : 1;
            for (int q = 0; q < np; ++q)
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                ptx::mma_bf16(d + (static_cast<uint32_t>(16 * q) << 16), ptx::sdesc_sw128(sa + q * 8192 + k * 32),
                              ptx::sdesc_sw128(sb + q * C::B_TILE + k * 32), IDESC64, (kb != klo || k != 0) ? 1u : 0u);
          } else if (P2) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              ptx::mma_bf16_2(d, ptx::sdesc_sw128(sa + k * 32), ptx::sdesc_sw128(sb + k * 32), IDESC2,
                              (kb != klo || k != 0) ? 1u : 0u);
          } else {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              ptx::mma_bf16(d, ptx::sdesc_sw128(sa + k * 32), ptx::sdesc_sw128(sb + k * 32), IDESC,
                              (kb != klo || k != 0) ? 1u : 0u);
            }
          }
          if (P2) ptx::mma_commit2(&empty[stage]);  // both CTAs' slots free
          else ptx::mma_commit(&empty[stage]);  // slot free once these MMAs have read smem
        }
        __syncwarp();
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) {  // accumulator ready (pair: in both CTAs)
        if (P2) ptx::mma_commit2(&tfull[acc]);
        else ptx::mma_commit(&tfull[acc]);
      }
      __syncwarp();
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // Each warp owns TMEM lanes (= tile rows) 32*quarter .. +31.  Per slab of SW
    // columns: tcgen05.ld (thread = row) -> fp32 staging in smem -> read back
    // transposed (lane = column pair) so that aux loads and output stores are
    // coalesced along n.
    const int ew = warp - 2;       // epilogue warp 0..7
    const int quarter = warp & 3;  // TMEM lane quarter (hardware: warp w reads lanes 32*(w%4)..)
    const int half = ew >> 2;      // which alternate slabs this warp handles
    float* stage = sEpi + ew * 32 * PITCH;
    constexpr int SW = C::SW;
    constexpr int NSLAB = BN / SW;
    int acc = 0;
    int sbuf = 0;
    uint32_t aphase = 0;
    uint32_t bphase = 0;  // MODE 3 bias-box barrier phase
    bool bias_pending = false;  // MODE 3: this warp's next bias box is already in flight
    if constexpr (MODE == 2) {
      // ---- f2 PV (post-scale, R19).  Warps 2-5 ("scale", thread = output row of
      // TMEM lane quarter warp % 4): every 64-key slab's product e_slab V_slab lands in
      // its own TMEM buffer (KBUF round robin); O += f_slab (e_slab V_slab) in fp32
      // registers, f_slab = 2^(m2_slab - M_run) against the row's running max (O and L
      // rescaled when it rises).  At a unit's end they hand (O, M_run, L) over through
      // a TMEM staging buffer + shared memory and go straight on with the next unit,
      // whose first statistics they already prefetched during the last slab block.
      // Warps 6-9 ("finish") run the unit end: o = O / L and the output epilogue, or,
      // split-K, the fp32 partial + (M, L) of the granule and, for the unit that
      // completes the tile, the in-order merge of its granules.
      uint64_t* kfull = bbar;
      uint64_t* kempty = bbar + 8;
      uint64_t* sfull = bbar + 16;   // staging written (4 scale warps)
      uint64_t* sempty = bbar + 17;  // staging read (4 finish warps)
      float2* sml = reinterpret_cast<float2*>(bbar + 18);  // (M_run, L) per row
      const uint32_t tstg = tmem_base + C::KBUF * BN;        // staging columns
      const float2 nost = make_float2(-CUDART_INF_F, 0.f);
      auto unit = [&](int t, PvUnit& u) { pv_unit(a, prefix, tpb, t, quarter, lane, u); };
      // slab kb's (m2, l) of the thread's row (float2 index b * sb1 + kb * ss + m)
      auto ldst = [&](const PvUnit& u, int kb) -> float2 {
        return __ldg(a.fstats + u.bb * a.fst_sb1 + static_cast<long long>(kb) * a.fst_ss + u.m);
      };
      if (warp < 6) {
        const bool lead = warp == 2;
        constexpr int PF = 4;  // slab statistics prefetched PF slabs ahead (next unit's included)
        const int r = quarter * 32 + lane;
        // statistics from the producer's shared-memory ring (no load latency on this warp),
        // else prefetched from global memory PF slabs ahead
        const bool sm = a.stats_smem != 0;
        uint64_t* stfull = bbar + 18 + 128;
        const float2* sst = reinterpret_cast<const float2*>(sEpi);
        int ss = 0;
        uint32_t sph = 0;
        int kbuf = 0;
        uint32_t kphase = 0, sphase = 0;
        int i = 0;
        int t = take(0);
        PvUnit u;
        float2 fr[PF];
        if (t < total) unit(t, u);
#pragma unroll
        for (int j = 0; j < PF; ++j) fr[j] = (!sm && t < total && u.mv && u.klo + j < u.khi) ? ldst(u, u.klo + j) : nost;
        while (t < total) {
          float Mr = -CUDART_INF_F, Lr = 0.f;
          float accv[BN];
#pragma unroll
          for (int c = 0; c < BN; ++c) accv[c] = 0.f;
          int tn = -1;
          PvUnit un;
          for (int kb0 = u.klo; kb0 < u.khi; kb0 += PF) {
            float2 nx[PF];
            if (kb0 + PF < u.khi) {
#pragma unroll
              for (int j = 0; j < PF; ++j) nx[j] = (!sm && u.mv && kb0 + PF + j < u.khi) ? ldst(u, kb0 + PF + j) : nost;
            } else {
              // last block of this unit: take the next unit now and prefetch its first
              // statistics behind this block's slabs
              tn = take(++i);
              if (tn < total) unit(tn, un);
#pragma unroll
              for (int j = 0; j < PF; ++j) nx[j] = (!sm && tn < total && un.mv && un.klo + j < un.khi) ? ldst(un, un.klo + j) : nost;
            }
#pragma unroll
            for (int j = 0; j < PF; ++j) {
              if (kb0 + j < u.khi) {
                ptx::mbar_wait(&kfull[kbuf], kphase);
                ptx::tc_fence_after();
                if (a.trace && lead && lane == 0 && kb0 == u.klo && j == 0) {
                  unsigned long long tnow;
                  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
                  a.trace[4 * t + 2] = tnow;
                }
                // the slab's e V product, 32 columns per TMEM load (the first load in
                // flight while f is formed; 32 live registers keep the warp under 168)
                const uint32_t tk = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + kbuf * BN;
                uint32_t v[32];
                ptx::tmem_ld32(tk, v);
                float2 st = fr[j];
                if (sm) {
                  ptx::mbar_wait(&stfull[ss], sph);
                  // racecheck: mbarrier handoff (bulk-loaded before stfull, freed by the stempty arrive)
                  st = u.mv ? sst[ss * 128 + r] : nost;
                  __syncwarp();
                  if (lane == 0) ptx::mbar_arrive(&stfull[C::SRING + ss]);
                  if (++ss == C::SRING) { ss = 0; sph ^= 1; }
                }
                // lazy reference (R19): O and L move to a new running max only when a slab's
                // m2 exceeds it by more than 8 (f <= 2^8), so a row rescales a few times, not
                // at every slab whose m2 sets a record (divergent over the warp's 32 rows)
                if (st.x > Mr + 8.f) {
                  const float cr = ptx::ex2(Mr - st.x);  // first slab: 2^-inf = 0, O and L are 0
                  Lr *= cr;
#pragma unroll
                  for (int c = 0; c < BN; ++c) accv[c] *= cr;
                  Mr = st.x;
                }
                const float f = st.x == -CUDART_INF_F ? 0.f : ptx::ex2(st.x - Mr);
                Lr = fmaf(st.y, f, Lr);
#pragma unroll
                for (int hh = 0; hh < BN / 32; ++hh) {
                  if (hh > 0) ptx::tmem_ld32(tk + hh * 32, v);
                  ptx::tmem_ld_wait();
#pragma unroll
                  for (int c = 0; c < 32; ++c) asm volatile("" : "+r"(v[c]));  // uses stay after the wait
                  if (u.mv) {
                    const uint64_t f2 = ptx::f32x2_splat(f);
#pragma unroll
                    for (int c = 0; c < 32; c += 2)  // FFMA2: same rounding as fmaf(f, v, acc)
                      ptx::fma2_acc(v[c], v[c + 1], f2, accv[hh * 32 + c], accv[hh * 32 + c + 1]);
                  }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&kempty[kbuf]);
                if (++kbuf == C::KBUF) { kbuf = 0; kphase ^= 1; }
              }
            }
#pragma unroll
            for (int j = 0; j < PF; ++j) fr[j] = nx[j];
          }
          if (tn < 0) {  // (a unit without slabs: nothing was prefetched)
            tn = take(++i);
            if (tn < total) unit(tn, un);
#pragma unroll
            for (int j = 0; j < PF; ++j) fr[j] = (tn < total && un.mv && un.klo + j < un.khi) ? ldst(un, un.klo + j) : nost;
          }
          if (a.trace && lead && lane == 0) {  // end of the unit's slab stream
            unsigned long long tnow;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
            a.trace[4 * t + 3] = tnow;
          }
          // hand over: O -> TMEM staging, (M_run, L) -> shared memory
          ptx::mbar_wait(sempty, sphase ^ 1);
          ptx::tc_fence_after();
#pragma unroll
          for (int hh = 0; hh < BN / 32; ++hh)
            ptx::tmem_st32(tstg + (static_cast<uint32_t>(quarter * 32) << 16) + hh * 32,
                           *reinterpret_cast<const uint32_t(*)[32]>(&accv[hh * 32]));
          // racecheck: mbarrier handoff (written after the sempty wait, read after sfull)
          sml[r] = make_float2(Mr, Lr);
          ptx::tmem_st_wait();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(sfull);
          sphase ^= 1;
          t = tn;
          u = un;
        }
      } else {
        const bool lead = warp == 6;
        const int r = quarter * 32 + lane;
        int* sk_old = prefix + MAX_MT + 1;  // counter value seen by this CTA (broadcast)
        uint32_t sphase = 0;
        for (int i = 0, t = take(0); t < total; t = take(++i)) {
          PvUnit u;
          unit(t, u);
          ptx::mbar_wait(sfull, sphase);
          ptx::tc_fence_after();
          float accv[BN];
#pragma unroll
          for (int hh = 0; hh < BN / 32; ++hh)
            ptx::tmem_ld32(tstg + (static_cast<uint32_t>(quarter * 32) << 16) + hh * 32,
                           *reinterpret_cast<uint32_t(*)[32]>(&accv[hh * 32]));
          // racecheck: mbarrier handoff (read after the sfull wait, freed by the sempty arrive)
          const float2 ml = sml[r];
          ptx::tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < BN; ++c) asm volatile("" : "+f"(accv[c]));
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(sempty);
          sphase ^= 1;
          const float Mr = ml.x, Lr = ml.y;
          const long long bb = u.bb;
          // chunk-loop overlap: once this unit's rows or partials are stored (and the
          // four finish warps are past their stores) the unit that completes the batch
          // publishes the chunk epoch (release, cumulative over the barrier)
          auto publish = [&]() {
            if (!a.done_cnt) return;
            asm volatile("bar.sync 2, 128;" ::: "memory");
            if (lead && lane == 0) {  // (lane 0: the pair's first batch; pairs count both)
              const int nq = a.pair && bb + 1 < static_cast<long long>(a.B1) * a.B2 ? 2 : 1;
              for (int q = 0; q < nq; ++q)
                if (ptx::atom_add_acqrel_gpu(a.done_cnt + bb + q, 1) == tpb - 1)
                  ptx::st_release_gpu(a.done_epoch + bb + q, a.epoch + 1);
            }
          };
          if (u.ng == 1) {
            const float il = Lr > 0.f ? 1.f / Lr : 0.f;
#pragma unroll
            for (int c = 0; c < BN; ++c) accv[c] *= il;
          } else {
            float* mine = a.skpart + (static_cast<long long>(u.unit0 + u.g) * BM + r) * BN;
#pragma unroll
            for (int q = 0; q < BN / 4; ++q)
              reinterpret_cast<float4*>(mine)[q] = make_float4(accv[4 * q], accv[4 * q + 1], accv[4 * q + 2], accv[4 * q + 3]);
            // this granule's O is relative to its own running max: keep (M, L) beside it
            a.skml[static_cast<long long>(u.unit0 + u.g) * BM + r] = make_float2(Mr, Lr);
            __threadfence();
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (lead && lane == 0) *sk_old = atomicAdd(a.skcnt + u.tile, 1);
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int old = *sk_old;
            asm volatile("bar.sync 1, 128;" ::: "memory");  // sk_old reusable
            if (old != u.ng - 1) {
              publish();
              continue;
            }
            __threadfence();
            // merge the granules in order: M = max M_g, O = sum 2^(M_g - M) O_g,
            // L = sum 2^(M_g - M) L_g, o = O / L (granules of masked keys only: M_g = -inf)
            const float4* base = reinterpret_cast<const float4*>(a.skpart + (static_cast<long long>(u.unit0) * BM + r) * BN);
            const float2* mlp = a.skml + static_cast<long long>(u.unit0) * BM + r;
            float Mt = -CUDART_INF_F;
            for (int gg = 0; gg < u.ng; ++gg) Mt = fmaxf(Mt, __ldcg(mlp + static_cast<long long>(gg) * BM).x);
#pragma unroll
            for (int c = 0; c < BN; ++c) accv[c] = 0.f;
            float Lt = 0.f;
            for (int gg = 0; gg < u.ng; ++gg) {
              const float2 mg = __ldcg(mlp + static_cast<long long>(gg) * BM);
              if (mg.x == -CUDART_INF_F) continue;
              const float w = ptx::ex2(mg.x - Mt);
              Lt = fmaf(mg.y, w, Lt);
              const float4* pp = base + static_cast<long long>(gg) * BM * BN / 4;
#pragma unroll
              for (int q = 0; q < BN / 4; ++q) {
                const float4 v4 = __ldcg(pp + q);
                accv[4 * q] = fmaf(w, v4.x, accv[4 * q]); accv[4 * q + 1] = fmaf(w, v4.y, accv[4 * q + 1]);
                accv[4 * q + 2] = fmaf(w, v4.z, accv[4 * q + 2]); accv[4 * q + 3] = fmaf(w, v4.w, accv[4 * q + 3]);
              }
            }
            const float il = Lt > 0.f ? 1.f / Lt : 0.f;
#pragma unroll
            for (int c = 0; c < BN; ++c) accv[c] *= il;
            if (lead && lane == 0) a.skcnt[u.tile] = 0;  // ready for the next launch
          }
          if (u.mv) {
#pragma unroll
            for (int hh = 0; hh < BN / 32; ++hh) {
              const int n = hh * 32;
              if (n >= a.N) break;
              uint32_t pk[16];
              epilogue_row32(a.ep, u.b1, u.b2, u.m, n, true, *reinterpret_cast<const uint32_t(*)[32]>(&accv[hh * 32]),
                             pk, a.N - n);
              uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.ep.out) +
                                                  static_cast<long long>(u.b1) * a.ep.out_sb1 +
                                                  static_cast<long long>(u.b2) * a.ep.out_sb2 +
                                                  static_cast<long long>(u.m) * a.ep.out_sm + n);
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (8 * q < a.N - n) o[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
            }
          }
          publish();
        }
      }
    } else if constexpr (MODE == 4) {
      // ---- paired f2 triangle scores for short chunks (M <= 64, R20): thread =
      // (row quarter*16 + lane%16) of the pair's first tile (lanes 0-15) or second
      // tile (lanes 16-31); one 64-column slab per warp.  Bias boxes [16 rows x 64]
      // per tile of the pair land in the warp's staging box, e is packed into it and
      // leaves as two 2 KB bulk stores (16 e-tile rows per tile).
      constexpr float L2E = 1.4426950408889634f;
      const int ew = warp - 2;
      const int quarter = warp & 3;
      const int c = ew >> 2;
      const int sel = lane >> 4;
      const int Bt = a.B1 * a.B2;
      uint8_t* sb = reinterpret_cast<uint8_t*>(sEpi) + ew * 4096;
      const float sc = a.ep.scale * L2E;
      int acc = 0;
      uint32_t aphase = 0, bph = 0;
      int dep_ok_pb = -1;  // last pair whose predecessor PV is known finished
      for (int i = 0, t = take(0); t < total; t = take(++i)) {
        const int pb = t / a.NT, nt = t - pb * a.NT;
        const int nb = 2 * pb + 1 < Bt ? 2 : 1;
        const int bb = 2 * pb + sel;
        const int n0 = nt * BN + c * 64;
        const int m = quarter * 16 + (lane & 15);
        const bool live = quarter * 16 < a.M;  // warp-uniform
        const bool mvalid = live && bb < Bt && m < a.M;
        ptx::mbar_wait(&tfull[acc], aphase);
        ptx::tc_fence_after();
        if (live) {
          if (lane == 0) {
            ptx::bulk_wait_read<0>();  // the previous e store has read the staging box
            ptx::mbar_expect_tx(&bbar[ew], nb * 2048);
            for (int q = 0; q < nb; ++q) {
              const int qb = 2 * pb + q, q1 = qb / a.B2, q2 = qb - (qb / a.B2) * a.B2;
              ptx::tma_load_4d(sb + q * 2048, &a.tadd, &bbar[ew], n0, quarter * 16, a.ep.add_sb1 ? q1 : 0,
                               a.ep.add_sb2 ? q2 : 0);
            }
          }
          __syncwarp();
          ptx::mbar_wait(&bbar[ew], bph);
          bph ^= 1;
          long long lim = a.N - 1 - n0;
          const uint32_t ta = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN + c * 64;
          uint32_t r[32];
          auto load_x = [&](int hh) {
            ptx::tmem_ld32(ta + hh * 32, r);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t addr = ptx::smem_u32(sb + lane * 128 + (((hh * 4 + q) ^ (lane & 7)) * 16));
              uint32_t w[4];
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                           : "r"(addr));
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 bf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
                r[8 * q + 2 * e] = __float_as_uint(fmaf(__uint_as_float(r[8 * q + 2 * e]), sc, bf.x * L2E));
                r[8 * q + 2 * e + 1] = __float_as_uint(fmaf(__uint_as_float(r[8 * q + 2 * e + 1]), sc, bf.y * L2E));
              }
            }
          };
          // biased redo path: the box holds e by then, so the bias comes from global memory
          auto load_x_gbias = [&](int hh) {
            ptx::tmem_ld32(ta + hh * 32, r);
            ptx::tmem_ld_wait();
            const int q1 = bb / a.B2, q2 = bb - (bb / a.B2) * a.B2;
            const __nv_bfloat16* brow = static_cast<const __nv_bfloat16*>(a.ep.add) +
                                        (a.ep.add_sb1 ? static_cast<long long>(q1) * a.ep.add_sb1 : 0) +
                                        (a.ep.add_sb2 ? static_cast<long long>(q2) * a.ep.add_sb2 : 0) +
                                        static_cast<long long>(mvalid ? m : 0) * a.ep.add_sm + n0 + hh * 32;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint32_t w[4] = {0u, 0u, 0u, 0u};
              const int n = n0 + hh * 32 + 8 * q;
              if (mvalid && n + 8 <= a.N) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(brow + 8 * q));
                w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
              } else if (mvalid) {
                __nv_bfloat16 h[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) h[e] = n + e < a.N ? brow[8 * q + e] : __float2bfloat16(0.f);
                memcpy(w, h, 16);
              }
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 bf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
                r[8 * q + 2 * e] = __float_as_uint(fmaf(__uint_as_float(r[8 * q + 2 * e]), sc, bf.x * L2E));
                r[8 * q + 2 * e + 1] = __float_as_uint(fmaf(__uint_as_float(r[8 * q + 2 * e + 1]), sc, bf.y * L2E));
              }
            }
          };
          float l0 = 0.f, l1 = 0.f;
          auto emit = [&](int hh, float mref) {
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float e0 = hh * 32 + 2 * j <= lim ? ptx::ex2(__uint_as_float(r[2 * j]) - mref) : 0.f;
              const float e1 = hh * 32 + 2 * j + 1 <= lim ? ptx::ex2(__uint_as_float(r[2 * j + 1]) - mref) : 0.f;
              l0 += e0;
              l1 += e1;
              __nv_bfloat162 h = __floats2bfloat162_rn(e0, e1);
              pk[j] = *reinterpret_cast<uint32_t*>(&h);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int ch = hh * 4 + q;
              const uint32_t addr = ptx::smem_u32(sb + lane * 128 + ((ch ^ (lane & 7)) * 16));
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pk[4 * q]),
                           "r"(pk[4 * q + 1]), "r"(pk[4 * q + 2]), "r"(pk[4 * q + 3])
                           : "memory");
            }
          };
          // one TMEM pass, reference = the slab's first score x0 (R19, as the 128-row
          // kernel: same x, same reference, same redo rule, so a row's e and statistics are
          // bitwise those of the unpaired kernel in any chunking)
          load_x(0);
          float mref = lim >= 0 ? __uint_as_float(r[0]) : 0.f;
          emit(0, mref);
          load_x(1);
          emit(1, mref);
          const bool redo = lim >= 0 && !(l0 + l1 <= 0x1p96f);
          const bool any_redo = __any_sync(0xffffffffu, redo);
          if (!any_redo) {
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) acc_free(acc);
          } else {
            float mx = -CUDART_INF_F;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              load_x_gbias(hh);
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (hh * 32 + j <= lim) mx = fmaxf(mx, __uint_as_float(r[j]));
            }
            if (redo) {
              mref = mx;
              l0 = l1 = 0.f;
            }
            load_x_gbias(0);
            if (redo) emit(0, mref);
            load_x_gbias(1);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) acc_free(acc);
            if (redo) emit(1, mref);
          }
          const float mx = lim >= 0 ? mref : -CUDART_INF_F;
          if (a.done_epoch && pb != dep_ok_pb) {
            // chunk-loop overlap: the previous chunk's PV must be done with both batches
            if (lane == 0) {
              for (int q = 0; q < nb; ++q)
                ptx::wait_geq_gpu(a.done_epoch + 2 * pb + q, a.dep_epoch);
              ptx::fence_proxy_async_global();
            }
            __syncwarp();
            dep_ok_pb = pb;
          }
          if (mvalid && n0 < a.N)
            a.ep.stats[static_cast<long long>(bb) * a.ep.stats_sb1 + static_cast<long long>(n0 / 64) * a.ep.stats_ss + m] =
                make_float2(mx, l0 + l1);
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && n0 < a.N) {
            for (int q = 0; q < nb; ++q) {
              char* dst = a.etile + ((static_cast<long long>(2 * pb + q) * a.MT) * a.e_nkb + n0 / 64) * 16384 +
                          quarter * 2048;
              ptx::bulk_store(dst, sb + q * 2048, 2048);
            }
            ptx::bulk_commit();
          }
        } else {
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) acc_free(acc);
        }
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
      if (lane == 0) ptx::bulk_wait_read<0>();
      __syncwarp();
    } else {
    TileWalk walk;
    int dep_ok_b = -1;  // MODE 1 / 3: last batch whose predecessor PV is known finished
    for (int i = 0, t = take_walk(0, walk); t < total; t = take_walk(++i, walk)) {
      int b1, b2, mt, nt, kbn;
      walk.get(a, b1, b2, mt, nt, kbn);
      ptx::mbar_wait(&tfull[acc], aphase);
      ptx::tc_fence_after();
      if (half >= NSLAB) {  // narrow tile: nothing for this warp, but keep the tempty count
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) acc_free(acc);
        if (++acc == 2) { acc = 0; aphase ^= 1; }
        continue;
      }
      const int m0 = (P2 ? 2 * mt + static_cast<int>(crank) : mt) * BM + quarter * 32;
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = half; c < NSLAB; c += C::EPI / 4) {
        const bool last = c + C::EPI / 4 >= NSLAB;
        const int n0 = nt * BN + c * SW;
        if constexpr (MODE == 1 || MODE == 3) {
          // MODE 3 = MODE 1 plus an added bias tensor (the AlphaFold triangle bias,
          // AF2 Alg. 13 line 5): compiled separately so the plain f2 scores keep
          // their register budget
          constexpr bool BIASED = MODE == 3;
          uint8_t* sb = reinterpret_cast<uint8_t*>(sEpi) + ew * 4096;
          if (m0 >= a.M) {  // quarter entirely past M (short chunk): nothing to compute or store
            if (last) {
              ptx::tc_fence_before();
              __syncwarp();
              if (lane == 0) acc_free(acc);
            }
            continue;
          }
          // ---- f2 scores, one 64-column slab: x = acc * scale * log2(e) (fp32,
          // scale > 0 so the max is taken on the raw accumulator) or, biased,
          // x = (acc * scale + b) * log2(e); the slab max m2, stored
          // e = bf16(2^(x - m2)), statistics (m2, fp32 sum of e).  Two TMEM passes
          // (max, then exponentials) keep 32 accumulators live at a time.
          constexpr float L2E = 1.4426950408889634f;
          if (lane == 0) {
            if (!BIASED || !bias_pending) ptx::bulk_wait_read<0>();  // previous store has read the staging box
            if (BIASED && !bias_pending) {
              // the slab's bias box [32 rows x 64 cols] (TMA, 128B-swizzled) lands in the
              // staging box; rows are read back per thread from shared memory
              ptx::mbar_expect_tx(&bbar[ew], 4096);
              ptx::tma_load_4d(sb, &a.tadd, &bbar[ew], n0, m0, a.ep.add_sb1 ? b1 : 0, a.ep.add_sb2 ? b2 : 0);
            }
          }
          __syncwarp();
          if constexpr (BIASED) {
            ptx::mbar_wait(&bbar[ew], bphase);
            bphase ^= 1;
            bias_pending = false;
          }
          const int m = m0 + lane;
          const bool mvalid = m < a.M;
          long long lim64 = a.ep.causal ? (a.ep.row_off + m - a.ep.col_off - n0) : (1ll << 40);
          if (lim64 > a.N - 1 - n0) lim64 = a.N - 1 - n0;  // columns past N are masked (and clipped by the store)
          const int lim = lim64 < -1 ? -1 : static_cast<int>(lim64);  // only lim < 0 / lim >= j matter
          const uint32_t ta = tbase + c * SW;
          // biased: registers hold x itself after the add (unit multiplier below)
          const float cl = BIASED ? 1.f : a.ep.scale * L2E;
          // x for the 32 columns hh*32.. of this row (biased: bias chunks from the box)
          auto load_x = [&](int hh, uint32_t (&r)[32]) {
            ptx::tmem_ld32(ta + hh * 32, r);
            ptx::tmem_ld_wait();
            if constexpr (BIASED) {
              // x = fmaf(acc, scale log2e, b log2e) on packed pairs (FMUL2 + FFMA2: per lane
              // the scalar roundings of the paired kernel); bf16 -> f32 by bit shifts
              const uint64_t sc2 = f2_splat(a.ep.scale * L2E), l2e2 = f2_splat(L2E);
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t addr = ptx::smem_u32(sb + lane * 128 + (((hh * 4 + q) ^ (lane & 7)) * 16));
                uint32_t w[4];
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                             : "r"(addr));
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const uint64_t b2 = f2_pack(__uint_as_float(w[e] << 16), __uint_as_float(w[e] & 0xffff0000u));
                  const uint64_t x2 = f2_fma(f2_pack(__uint_as_float(r[8 * q + 2 * e]), __uint_as_float(r[8 * q + 2 * e + 1])),
                                             sc2, f2_mul(b2, l2e2));
                  float x0, x1;
                  f2_unpack(x2, x0, x1);
                  r[8 * q + 2 * e] = __float_as_uint(x0);
                  r[8 * q + 2 * e + 1] = __float_as_uint(x1);
                }
              }
            }
          };
          // biased redo path: the staging box already holds this slab's e chunks, so the
          // bias comes from global memory (L2) - the same bf16 values, the same arithmetic
          auto load_x_gbias = [&](int hh, uint32_t (&r)[32]) {
            ptx::tmem_ld32(ta + hh * 32, r);
            ptx::tmem_ld_wait();
            if constexpr (BIASED) {
              const float sc = a.ep.scale * L2E;
              const __nv_bfloat16* brow = static_cast<const __nv_bfloat16*>(a.ep.add) +
                                          (a.ep.add_sb1 ? static_cast<long long>(b1) * a.ep.add_sb1 : 0) +
                                          (a.ep.add_sb2 ? static_cast<long long>(b2) * a.ep.add_sb2 : 0) +
                                          static_cast<long long>(mvalid ? m : 0) * a.ep.add_sm + n0 + hh * 32;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                uint32_t w[4] = {0u, 0u, 0u, 0u};
                const int n = n0 + hh * 32 + 8 * q;
                if (mvalid && n + 8 <= a.N) {
                  const uint4 v = __ldg(reinterpret_cast<const uint4*>(brow + 8 * q));
                  w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
                } else if (mvalid) {
                  __nv_bfloat16 h[8];
#pragma unroll
                  for (int e = 0; e < 8; ++e) h[e] = n + e < a.N ? brow[8 * q + e] : __float2bfloat16(0.f);
                  memcpy(w, h, 16);
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 bf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
                  r[8 * q + 2 * e] = __float_as_uint(fmaf(__uint_as_float(r[8 * q + 2 * e]), sc, bf.x * L2E));
                  r[8 * q + 2 * e + 1] = __float_as_uint(fmaf(__uint_as_float(r[8 * q + 2 * e + 1]), sc, bf.y * L2E));
                }
              }
            }
          };
          uint32_t r[32];
          float mx = -CUDART_INF_F;
          float l0 = 0.f, l1 = 0.f;
          float m2;
          // exponentials of the 32 columns hh*32.. in r against reference mref, packed into
          // the staging box (chunks hh*4..hh*4+3 of this thread's row)
          auto emit = [&](int hh, float mref, float& s0, float& s1) {
            uint32_t pk[16];
            if (lim >= hh * 32 + 31) {
              const uint64_t cl2 = ptx::f32x2_splat(cl), nm2 = ptx::f32x2_splat(-mref);
              uint64_t sp = f2_pack(s0, s1);  // (s0, s1) summed as one FADD2 per pair: same rounding
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                float x0, x1;
                if constexpr (!BIASED) {  // one FFMA2 per column pair (same rounding as fmaf)
                  ptx::fma2(r[2 * j], r[2 * j + 1], cl2, nm2, x0, x1);
                } else {  // x - mref as one FADD2 (= fmaf(x, 1, -mref) per lane)
                  f2_unpack(f2_add(f2_pack(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1])), nm2), x0, x1);
                }
                // one column pair in F2_POLY_EVERY on the FMA pipe (the MUFU pipe saturates
                // while the warps exponentiate; columns fixed, so chunking changes nothing)
                float e0, e1;
                if (!BIASED && F2_POLY_EVERY > 0 && j % (F2_POLY_EVERY > 0 ? F2_POLY_EVERY : 1) == F2_POLY_EVERY - 1) {
                  ptx::exp2_poly2(x0, x1, e0, e1);
                } else {
                  e0 = ptx::ex2(x0);
                  e1 = ptx::ex2(x1);
                }
                sp = f2_add(sp, f2_pack(e0, e1));
                __nv_bfloat162 h = __floats2bfloat162_rn(e0, e1);
                pk[j] = *reinterpret_cast<uint32_t*>(&h);
              }
              f2_unpack(sp, s0, s1);
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float e0 = hh * 32 + 2 * j <= lim ? ptx::ex2(fmaf(__uint_as_float(r[2 * j]), cl, -mref)) : 0.f;
                const float e1 = hh * 32 + 2 * j + 1 <= lim ? ptx::ex2(fmaf(__uint_as_float(r[2 * j + 1]), cl, -mref)) : 0.f;
                s0 += e0;
                s1 += e1;
                __nv_bfloat162 h = __floats2bfloat162_rn(e0, e1);
                pk[j] = *reinterpret_cast<uint32_t*>(&h);
              }
            }
            // (biased: this row's bias chunks hh*4.. were read above; the e chunks
            // overwrite exactly those, in this thread's own row)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int ch = hh * 4 + q;
              const uint32_t addr = ptx::smem_u32(sb + lane * 128 + ((ch ^ (lane & 7)) * 16));
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pk[4 * q]),
                           "r"(pk[4 * q + 1]), "r"(pk[4 * q + 2]), "r"(pk[4 * q + 3])
                           : "memory");
            }
          };
          auto slab_max = [&](int hh) {
            float q0 = -CUDART_INF_F, q1 = -CUDART_INF_F, q2 = -CUDART_INF_F, q3 = -CUDART_INF_F;
            if (lim >= hh * 32 + 31) {
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                q0 = fmaxf(q0, __uint_as_float(r[j])); q1 = fmaxf(q1, __uint_as_float(r[j + 1]));
                q2 = fmaxf(q2, __uint_as_float(r[j + 2])); q3 = fmaxf(q3, __uint_as_float(r[j + 3]));
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (hh * 32 + j <= lim) q0 = fmaxf(q0, __uint_as_float(r[j]));
            }
            mx = fmaxf(mx, fmaxf(fmaxf(q0, q1), fmaxf(q2, q3)));
          };
          {
            // one TMEM pass (reading R19, plain and biased chains alike): the slab's reference is its first score x0
            // (column 0 is valid whenever any column is: masks are suffixes), so the
            // exponentials need no slab max; a row whose sum of 2^(x - x0) exceeds 2^96
            // (its max exceeds x0 by more than 96, or nearly so) is redone against its
            // max in a second TMEM pass (warp-collective reloads, the decision per row:
            // results depend only on the row's own data)
            load_x(0, r);
            float mref = lim >= 0 ? __uint_as_float(r[0]) * cl : 0.f;
            emit(0, mref, l0, l1);
            load_x(1, r);
            emit(1, mref, l0, l1);
            const bool redo = lim >= 0 && !(l0 + l1 <= 0x1p96f);
            const bool any_redo = __any_sync(0xffffffffu, redo);
            if (!any_redo && last) {
              ptx::tc_fence_before();
              __syncwarp();
              if (lane == 0) acc_free(acc);
            }
            if (any_redo) {
              // (biased: the bias from global memory, the box now holds e)
              auto reload = [&](int hh) {
                if constexpr (BIASED) load_x_gbias(hh, r);
                else load_x(hh, r);
              };
              reload(0);
              slab_max(0);
              reload(1);
              slab_max(1);
              if (redo) {
                mref = mx * cl;
                l0 = l1 = 0.f;
              }
              reload(0);
              if (redo) emit(0, mref, l0, l1);
              reload(1);
              if (last) {
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) acc_free(acc);
              }
              if (redo) emit(1, mref, l0, l1);
            }
            m2 = lim >= 0 ? mref : -CUDART_INF_F;
          }
          if (a.done_epoch) {
            // chunk-loop overlap: the previous chunk's PV must have finished reading this
            // batch's e-tiles and statistics before they are overwritten
            const int bb = b1 * a.B2 + b2;
            if (bb != dep_ok_b) {
              if (lane == 0) {
                ptx::wait_geq_gpu(a.done_epoch + bb, a.dep_epoch);
                ptx::fence_proxy_async_global();
              }
              __syncwarp();
              dep_ok_b = bb;
            }
          }
          if (mvalid && n0 < a.N)
            a.ep.stats[static_cast<long long>(b1 * a.B2 + b2) * a.ep.stats_sb1 +
                       static_cast<long long>(n0 / 64) * a.ep.stats_ss + m] = make_float2(m2, l0 + l1);
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (a.etile) {
              // (slabs past N would land in the next tile row: not stored)
              char* dst = a.etile + ((static_cast<long long>(b1 * a.B2 + b2) * a.MT + mt) * a.e_nkb + n0 / 64) * 16384 +
                          quarter * 4096;
              if (n0 < a.N && m0 < a.M) {  // quarters past M: never read
                ptx::bulk_store_hint(dst, sb, 4096, ptx::policy_evict_first());  // e-tiles: L2 evict-first
              }
            } else {
              ptx::tma_store_4d(&a.tout, sb, n0, m0, b1, b2);
            }
            ptx::bulk_commit();
            if constexpr (BIASED) {
              // prefetch the bias box of this warp's slab in the CTA's next tile (same
              // slab index c) as soon as the store has read the staging box, so its L2
              // latency overlaps the next accumulator's MMA
              const int tn = t + ncl;
              if (tn < total && last && !a.tsched) {
                TileWalk w2 = walk;
                w2.next(a, prefix, tpb, tn, ncl);
                int nb1, nb2, nmt, nnt, nkb;
                w2.get(a, nb1, nb2, nmt, nnt, nkb);
                const int nm0 = nmt * BM + quarter * 32;
                if (nm0 < a.M) {
                  ptx::bulk_wait_read<0>();
                  ptx::mbar_expect_tx(&bbar[ew], 4096);
                  ptx::tma_load_4d(sb, &a.tadd, &bbar[ew], nnt * BN + c * SW, nm0, a.ep.add_sb1 ? nb1 : 0,
                                   a.ep.add_sb2 ? nb2 : 0);
                  bias_pending = true;
                }
              }
            }
          }
          if constexpr (BIASED) bias_pending = __shfl_sync(0xffffffffu, bias_pending, 0);
          continue;
        }
        if constexpr (SW == 64) {
          if (a.tma_store) {
            // row-oriented path: thread = output row; the epilogue (scale, bias,
            // triangle bias, activation, gate, residual, causal) runs in registers
            // with each thread reading its row's contiguous aux segments, then bf16
            // pack, 128B-swizzled staging, one TMA tensor store per warp and slab
            uint8_t* sb = reinterpret_cast<uint8_t*>(sEpi) + ew * 8192 + sbuf * 4096;
            if (lane == 0) ptx::bulk_wait_read<1>();  // the store issued two slabs ago has read its buffer
            __syncwarp();
            const int m = m0 + lane;
            const bool mvalid = m < a.M;
            if (a.lean) {
              // scale (+ causal) only: both TMEM loads in flight, no aux traffic
              uint32_t r[32], r2[32];
              ptx::tmem_ld32(tbase + c * SW, r);
              ptx::tmem_ld32(tbase + c * SW + 32, r2);
              ptx::tmem_ld_wait();
              if (last) {
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) acc_free(acc);
              }
              long long lim = a.ep.causal ? (a.ep.row_off + m - a.ep.col_off - n0) : (1ll << 40);
              if (lim > a.N - 1 - n0) lim = a.N - 1 - n0;  // columns past N: masked (clipped by the store)
              uint32_t pk[32];
              const float sc = a.ep.scale;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                float x0 = __uint_as_float(r[2 * j]) * sc, x1 = __uint_as_float(r[2 * j + 1]) * sc;
                float y0 = __uint_as_float(r2[2 * j]) * sc, y1 = __uint_as_float(r2[2 * j + 1]) * sc;
                if (2 * j > lim) x0 = -CUDART_INF_F;
                if (2 * j + 1 > lim) x1 = -CUDART_INF_F;
                if (32 + 2 * j > lim) y0 = -CUDART_INF_F;
                if (33 + 2 * j > lim) y1 = -CUDART_INF_F;
                __nv_bfloat162 hx = __floats2bfloat162_rn(x0, x1), hy = __floats2bfloat162_rn(y0, y1);
                pk[j] = *reinterpret_cast<uint32_t*>(&hx);
                pk[16 + j] = *reinterpret_cast<uint32_t*>(&hy);
              }
#pragma unroll
              for (int ch = 0; ch < 8; ++ch) {
                const uint32_t addr = ptx::smem_u32(sb + lane * 128 + ((ch ^ (lane & 7)) * 16));
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pk[4 * ch]),
                             "r"(pk[4 * ch + 1]), "r"(pk[4 * ch + 2]), "r"(pk[4 * ch + 3])
                             : "memory");
              }
            } else
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              uint32_t r[32];
              ptx::tmem_ld32(tbase + c * SW + hh * 32, r);
              ptx::tmem_ld_wait();
              if (hh == 1 && last) {
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) acc_free(acc);
              }
              uint32_t pk[16];
              epilogue_row32(a.ep, b1, b2, m, n0 + hh * 32, mvalid, r, pk, a.N - (n0 + hh * 32));
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int ch = hh * 4 + q;
                const uint32_t addr = ptx::smem_u32(sb + lane * 128 + ((ch ^ (lane & 7)) * 16));
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pk[4 * q]),
                             "r"(pk[4 * q + 1]), "r"(pk[4 * q + 2]), "r"(pk[4 * q + 3])
                             : "memory");
              }
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              ptx::tma_store_4d(&a.tout, sb, n0, m0, b1, b2);
              ptx::bulk_commit();
            }
            sbuf ^= 1;
            continue;
          }
        }
        uint32_t r[32];
        ptx::tmem_ld32(tbase + c * SW, r);
        if constexpr (SW == 64) {
          uint32_t r2[32];
          ptx::tmem_ld32(tbase + c * SW + 32, r2);
          ptx::tmem_ld_wait();
          float4* dst = reinterpret_cast<float4*>(stage + lane * PITCH);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                 __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
            dst[8 + j] = make_float4(__uint_as_float(r2[4 * j]), __uint_as_float(r2[4 * j + 1]),
                                     __uint_as_float(r2[4 * j + 2]), __uint_as_float(r2[4 * j + 3]));
          }
        } else {
          ptx::tmem_ld_wait();
          float4* dst = reinterpret_cast<float4*>(stage + lane * PITCH);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                 __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
        }
        if (last) {  // this warp's share of the accumulator is read: release TMEM
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) acc_free(acc);
        }
        __syncwarp();
        if (n0 < a.N) {
          const int rows = min(32, a.M - m0);
          if (a.vec) {
            // 8 consecutive columns per lane: SW/8 lanes cover a row segment, 32/(SW/8) rows per pass
            constexpr int LPR = SW / 8;
            constexpr int RPI = 32 / LPR;
            constexpr int NIT = 32 / RPI;     // row passes per slab
            constexpr int BATCH = 4;          // rows whose aux loads are in flight together
            const int sub = lane / LPR, seg = lane % LPR;
            const int n = n0 + seg * 8;
            const bool col_ok = n < a.N;
            float bias_n[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (a.ep.bias && !a.ep.bias_along_m && col_ok)
              bf16x8_to_f(*reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.ep.bias) + n), bias_n);
#pragma unroll
            for (int it0 = 0; it0 < NIT; it0 += BATCH) {
              Aux8 aux[BATCH];
#pragma unroll
              for (int q = 0; q < BATCH; ++q) {
                const int r = (it0 + q) * RPI + sub;
                if (r < rows && col_ok) load_aux8(a.ep, b1, b2, m0 + r, n, aux[q]);
              }
#pragma unroll
              for (int q = 0; q < BATCH; ++q) {
                const int r = (it0 + q) * RPI + sub;
                if (r < rows && col_ok) {
                  const float4* src = reinterpret_cast<const float4*>(stage + r * PITCH + seg * 8);
                  const float4 u0 = src[0], u1 = src[1];
                  float v8[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
                  epilogue8p(a.ep, b1, b2, m0 + r, n, v8, aux[q], bias_n);
                }
              }
            }
          } else {
#pragma unroll 4
            for (int rr = 0; rr < rows; ++rr) {
              if constexpr (SW == 64) {
                const float2 v = reinterpret_cast<const float2*>(stage + rr * PITCH)[lane];
                epilogue_pair<__nv_bfloat16>(a.ep, a.N, b1, b2, m0 + rr, n0 + 2 * lane, v.x, v.y);
              } else {
                const float v = stage[rr * PITCH + lane];
                epilogue_one<__nv_bfloat16>(a.ep, a.N, b1, b2, m0 + rr, n0 + lane, v);
              }
            }
          }
        }
        __syncwarp();
      }
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
    }
    if (lane == 0) ptx::bulk_wait_read<0>();  // staging buffers must outlive the TMA stores' reads
    __syncwarp();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (P2) ptx::cluster_sync();  // both CTAs of the pair are done with the paired TMEM
  if (warp == 1) {
    ptx::tc_fence_after();
    if (P2) ptx::tmem_dealloc2<C::TMEM_COLS>(tmem_base);
    else ptx::tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
#ifdef AC_DEBUG_HANG
  if (blockIdx.x == 0 && threadIdx.x == 0) printf("gemm_tc<%d,%d> exit\n", BN, MODE);
#endif
}

template <int BN, int MODE>
__global__ void __launch_bounds__(Cfg<BN, MODE>::THREADS, Cfg<BN, MODE>::MINB) gemm_tc_kernel(const __grid_constant__ GemmArgs a) {
  gemm_tc_body<BN, MODE, false>(a);
}

// the CTA-pair launches of MODE 0 (a.pair2 = 1) get their own function, the only one that
// contains cta_group::2 instructions: once a kernel with them has run as a cluster of 2,
// launches of such kernels without that cluster shape fail (cudaErrorInvalidClusterSize;
// scripts/micro/pair_alloc.cu, cluster_seq.cu)
template <int BN>
__global__ void __launch_bounds__(Cfg<BN, 0>::THREADS, 1) gemm_tc_pair_kernel(const __grid_constant__ GemmArgs a) {
  gemm_tc_body<BN, 0, true>(a);
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 4-D map {K, rows, b1, b2} over bf16, box {64, box_rows, 1, 1}, 128B swizzle.
bool make_map(CUtensorMap* m, const Operand& op, int K, int rows, int B1, int B2, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows),
                        static_cast<cuuint64_t>(op.use_b1 ? B1 : 1), static_cast<cuuint64_t>(op.use_b2 ? B2 : 1)};
  const int64_t big = (op.srow * static_cast<int64_t>(rows) + 8) * 2;
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(op.srow * 2),
                           static_cast<cuuint64_t>(op.use_b1 ? op.sb1 * 2 : ((big + 15) / 16) * 16),
                           static_cast<cuuint64_t>(op.use_b2 ? op.sb2 * 2 : ((big + 15) / 16) * 16)};
  for (int i = 0; i < 3; ++i)
    if (strides[i] % 16 != 0 || strides[i] == 0) return false;
  if ((reinterpret_cast<uintptr_t>(op.p) & 15) != 0) return false;
  cuuint32_t box[4] = {64, static_cast<cuuint32_t>(box_rows), 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(op.p), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, int MODE>
cudaError_t launch(const GemmProblem& p, cudaStream_t s) {
  using C = Cfg<BN, MODE>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    if constexpr (MODE == 0 && BN == 256) {
      e = cudaFuncSetAttribute(gemm_tc_pair_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
      if (e != cudaSuccess) return e;
    }
    attr = true;
  }
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  if (!(MODE == 2 && p.etile) &&
      !make_map(&a.ta, p.A, p.K, p.a_rows_total ? p.a_rows_total : p.M, p.B1, p.B2, MODE == 4 ? 64 : BM))
    return cudaErrorInvalidValue;
  a.etile = static_cast<char*>(p.etile);
  a.sched = MODE == 2 ? p.sched : nullptr;
  a.e_nkb = (MODE == 1 || MODE == 3 || MODE == 4) ? (p.N + 63) / 64 : (p.K + 63) / 64;
  if (p.etile && (reinterpret_cast<uintptr_t>(p.etile) & 127)) return cudaErrorInvalidValue;
  if (!make_map(&a.tb, p.B, p.K, p.b_rows_total ? p.b_rows_total : p.N, p.B1, p.B2, BN)) return cudaErrorInvalidValue;
  a.ep = p.ep;
  a.M = p.M; a.N = p.N; a.K = p.K; a.B1 = p.B1; a.B2 = p.B2;
  a.a_b1 = p.A.use_b1; a.a_b2 = p.A.use_b2; a.b_b1 = p.B.use_b1; a.b_b2 = p.B.use_b2;
  a.causal_tiles = p.causal_tiles; a.causal_k = p.causal_k; a.k_row_off = p.k_row_off;
  a.MT = (p.M + BM - 1) / BM;
  a.NT = (p.N + BN - 1) / BN;
  if (p.causal_tiles && a.MT > MAX_MT) return cudaErrorInvalidValue;  // prefix table size
  {
    // vectorised epilogue: n-contiguous 16-byte aligned output / aux rows, N % 8 == 0
    const Epilogue& e = p.ep;
    auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    auto m8 = [](int64_t v) { return v % 8 == 0; };
    bool v = p.N % 8 == 0 && e.out_sn == 1 && al(e.out) && m8(e.out_sm) && m8(e.out_sb1) && m8(e.out_sb2);
    if (e.add) v = v && e.add_sn == 1 && al(e.add) && m8(e.add_sm) && m8(e.add_sb1) && m8(e.add_sb2);
    if (e.gate) v = v && e.gate_sn == 1 && al(e.gate) && m8(e.gate_sm) && m8(e.gate_sb1) && m8(e.gate_sb2);
    if (e.res) v = v && e.res_sn == 1 && al(e.res) && m8(e.res_sm) && m8(e.res_sb1) && m8(e.res_sb2);
    if (e.bias && !e.bias_along_m) v = v && al(e.bias);
    a.vec = v ? 1 : 0;
    // row-oriented TMA-store epilogue: 64-column slabs, n-contiguous aligned output and aux
    if (BN >= 64 && v) {
      EncodeTiledFn enc = get_encode();
      cuuint64_t dims[4] = {static_cast<cuuint64_t>(p.N), static_cast<cuuint64_t>(p.M),
                            static_cast<cuuint64_t>(p.B1), static_cast<cuuint64_t>(p.B2)};
      const int64_t big = ((e.out_sm * p.M + 8) * 2 + 15) / 16 * 16;
      cuuint64_t strides[3] = {static_cast<cuuint64_t>(e.out_sm * 2),
                               static_cast<cuuint64_t>(p.B1 > 1 ? e.out_sb1 * 2 : big),
                               static_cast<cuuint64_t>(p.B2 > 1 ? e.out_sb2 * 2 : big)};
      cuuint32_t box[4] = {64, 32, 1, 1};
      cuuint32_t es[4] = {1, 1, 1, 1};
      bool ok = enc && strides[0] > 0 && strides[1] > 0 && strides[2] > 0;
      if (ok)
        ok = enc(&a.tout, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, e.out, dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
      a.tma_store = ok ? 1 : 0;
      a.lean = (!e.add && !e.bias && !e.gate && !e.res && e.act == ACT_NONE) ? 1 : 0;
    }
  }
  if ((MODE == 3 || MODE == 4) && p.ep.add && p.ep.add_sn == 1) {
    // bias map {N, M, B1, B2} (a batch dim the bias does not vary over gets extent 1)
    const Epilogue& e = p.ep;
    EncodeTiledFn enc = get_encode();
    const int64_t big = ((e.add_sm * p.M + 8) * 2 + 15) / 16 * 16;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(p.N), static_cast<cuuint64_t>(p.M),
                          static_cast<cuuint64_t>(e.add_sb1 ? p.B1 : 1), static_cast<cuuint64_t>(e.add_sb2 ? p.B2 : 1)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(e.add_sm * 2),
                             static_cast<cuuint64_t>(e.add_sb1 ? e.add_sb1 * 2 : big),
                             static_cast<cuuint64_t>(e.add_sb2 ? e.add_sb2 * 2 : big)};
    bool ok = enc && (reinterpret_cast<uintptr_t>(e.add) & 15) == 0;
    for (int i = 0; i < 3; ++i) ok = ok && strides[i] % 16 == 0 && strides[i] > 0;
    cuuint32_t box[4] = {64, MODE == 4 ? 16u : 32u, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (ok)
      ok = enc(&a.tadd, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(e.add), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    a.add_tma = ok ? 1 : 0;
  }
  a.tiles_per_batch_dense = a.MT * a.NT;
  a.total_tiles_dense = a.tiles_per_batch_dense * p.B1 * p.B2;
  // f2 modes: scores need the lean TMA-store epilogue and a positive scale; PV the
  // 64-wide tile with an n-contiguous aligned output
  // (MODE 1 may add an n-contiguous bias tensor, the AlphaFold triangle bias)
  if (MODE == 1 && !(a.tma_store && a.lean && p.ep.scale > 0.f)) return cudaErrorInvalidValue;
  if (MODE == 3 || MODE == 4) {
    const Epilogue& e = p.ep;
    if (MODE == 4 && !(p.M <= 64 && p.K <= BK && p.etile)) return cudaErrorInvalidValue;
    const bool only_add = !e.bias && !e.gate && !e.res && e.act == ACT_NONE && !e.causal && e.add;
    if (!(a.tma_store && a.add_tma && only_add && p.ep.scale > 0.f)) return cudaErrorInvalidValue;
  }
  if (MODE == 2 && !((BN == 64 || BN == 32) && a.vec)) return cudaErrorInvalidValue;
  a.fuse = MODE == 2 ? 1 : 0;
  if (MODE == 2) {
    const int kbn = (p.K + BK - 1) / BK;
    if (p.sk_part && p.sk_gk > 0 && a.NT == 1) {
      a.skgk = p.sk_gk;
      a.skpart = p.sk_part;
      a.skcnt = p.sk_cnt;
      a.skml = static_cast<float2*>(p.sk_ml);
    } else {
      a.skgk = kbn;  // one unit per tile
    }
    a.skng = (kbn + a.skgk - 1) / a.skgk;
    if (a.skng > 1 && !a.skcnt) return cudaErrorInvalidValue;
    if (a.skgk < kbn && !p.sk_ml) return cudaErrorInvalidValue;  // split online fold: (M, L) per granule
    if (p.causal_k && a.MT > MAX_MT) return cudaErrorInvalidValue;
  }
  a.pdl_wait = p.pdl_wait;
  a.done_cnt = MODE == 2 ? p.done_cnt : nullptr;
  a.done_epoch = (MODE == 2 && p.done_cnt) || (MODE != 2 && MODE != 0) ? p.done_epoch : nullptr;
  a.epoch = p.epoch;
  a.dep_epoch = p.dep_epoch;
  a.tsched = (MODE == 1 || MODE == 3 || MODE == 4) ? p.tsched : nullptr;
  a.fstats = p.fuse_stats;
  // statistics staged by 16-byte bulk copies: rows of a slab (M, even) at an even float2 offset
  a.stats_smem = (MODE == 2 && p.etile && p.fuse_stats && !(p.M & 1) && !(p.fuse_ss & 1) && !(p.fuse_sb1 & 1) &&
                  !(reinterpret_cast<uintptr_t>(p.fuse_stats) & 15))
                     ? 1
                     : 0;
  a.fst_sb1 = p.fuse_sb1;
  a.fst_ss = p.fuse_ss;
  const int sms = num_sms();
  // CTA pair (cta_group::2, M = 256 per MMA): halves each SM's shared-memory operand
  // traffic per FLOP (B halves).  Bitwise equal to single CTAs, but measured no faster on
  // the GPT / ViT linears (FFN1 142.6 vs 136.9 us, proj 39.0 vs 33.4 us; scripts/gemm_bench.py):
  // these GEMMs are bound by the epilogue warps, not by shared-memory bandwidth - so
  // only on request (ac_gemm_desc.cta_pair = 1)
  a.pair2 = (MODE == 0 && BN == 256 && a.vec && p.cta_pair > 0) ? 1 : 0;
  if (a.pair2) {
    if (!make_map(&a.tb, p.B, p.K, p.b_rows_total ? p.b_rows_total : p.N, p.B1, p.B2, BN / 2))
      return cudaErrorInvalidValue;
    a.MT = (p.M + 2 * BM - 1) / (2 * BM);  // tile rows in 256-row units
    a.tiles_per_batch_dense = a.MT * a.NT;
    a.total_tiles_dense = a.tiles_per_batch_dense * p.B1 * p.B2;
  }
  a.pair = (MODE == 2 && BN == 32 && p.etile && p.M <= 64 && a.skng == 1 && !p.causal_k) ? 1 : 0;
  if (a.pair) a.stats_smem = 0;  // pairs: two batches' rows per unit, global loads
  a.zero_word = (MODE == 1 || MODE == 3 || MODE == 4) ? p.zero_word : nullptr;
  a.zero_n = p.zero_n;
  const int cw = a.pair2 ? 2 : 1;  // CTAs per tile
  int grid = MODE == 4 ? ((p.B1 * p.B2 + 1) / 2) * a.NT
                       : (a.pair ? (p.B1 * p.B2 + 1) / 2 : a.total_tiles_dense) * cw * (MODE == 2 ? a.skng : 1);
  int cap = C::DUAL ? 2 * sms : (sms / cw) * cw;
  static int trace_on = -1;
  static unsigned long long* trace_buf = nullptr;
  static int trace_launch = 0;
  const long long trace_units = static_cast<long long>(a.total_tiles_dense) * (MODE == 2 ? a.skng : 1);
  if (trace_on < 0) trace_on = getenv("AC_TRACE") ? 1 : 0;
  if (MODE == 2 && trace_on) {
    if (!trace_buf) cudaMalloc(&trace_buf, 8 << 20);
    if (trace_units * 4 * 8 <= (8 << 20)) {
      cudaMemsetAsync(trace_buf, 0, trace_units * 32, s);
      a.trace = trace_buf;
    }
  }
  if (grid > cap) grid = cap;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute lattr[2];
  int na = 0;
  if (p.pdl) {
    lattr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    lattr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (a.pair2) {
    lattr[na].id = cudaLaunchAttributeClusterDimension;
    lattr[na].val.clusterDim.x = 2;
    lattr[na].val.clusterDim.y = 1;
    lattr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = lattr;
  cfg.numAttrs = na;
  auto kfn = gemm_tc_kernel<BN, MODE>;
  if constexpr (MODE == 0 && BN == 256)
    if (a.pair2) kfn = gemm_tc_pair_kernel<BN>;
  if (a.pair2) {
    static int diag = 0;
    int nclu = 0;
    cudaError_t oe = cudaOccupancyMaxActiveClusters(&nclu, kfn, &cfg);
    if (oe != cudaSuccess || nclu <= 0) {
      if (!diag++)
        fprintf(stderr, "gemm_tc: CTA pair not schedulable (%s, %d clusters, smem %d): single CTAs\n",
                cudaGetErrorString(oe), nclu, C::SMEM);
      cudaGetLastError();
      GemmProblem q = p;
      q.cta_pair = 0;
      return launch<BN, MODE>(q, s);
    }
  }
  cudaError_t err = cudaLaunchKernelEx(&cfg, kfn, a);
  if (err != cudaSuccess && a.pair2)
    fprintf(stderr, "gemm_tc<%d,%d> pair launch: %s grid %d block %d smem %d attrs %d (cluster %d)\n", BN, MODE,
            cudaGetErrorString(err), grid, C::THREADS, C::SMEM, na, a.pair2);
  if (err == cudaSuccess && a.trace) {  // debug only: dump {cta, t_load0, t_tfull, t_done} per unit
    std::vector<unsigned long long> h(trace_units * 4);
    cudaMemcpy(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost);
    char fn[256];
    snprintf(fn, sizeof fn, "%s/trace_%03d.txt", getenv("AC_TRACE"), trace_launch++);
    if (FILE* f = fopen(fn, "w")) {
      for (long long u = 0; u < trace_units; ++u)
        fprintf(f, "%lld %llu %llu %llu %llu\n", u, h[4 * u], h[4 * u + 1], h[4 * u + 2], h[4 * u + 3]);
      fclose(f);
    }
  }
  return err;
}

}  // namespace

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

cudaError_t gemm_tc(const GemmProblem& p, cudaStream_t s, int bn_hint) {
  if (p.M <= 0 || p.N <= 0 || p.K <= 0 || p.B1 <= 0 || p.B2 <= 0) return cudaErrorInvalidValue;
  int bn = bn_hint;
  if (bn == 0) {
    bn = p.N <= 32 ? 32 : p.N <= 64 ? 64 : p.N <= 128 ? 128 : 256;
    if (!p.ep.stats && !p.fuse_stats) {
      // short-M GEMMs (a row chunk of a linear): BN = 128 when BN = 256 leaves most SMs
      // idle, never narrower (a 128x64 tile halves the MMA width and measured slower in
      // every row-chunk shape: M = 2048, N = 1024, K = 4096: 25 us at 128, 42 us at 64;
      // scripts/gemm_bench.py)
      auto tiles = [&](int b) {
        return static_cast<long long>((p.M + 127) / 128) * ((p.N + b - 1) / b) * p.B1 * p.B2;
      };
      if (bn == 256 && tiles(256) < num_sms() * 3 / 4) bn = 128;
    }
  }
  if (p.fuse_stats) return p.N <= 32 ? launch<32, 2>(p, s) : bn == 64 ? launch<64, 2>(p, s) : cudaErrorInvalidValue;
  if (p.ep.stats && p.ep.add && p.M <= 64 && p.etile && p.K <= 64)
    return launch<256, 4>(p, s);  // short chunks: paired 64-row tiles
  if (p.ep.stats && p.ep.add) {
    switch (bn) {
      case 64: return launch<64, 3>(p, s);
      case 128: return launch<128, 3>(p, s);
      case 256: return launch<256, 3>(p, s);
      default: return cudaErrorInvalidValue;
    }
  }
  if (p.ep.stats) {
    switch (bn) {
      case 64: return launch<64, 1>(p, s);
      case 128: return launch<128, 1>(p, s);
      case 256: return launch<256, 1>(p, s);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (bn) {
    case 32: return launch<32, 0>(p, s);
    case 64: return launch<64, 0>(p, s);
    case 128: return launch<128, 0>(p, s);
    case 256: return launch<256, 0>(p, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ac
