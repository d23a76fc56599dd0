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

#include <mutex>

#include "epilogue.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace ac {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int NUM_THREADS = 192;
constexpr int MAX_MT = 2048;

struct alignas(64) GemmArgs {
  CUtensorMap ta;
  CUtensorMap tb;
  Epilogue ep;
  int M, N, K, B1, B2;
  int a_b1, a_b2, b_b1, b_b2;
  int causal_tiles, causal_k;
  long long k_row_off;
  int MT, NT;
  int tiles_per_batch_dense;
  int total_tiles_dense;
};

template <int BN>
struct Cfg {
  static constexpr int STAGES = BN >= 256 ? 4 : (BN >= 128 ? 6 : 8);
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int TMEM_COLS = (2 * BN) <= 32 ? 32 : (2 * BN) <= 64 ? 64 : (2 * BN) <= 128 ? 128 : (2 * BN) <= 256 ? 256 : 512;
  static constexpr int SMEM = 1024 /*align slack*/ + STAGES * (A_BYTES + B_BYTES) + 256 /*barriers*/ +
                              (MAX_MT + 1) * 4;
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

template <int BN>
__global__ void __launch_bounds__(NUM_THREADS, 1) gemm_tc_kernel(const __grid_constant__ GemmArgs a) {
  using C = Cfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  int* prefix = reinterpret_cast<int*>(full + 32);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // --- tile table for causal QK^T: live n-tiles per m-tile, prefix-summed
  int tpb = a.tiles_per_batch_dense;
  if (a.causal_tiles) {
    for (int mt = threadIdx.x; mt < a.MT; mt += NUM_THREADS) {
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
  const int total = tpb * a.B1 * a.B2;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&a.ta);
    ptx::prefetch_tmap(&a.tb);
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 4);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<C::TMEM_COLS>(tmem_holder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int b1, b2, mt, nt, kbn;
        decode_tile(a, prefix, tpb, t, b1, b2, mt, nt, kbn);
        const int ac2 = a.a_b1 ? b1 : 0, ac3 = a.a_b2 ? b2 : 0;
        const int bc2 = a.b_b1 ? b1 : 0, bc3 = a.b_b2 ? b2 : 0;
        for (int kb = 0; kb < kbn; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_expect_tx(&full[stage], C::A_BYTES + C::B_BYTES);
          ptx::tma_load_4d(sA + stage * C::A_BYTES, &a.ta, &full[stage], kb * BK, mt * BM, ac2, ac3);
          ptx::tma_load_4d(sB + stage * C::B_BYTES, &a.tb, &full[stage], kb * BK, nt * BN, bc2, bc3);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t IDESC = ptx::idesc_bf16(BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t aphase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int b1, b2, mt, nt, kbn;
      decode_tile(a, prefix, tpb, t, b1, b2, mt, nt, kbn);
      ptx::mbar_wait(&tempty[acc], aphase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d = tmem_base + acc * BN;
      for (int kb = 0; kb < kbn; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = ptx::smem_u32(sA + stage * C::A_BYTES);
          const uint32_t sb = ptx::smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            ptx::mma_bf16(d, ptx::sdesc_sw128(sa + k * 32), ptx::sdesc_sw128(sb + k * 32), IDESC,
                          (kb | k) != 0);
          }
          ptx::mma_commit(&empty[stage]);  // slot free once these MMAs have read smem
        }
        __syncwarp();
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) ptx::mma_commit(&tfull[acc]);  // accumulator ready
      __syncwarp();
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31
    const int row = quarter * 32 + lane;
    int acc = 0;
    uint32_t aphase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int b1, b2, mt, nt, kbn;
      decode_tile(a, prefix, tpb, t, b1, b2, mt, nt, kbn);
      ptx::mbar_wait(&tfull[acc], aphase);
      ptx::tc_fence_after();
      const int m = mt * BM + row;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        ptx::tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN + c * 32, r);
        ptx::tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if (nt * BN + c * 32 < a.N)
          epilogue_row32<__nv_bfloat16>(a.ep, a.M, a.N, b1, b2, m, nt * BN + c * 32, v);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
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

template <int BN>
cudaError_t launch(const GemmProblem& p, cudaStream_t s) {
  using C = Cfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  if (!make_map(&a.ta, p.A, p.K, p.a_rows_total ? p.a_rows_total : p.M, p.B1, p.B2, BM)) return cudaErrorInvalidValue;
  if (!make_map(&a.tb, p.B, p.K, p.b_rows_total ? p.b_rows_total : p.N, p.B1, p.B2, BN)) return cudaErrorInvalidValue;
  a.ep = p.ep;
  a.M = p.M; a.N = p.N; a.K = p.K; a.B1 = p.B1; a.B2 = p.B2;
  a.a_b1 = p.A.use_b1; a.a_b2 = p.A.use_b2; a.b_b1 = p.B.use_b1; a.b_b2 = p.B.use_b2;
  a.causal_tiles = p.causal_tiles; a.causal_k = p.causal_k; a.k_row_off = p.k_row_off;
  a.MT = (p.M + BM - 1) / BM;
  a.NT = (p.N + BN - 1) / BN;
  if (a.MT > MAX_MT) return cudaErrorInvalidValue;
  a.tiles_per_batch_dense = a.MT * a.NT;
  a.total_tiles_dense = a.tiles_per_batch_dense * p.B1 * p.B2;
  int grid = a.total_tiles_dense;
  const int sms = num_sms();
  if (grid > sms) grid = sms;
  if (grid < 1) grid = 1;
  gemm_tc_kernel<BN><<<grid, NUM_THREADS, C::SMEM, s>>>(a);
  return cudaGetLastError();
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
  if (bn == 0) bn = p.N <= 32 ? 32 : p.N <= 64 ? 64 : p.N <= 128 ? 128 : 256;
  switch (bn) {
    case 32: return launch<32>(p, s);
    case 64: return launch<64>(p, s);
    case 128: return launch<128>(p, s);
    case 256: return launch<256>(p, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ac
