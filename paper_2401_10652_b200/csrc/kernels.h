// Host-side launch API of the sm_100a kernels (internal to libautochunk).
// Every kernel works on dense strided tensors owned by the caller; nothing here
// allocates device memory.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ac {

enum Act : int { ACT_NONE = 0, ACT_GELU = 1, ACT_SIGMOID = 2, ACT_RELU = 3 };

// One K-major GEMM operand: element (b1, b2, row, k) lives at
//   p + b1*sb1 + b2*sb2 + row*srow + k        (element units, k contiguous).
// use_b1 / use_b2 = 0 means the operand is shared across that batch dim.
struct Operand {
  const void* p = nullptr;
  int64_t srow = 0, sb1 = 0, sb2 = 0;
  int use_b1 = 0, use_b2 = 0;
};

// Epilogue applied to acc (fp32) in this order (DESIGN.md §5 "G1 epilogue"):
//   v = acc * scale
//   v += add[b1,b2,m,n]            (triangle bias)
//   v += bias[n] | bias[m]         (linear bias)
//   v = act(v)
//   v *= gate[b1,b2,m,n]           (AlphaFold sigmoid gate)
//   v += res[b1,b2,m,n]            (residual)
//   causal: v = -inf where (col_off + n) > (row_off + m)
//   out[b1,b2,m,n] = v
struct Epilogue {
  float scale = 1.f;
  int act = ACT_NONE;
  int causal = 0;
  int64_t row_off = 0, col_off = 0;
  const void* bias = nullptr;
  int bias_along_m = 0;
  const void* add = nullptr;
  int64_t add_sb1 = 0, add_sb2 = 0, add_sm = 0, add_sn = 0;
  const void* gate = nullptr;
  int64_t gate_sb1 = 0, gate_sb2 = 0, gate_sm = 0, gate_sn = 1;
  const void* res = nullptr;
  int64_t res_sb1 = 0, res_sb2 = 0, res_sm = 0, res_sn = 1;
  void* out = nullptr;
  int64_t out_sb1 = 0, out_sb2 = 0, out_sm = 0, out_sn = 1;
  // fused softmax (NEXT f2), QK^T lean epilogue only (scale > 0): with stats
  // non-null the score is taken in the log2 domain, x = acc * scale * log2(e)
  // (fp32, never rounded), the stored value is e = bf16(2^(x - m2)) with m2 the
  // slab max, and stats[b1*stats_sb1 + (n/64)*stats_ss + m] = (m2, fp32 sum of e)
  // per (b1, 64-column slab, row) - slab-major so a warp's 32 rows write 256 B
  float2* stats = nullptr;
  int64_t stats_sb1 = 0, stats_ss = 0;
};

// D[b1,b2][m][n] = sum_k A[b1,b2][m][k] * B[b1,b2][n][k]
struct GemmProblem {
  int M = 0, N = 0, K = 0, B1 = 1, B2 = 1;
  int a_rows_total = 0;  // extent of A's row dim in memory (for TMA bounds); 0 -> M
  int b_rows_total = 0;  // extent of B's row dim in memory; 0 -> N
  Operand A, B;
  Epilogue ep;
  int causal_tiles = 0;  // skip (m,n) tiles entirely above the diagonal (QK^T)
  int causal_k = 0;      // K loop stops after the tile's last row (PV, keys = K)
  int64_t k_row_off = 0; // global row of m = 0 for causal_k
  // split-K across a thread-block cluster (tcgen05 path, BN = 64): the KS CTAs of
  // a cluster take contiguous K ranges of the same tile and the leader sums the
  // fp32 partials through distributed shared memory in rank order (deterministic;
  // the split depends only on the tile's K range, never on the chunking)
  int cta_pair = 0;  // MODE 0, BN = 256: 1 = CTA pair (cta_group::2)
  // fused softmax-normalised PV (NEXT f2): A holds e = 2^(x - m2_slab) written by
  // the QK^T epilogue (Epilogue::stats, the slab statistics (m2, l) in fuse_stats);
  // each 64-key slab's product e V lands in its own TMEM buffer and is folded into
  // the row's output with f = 2^(m2_slab - M_run) against the running max (online,
  // in slab order), o = O / L at the end, so P is never written.  BN = 32 / 64.
  const float2* fuse_stats = nullptr;
  int64_t fuse_sb1 = 0, fuse_ss = 0;
  // fixed split-K of the fused PV (SURVEY H-g): the key range is cut into
  // granules of sk_gk k-blocks at fixed key positions (0 = off); one work unit
  // per (tile, granule) balances the waves, multi-granule tiles leave fp32 partials
  // (BM x 64 per unit) in sk_part and the unit that completes a tile sums them in
  // granule order, so the result does not depend on the scheduling or chunking.
  // sk_cnt: one zero-initialised int per tile (B1*B2*MT), left zero on return.
  int sk_gk = 0;
  float* sk_part = nullptr;
  int* sk_cnt = nullptr;
  void* sk_ml = nullptr;  // float2 per (unit, row): online fold with split-K
  // f2 e-tiles: e = 2^(x - m2) stored as pre-swizzled 16 KB tiles, tile
  // (b1, mt, kb) = the 128-row x 64-key block exactly as the 128B-swizzled UMMA
  // operand sits in shared memory, at etile + ((b1 * MT + mt) * NKB + kb) * 16384
  // (MT = ceil(M / 128), NKB = ceil(keys / 64)).  The QK^T (Epilogue::stats set)
  // writes it with 4 KB bulk stores instead of its output tensor; the PV
  // (fuse_stats set) reads its A operand from it with 16 KB bulk loads.
  void* etile = nullptr;
  // f2 PV: zero-initialised int; CTAs take work units from it dynamically (faster
  // SMs take more), null = static round-robin.  Results do not depend on it.
  int* sched = nullptr;
  // Chunk-loop overlap (f2 chains): launched with programmatic
  // stream serialisation (pdl) so the kernel may start while the previous one
  // drains; pdl_wait: griddepcontrol.wait before reading the predecessor's output.
  // MODE 2 (PV) marks a batch finished for chunk `epoch`: done_cnt[b] counts its
  // units and the unit completing the batch stores epoch + 1 to done_epoch[b]
  // (release).  MODE 1 (scores of the next chunk) stores nothing of batch b before
  // done_epoch[b] >= dep_epoch (acquire): the PV of the previous chunk has read
  // that batch's e-tiles and statistics.  tsched: zero-initialised tile counter
  // (MODE 1 dynamic tiles, so CTAs that start late on SMs the PV frees take fewer).
  int pdl = 0, pdl_wait = 0;
  int* done_cnt = nullptr;
  int* done_epoch = nullptr;
  int epoch = 0;
  int dep_epoch = 0;
  int* tsched = nullptr;
  // the scores zero the PV's unit counter (and split-K tile counters) at start
  int* zero_word = nullptr;
  int zero_n = 1;  // words zeroed from zero_word
};

// NEXT f1: fused attention o = softmax(q k^T * scale) v, no N x N tensor (attn_fused.cu).
// q [M, H, dh] (row stride q_srow, head stride q_sh; dh contiguous), k [Nk, H, dh],
// vt [H, dh, Nk] (keys contiguous), out [M, H, dh]; element strides.  dh = 64.
// causal: key j > row_off + m masked (row_off = global row of local row 0).
struct AttnFusedProblem {
  const void* q = nullptr;
  const void* k = nullptr;
  const void* vt = nullptr;
  void* out = nullptr;
  int64_t M = 0, Nk = 0, H = 0, dh = 0;
  int64_t q_srow = 0, q_sh = 0, k_srow = 0, k_sh = 0, v_sh = 0, v_sdh = 0, o_srow = 0, o_sh = 0;
  float scale = 1.f;
  int causal = 0;
  int64_t row_off = 0;
  int pdl = 0;  // programmatic dependent launch (chunk loop): wait for the predecessor in-kernel
};
cudaError_t attn_fused(const AttnFusedProblem& p, cudaStream_t s);

// bf16 x bf16 -> fp32 (TMEM) -> bf16, tcgen05 + TMA, sm_100a.  Returns a
// cudaError_t (cudaErrorInvalidValue for shapes it cannot take).
cudaError_t gemm_tc(const GemmProblem& p, cudaStream_t s, int bn_hint = 0);
// fp32 SIMT (FFMA) path for fp32 graphs (G8).
cudaError_t gemm_f32(const GemmProblem& p, cudaStream_t s);

// Row ops.  dtype: 0 = fp32, 1 = bf16.
// LayerNorm over the last C elements of `rows` rows (row stride = C).
// rows: `group` contiguous rows per group, groups gx / gy elements apart in x / y
// (group <= 0: all rows contiguous)
cudaError_t layernorm(const void* x, const void* gamma, const void* beta, void* y, int64_t rows,
                      int C, float eps, int dtype, cudaStream_t s, int pdl = 0, int64_t group = 0, int64_t gx = 0,
                      int64_t gy = 0);
// ln_cfirst: x [C, I, J] (element strides xs_c, xs_i; j contiguous) -> y [I, J, C]
// (strides ys_i, ys_j; c contiguous), LayerNorm over c with fp32 two-pass statistics.
cudaError_t layernorm_cfirst(const void* x, int64_t xs_c, int64_t xs_i, const void* gamma, const void* beta, void* y,
                             int64_t ys_i, int64_t ys_j, int C, int64_t I, int64_t J, float eps, int dtype,
                             cudaStream_t s, int pdl = 0);
// Row softmax: rows of `ncols` values with row stride `ld` (elements).  With
// causal, row r is query row R = row_off + (r % group) (rows of several heads
// are stacked); it reads columns <= R and writes columns [0, ceil128(R+1)) with
// zeros above the diagonal (the causal PV reads whole 128-key blocks);
// otherwise the full row.  Input row r lives at (r / group) * gstride + (r % group) * ld
// (group = 0: r * ld); output rows likewise with gstrideo / ldo.
cudaError_t softmax_rows(const void* s_in, void* p_out, int64_t rows, int64_t ncols, int64_t ld, int64_t gstride,
                         int64_t ldo, int64_t gstrideo, int causal, int64_t row_off, int64_t group, int dtype,
                         cudaStream_t s);

int num_sms();

}  // namespace ac
