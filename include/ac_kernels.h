/*
 * ac_kernels.h — kernel-level entry points of libautochunk, for unit tests and
 * micro-benchmarks of the individual sm_100a kernels that ac_run composes.
 * Same conventions as ac.h: caller-owned device pointers, asynchronous on
 * `stream` (a cudaStream_t, NULL = default stream), ac_status return codes,
 * AC_ERR_ARG for shapes / alignments a kernel cannot take, AC_ERR_CUDA for
 * launch failures (message in ac_last_error()).
 */
#ifndef AUTOCHUNK_AC_KERNELS_H
#define AUTOCHUNK_AC_KERNELS_H

#include "ac.h"

#ifdef __cplusplus
extern "C" {
#endif

/* One batched GEMM with the fused epilogue of DESIGN.md §5 (G1/G2/G4):
 *   D[b1,b2][m][n] = epi( sum_k A[b1,b2][m][k] * B[b1,b2][n][k] )
 * Operand X element (b1,b2,r,k) is at X + b1*x_sb1 + b2*x_sb2 + r*x_srow + k
 * (elements, k contiguous); x_use_b1/x_use_b2 = 0 shares the operand across
 * that batch dim.  Epilogue order: *scale, +add, +bias, act, *gate, +res,
 * causal mask (-inf where col_off+n > row_off+m), store.  gate/res use the
 * output strides.  dtype AC_BF16 runs the tcgen05 tensor-core kernel (bf16 in,
 * fp32 TMEM accumulate, bf16 out); AC_F32 runs the FFMA SIMT kernel. */
typedef struct ac_gemm_desc {
  int32_t dtype;
  int32_t M, N, K, B1, B2;
  const void* a; int64_t a_srow, a_sb1, a_sb2; int32_t a_use_b1, a_use_b2;
  const void* b; int64_t b_srow, b_sb1, b_sb2; int32_t b_use_b1, b_use_b2;
  float scale;
  int32_t act;               /* 0 none, 1 erf-GELU, 2 sigmoid, 3 relu */
  int32_t causal;            /* mask in the epilogue */
  int64_t row_off, col_off;
  int32_t causal_tiles;      /* skip tiles above the diagonal (QK^T) */
  int32_t causal_k;          /* stop K at the tile's last row (PV) */
  int64_t k_row_off;
  const void* bias; int32_t bias_along_m;
  const void* add; int64_t add_sb1, add_sb2, add_sm, add_sn;
  const void* gate;
  const void* res;
  void* out; int64_t out_sb1, out_sb2, out_sm, out_sn;
  int32_t bn;                /* tcgen05 N tile (32/64/128/256), 0 = auto */
  int32_t cta_pair;          /* BN = 256 plain GEMMs: 1 = run as CTA pairs (cta_group::2, M = 256 per
                                MMA, bitwise equal to single CTAs); <= 0 single CTAs */
} ac_gemm_desc;

ac_status ac_kernel_gemm(const ac_gemm_desc* d, void* stream);

/* Row LayerNorm over the last C elements (row stride C), fp32 statistics. */
ac_status ac_kernel_layernorm(const void* x, const void* gamma, const void* beta, void* y, int64_t rows,
                              int32_t C, float eps, int32_t dtype, void* stream);

/* Row softmax (stable), rows of ncols with row stride ld.  causal: row r is
 * query row R = row_off + (r % group) (group = rows per head, 0 = no wrap); it
 * reads columns <= R and writes columns < ceil128(R+1), zeros above the
 * diagonal. */
ac_status ac_kernel_softmax(const void* s, void* p, int64_t rows, int64_t ncols, int64_t ld, int32_t causal,
                            int64_t row_off, int64_t group, int32_t dtype, void* stream);

#ifdef __cplusplus
}
#endif
#endif
