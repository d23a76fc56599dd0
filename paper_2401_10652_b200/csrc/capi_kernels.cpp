// C ABI wrappers of the individual kernels (include/ac_kernels.h).
#include <cuda_runtime.h>

#include <string>

#include "../../include/ac_kernels.h"
#include "errors.h"
#include "kernels.h"

using namespace ac;

extern "C" ac_status ac_kernel_gemm(const ac_gemm_desc* d, void* stream) {
  if (!d) return set_error(AC_ERR_ARG, "ac_kernel_gemm: NULL desc");
  GemmProblem p;
  p.M = d->M; p.N = d->N; p.K = d->K; p.B1 = d->B1 < 1 ? 1 : d->B1; p.B2 = d->B2 < 1 ? 1 : d->B2;
  p.A.p = d->a; p.A.srow = d->a_srow; p.A.sb1 = d->a_sb1; p.A.sb2 = d->a_sb2;
  p.A.use_b1 = d->a_use_b1; p.A.use_b2 = d->a_use_b2;
  p.B.p = d->b; p.B.srow = d->b_srow; p.B.sb1 = d->b_sb1; p.B.sb2 = d->b_sb2;
  p.B.use_b1 = d->b_use_b1; p.B.use_b2 = d->b_use_b2;
  p.causal_tiles = d->causal_tiles; p.causal_k = d->causal_k; p.k_row_off = d->k_row_off;
  Epilogue& e = p.ep;
  e.scale = d->scale; e.act = d->act; e.causal = d->causal; e.row_off = d->row_off; e.col_off = d->col_off;
  e.bias = d->bias; e.bias_along_m = d->bias_along_m;
  e.add = d->add; e.add_sb1 = d->add_sb1; e.add_sb2 = d->add_sb2; e.add_sm = d->add_sm; e.add_sn = d->add_sn;
  e.gate = d->gate; e.res = d->res;
  e.out = d->out; e.out_sb1 = d->out_sb1; e.out_sb2 = d->out_sb2; e.out_sm = d->out_sm; e.out_sn = d->out_sn;
  // gate and residual share the output layout at this entry point
  e.gate_sb1 = e.res_sb1 = d->out_sb1;
  e.gate_sb2 = e.res_sb2 = d->out_sb2;
  e.gate_sm = e.res_sm = d->out_sm;
  e.gate_sn = e.res_sn = d->out_sn;
  cudaError_t err;
  p.cta_pair = d->cta_pair;
  if (d->dtype == 1) err = gemm_tc(p, static_cast<cudaStream_t>(stream), d->bn);
  else if (d->dtype == 0) err = gemm_f32(p, static_cast<cudaStream_t>(stream));
  else return set_error(AC_ERR_ARG, "ac_kernel_gemm: dtype must be AC_F32 or AC_BF16");
  return cuda_status(err, "ac_kernel_gemm");
}

extern "C" ac_status ac_kernel_layernorm(const void* x, const void* gamma, const void* beta, void* y, int64_t rows,
                                         int32_t C, float eps, int32_t dtype, void* stream) {
  return cuda_status(layernorm(x, gamma, beta, y, rows, C, eps, dtype, static_cast<cudaStream_t>(stream)),
                     "ac_kernel_layernorm");
}

extern "C" ac_status ac_kernel_softmax(const void* s, void* p, int64_t rows, int64_t ncols, int64_t ld,
                                       int32_t causal, int64_t row_off, int64_t group, int32_t dtype, void* stream) {
  return cuda_status(softmax_rows(s, p, rows, ncols, ld, group * ld, ld, group * ld, causal, row_off, group, dtype,
                                  static_cast<cudaStream_t>(stream)),
                     "ac_kernel_softmax");
}
