"""Thin wrappers of include/ac_kernels.h for torch tensors (marshalling only)."""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import AC_BF16, AC_F32, GemmDesc, check, lib

_DT = {torch.bfloat16: AC_BF16, torch.float32: AC_F32}


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def gemm(a, a_srow, b, b_srow, out, M, N, K, B1=1, B2=1, a_sb=(0, 0), a_use=(0, 0), b_sb=(0, 0),
         b_use=(0, 0), out_s=(0, 0, 0, 1), scale=1.0, act=0, causal=0, row_off=0, col_off=0,
         causal_tiles=0, causal_k=0, k_row_off=0, bias=None, bias_along_m=0, add=None,
         add_s=(0, 0, 0, 0), gate=None, res=None, bn=0, cta_pair=-1, stream=None):
    d = GemmDesc()
    d.dtype = _DT[a.dtype]
    d.M, d.N, d.K, d.B1, d.B2 = M, N, K, B1, B2
    d.a, d.a_srow, d.a_sb1, d.a_sb2, d.a_use_b1, d.a_use_b2 = a.data_ptr(), a_srow, a_sb[0], a_sb[1], a_use[0], a_use[1]
    d.b, d.b_srow, d.b_sb1, d.b_sb2, d.b_use_b1, d.b_use_b2 = b.data_ptr(), b_srow, b_sb[0], b_sb[1], b_use[0], b_use[1]
    d.scale, d.act, d.causal, d.row_off, d.col_off = scale, act, causal, row_off, col_off
    d.causal_tiles, d.causal_k, d.k_row_off = causal_tiles, causal_k, k_row_off
    d.bias = None if bias is None else bias.data_ptr()
    d.bias_along_m = bias_along_m
    d.add = None if add is None else add.data_ptr()
    d.add_sb1, d.add_sb2, d.add_sm, d.add_sn = add_s
    d.gate = None if gate is None else gate.data_ptr()
    d.res = None if res is None else res.data_ptr()
    d.out = out.data_ptr()
    d.out_sb1, d.out_sb2, d.out_sm, d.out_sn = out_s
    d.bn = bn
    d.cta_pair = cta_pair
    check(lib().ac_kernel_gemm(C.byref(d), _stream(stream)))
    return out


def layernorm(x, gamma, beta, y, eps=1e-5, stream=None):
    C_ = x.shape[-1]
    rows = x.numel() // C_
    check(lib().ac_kernel_layernorm(_ptr(x), _ptr(gamma), _ptr(beta), _ptr(y), rows, C_, eps, _DT[x.dtype],
                                    _stream(stream)))
    return y


def softmax(s, p, rows, ncols, ld, causal=0, row_off=0, group=0, stream=None):
    check(lib().ac_kernel_softmax(_ptr(s), _ptr(p), rows, ncols, ld, causal, row_off, group, _DT[s.dtype],
                                  _stream(stream)))
    return p
