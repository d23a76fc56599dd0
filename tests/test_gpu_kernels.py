"""Kernel-level parity (through include/ac_kernels.h) against plain PyTorch fp32
references of the same op.  GPU only."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2401_10652_b200 import kernels
    return kernels


def _rel(a, b):
    a = a.float()
    b = b.float()
    return ((a - b).abs().max() / b.abs().max().clamp_min(1e-30)).item()


@pytest.mark.parametrize("M,N,Kd,bn", [(256, 512, 256, 0), (200, 300, 104, 0), (128, 64, 64, 64),
                                       (384, 32, 1024, 32), (1000, 1000, 1000, 128), (4096, 4096, 1024, 256)])
def test_gemm_tc_plain(K, M, N, Kd, bn):
    torch.manual_seed(0)
    a = torch.randn(M, Kd, device="cuda").bfloat16()
    b = torch.randn(N, Kd, device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    K.gemm(a, Kd, b, Kd, out, M, N, Kd, out_s=(0, 0, N, 1), bn=bn)
    ref = a.float() @ b.float().T
    torch.cuda.synchronize()
    assert _rel(out, ref) < 1e-2


def test_gemm_tc_epilogue_bias_gelu_res(K):
    torch.manual_seed(1)
    M, N, Kd = 300, 384, 256
    a = torch.randn(M, Kd, device="cuda").bfloat16()
    w = (torch.randn(N, Kd, device="cuda") / 16).bfloat16()
    bias = torch.randn(N, device="cuda").bfloat16()
    res = torch.randn(M, N, device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    K.gemm(a, Kd, w, Kd, out, M, N, Kd, out_s=(0, 0, N, 1), bias=bias, act=1, res=res)
    ref = torch.nn.functional.gelu(a.float() @ w.float().T + bias.float()) + res.float()
    assert _rel(out, ref) < 1e-2
    # transposed output with per-row bias (linear trans=1: D[o, r] = W A^T)
    outT = torch.empty(N, M, device="cuda", dtype=torch.bfloat16)
    K.gemm(w, Kd, a, Kd, outT, N, M, Kd, out_s=(0, 0, M, 1), bias=bias, bias_along_m=1)
    assert _rel(outT, (a.float() @ w.float().T + bias.float()).T) < 1e-2


def test_gemm_tc_batched_heads_scores_causal(K):
    """QK^T per head from [N, h, dh] layouts, scale + causal mask, tile skipping."""
    torch.manual_seed(2)
    N, h, dh = 1024, 4, 64
    q = torch.randn(N, h, dh, device="cuda").bfloat16()
    k = torch.randn(N, h, dh, device="cuda").bfloat16()
    for row_off, rows in ((0, N), (256, 256), (512, 512)):
        s = torch.full((h, rows, N), 7.0, device="cuda", dtype=torch.bfloat16)
        sc = 1 / math.sqrt(dh)
        K.gemm(q[row_off:], h * dh, k, h * dh, s, rows, N, dh, B1=h, a_sb=(dh, 0), a_use=(1, 0), b_sb=(dh, 0),
               b_use=(1, 0), out_s=(rows * N, 0, N, 1), scale=sc, causal=1, row_off=row_off, causal_tiles=1)
        ref = torch.einsum("ihc,jhc->hij", q[row_off:row_off + rows].float(), k.float()) * sc
        i = torch.arange(rows, device="cuda")[:, None] + row_off
        j = torch.arange(N, device="cuda")[None, :]
        mask = (j <= i)[None].expand(h, rows, N)
        got = s.float()
        assert _rel(got[mask], ref[mask]) < 1e-2
        # keys above the diagonal inside the row's 128-block span are written as -inf
        above = ((j > i) & (j < (i // 128 + 1) * 128))[None].expand(h, rows, N)
        assert torch.isinf(got[above]).all() and (got[above] < 0).all()


def test_gemm_tc_pv_causal_k(K):
    torch.manual_seed(3)
    N, h, dh, rows, row_off = 1024, 2, 64, 512, 256
    p = torch.rand(h, rows, N, device="cuda")
    i = torch.arange(rows, device="cuda")[:, None] + row_off
    j = torch.arange(N, device="cuda")[None, :]
    p = torch.where((j <= i)[None], p, torch.zeros_like(p)).bfloat16()
    vt = torch.randn(h, dh, N, device="cuda").bfloat16()
    o = torch.empty(rows, h, dh, device="cuda", dtype=torch.bfloat16)
    K.gemm(p, N, vt, N, o, rows, dh, N, B1=h, a_sb=(rows * N, 0), a_use=(1, 0), b_sb=(dh * N, 0), b_use=(1, 0),
           out_s=(dh, 0, h * dh, 1), causal_k=1, k_row_off=row_off)
    ref = torch.einsum("hij,hcj->ihc", p.float(), vt.float())
    assert _rel(o, ref) < 1e-2


@pytest.mark.parametrize("M,N,Kd,act,bias,res", [(4096, 4096, 1024, 1, True, False),
                                                  (2048 + 128 + 64, 1024, 4096, 0, True, True),
                                                  (1000, 512, 256, 0, False, False)])
def test_gemm_tc_cta_pair(K, M, N, Kd, act, bias, res):
    """CTA pairs (cta_group::2: the leader's M = 256 MMAs over both CTAs' shared-memory
    halves, multicast commits, the peer's rows written by the peer's epilogue) give the
    same bits as single CTAs (the K reduction order per element is unchanged, so chunked
    linears stay bitwise equal to unchunked ones), and match the fp32 reference; ragged
    M leaves the peer's half partly past the rows."""
    torch.manual_seed(3)
    a = torch.randn(M, Kd, device="cuda").bfloat16()
    w = (torch.randn(N, Kd, device="cuda") / Kd ** 0.5).bfloat16()
    bv = torch.randn(N, device="cuda").bfloat16() if bias else None
    rv = torch.randn(M, N, device="cuda").bfloat16() if res else None
    outs = []
    for pair in (1, 0):
        o = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        K.gemm(a, Kd, w, Kd, o, M, N, Kd, out_s=(0, 0, N, 1), bias=bv, act=act, res=rv, bn=256, cta_pair=pair)
        outs.append(o)
    torch.cuda.synchronize()
    ref = a.float() @ w.float().T + (bv.float() if bias else 0)
    if act == 1:
        ref = torch.nn.functional.gelu(ref)
    if res:
        ref = ref + rv.float()
    assert _rel(outs[0], ref) < 1e-2
    assert torch.equal(outs[0], outs[1])


def test_gemm_f32_path(K):
    torch.manual_seed(4)
    M, N, Kd = 100, 70, 33
    a = torch.randn(M, Kd, device="cuda")
    b = torch.randn(N, Kd, device="cuda")
    bias = torch.randn(N, device="cuda")
    out = torch.empty(M, N, device="cuda")
    K.gemm(a, Kd, b, Kd, out, M, N, Kd, out_s=(0, 0, N, 1), bias=bias, act=2)
    ref = torch.sigmoid(a.double() @ b.double().T + bias.double())
    assert _rel(out, ref) < 1e-5


@pytest.mark.parametrize("dtype,C", [(torch.bfloat16, 1024), (torch.bfloat16, 640), (torch.bfloat16, 128),
                                     (torch.float32, 64)])
def test_layernorm(K, dtype, C):
    torch.manual_seed(5)
    x = torch.randn(333, C, device="cuda").to(dtype)
    g = (1 + 0.1 * torch.randn(C, device="cuda")).to(dtype)
    b = (0.1 * torch.randn(C, device="cuda")).to(dtype)
    y = torch.empty_like(x)
    K.layernorm(x, g, b, y)
    ref = torch.nn.functional.layer_norm(x.double(), (C,), g.double(), b.double(), 1e-5)
    assert _rel(y, ref) < (1e-2 if dtype == torch.bfloat16 else 1e-5)


@pytest.mark.parametrize("dtype,ncols,causal", [(torch.bfloat16, 16384, 1), (torch.bfloat16, 1024, 0),
                                                (torch.bfloat16, 65536, 0), (torch.float32, 256, 0),
                                                (torch.bfloat16, 2048, 1)])
def test_softmax(K, dtype, ncols, causal):
    torch.manual_seed(6)
    rows = 64 if ncols > 4096 else 300
    row_off = 512 if causal else 0
    s = (3 * torch.randn(rows, ncols, device="cuda")).to(dtype)
    p = torch.full_like(s, 9.0)
    K.softmax(s, p, rows, ncols, ncols, causal, row_off)
    ref = s.double()
    if causal:
        i = torch.arange(rows, device="cuda")[:, None] + row_off
        j = torch.arange(ncols, device="cuda")[None, :]
        ref = torch.where(j <= i, ref, torch.full_like(ref, -float("inf")))
        ref = torch.softmax(ref, -1)
        kend = ((i // 128) + 1) * 128
        written = (j < kend).expand(rows, ncols)
        assert _rel(p[written], ref[written]) < 1e-2
        assert (p[written & (j > i)] == 0).all()
    else:
        assert _rel(p, torch.softmax(ref, -1)) < (1e-2 if dtype == torch.bfloat16 else 1e-5)
