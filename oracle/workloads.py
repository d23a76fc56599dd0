"""Graphs of the BASELINE.json configurations and the SPEC desk-scale corpus
(oracle side; test infrastructure only).  The C++ library builds the same
graphs independently (ac_graph_block); tests compare the two documents.

Kernel-granularity node kinds; weights use the nn.Linear
layout W[out, in].  Block maths = SURVEY §8(c) O1; AlphaFold triangle
attention follows AF2 supplement Alg. 13 (starting node) / Alg. 14 (ending
node) — DESIGN.md reading R16.
"""
from __future__ import annotations

import math

from .graph import Builder, Graph


def _transformer_block(B: Builder, d, h, f, causal, attn_only, eps, pre: str, xin: str, fused=False) -> str:
    """Pre-LN block reading `xin`: a = LN1(x); q,k,v = a W + b; softmax(q k^T / sqrt(dh)) v;
    x1 = x + o Wo + bo; (y = x1 + GELU(LN2(x1) W1 + b1) W2 + b2).  Every other id
    carries the prefix `pre`; returns the output id."""
    dh = d // h
    P = (lambda s: pre + s)
    B.weight(P("ln1_g"), (d,), "ln_gamma", d)
    B.weight(P("ln1_b"), (d,), "ln_beta", d)
    for nm in ("q", "k", "v", "o"):
        B.weight(P(f"w{nm}"), (d, d), "matrix", d)
        B.weight(P(f"b{nm}"), (d,), "bias", d)
    if not attn_only:
        B.weight(P("ln2_g"), (d,), "ln_gamma", d)
        B.weight(P("ln2_b"), (d,), "ln_beta", d)
        B.weight(P("w1"), (f, d), "matrix", d)
        B.weight(P("b1"), (f,), "bias", d)
        B.weight(P("w2"), (d, f), "matrix", f)
        B.weight(P("b2"), (d,), "bias", f)
    B.op("layernorm", [xin, P("ln1_g"), P("ln1_b")], P("a"), nid=P("ln1"), naxes=1, eps=eps)
    B.op("linear", [P("a"), P("wq"), P("bq")], P("q"), nid=P("proj_q"), kin=1, out=[h, dh], act="none",
         trans=0, swap=0, bias=1, res=0)
    B.op("linear", [P("a"), P("wk"), P("bk")], P("k"), nid=P("proj_k"), kin=1, out=[h, dh], act="none",
         trans=0, swap=0, bias=1, res=0)
    B.op("linear", [P("a"), P("wv"), P("bv")], P("vt"), nid=P("proj_v"), kin=1, out=[h, dh], act="none",
         trans=1, swap=0, bias=1, res=0)
    if fused:  # NEXT f1: memory-efficient attention kernel, no N x N tensor
        B.op("attn_fused", [P("q"), P("k"), P("vt")], P("o"), nid=P("attn"), scale=1.0 / math.sqrt(dh),
             causal=int(causal))
    else:
        B.op("attn_scores", [P("q"), P("k")], P("s"), nid=P("scores"), scale=1.0 / math.sqrt(dh),
             causal=int(causal))
        B.op("softmax", [P("s")], P("p"), nid=P("softmax"), dim=2)
        B.op("attn_pv", [P("p"), P("vt")], P("o"), nid=P("pv"))
    B.op("linear", [P("o"), P("wo"), P("bo"), xin], P("x1"), nid=P("proj_o"), kin=2, out=[d], act="none",
         trans=0, swap=0, bias=1, res=1)
    if attn_only:
        return P("x1")
    B.op("layernorm", [P("x1"), P("ln2_g"), P("ln2_b")], P("c"), nid=P("ln2"), naxes=1, eps=eps)
    B.op("linear", [P("c"), P("w1"), P("b1")], P("hid"), nid=P("ffn1"), kin=1, out=[f], act="gelu", trans=0,
         swap=0, bias=1, res=0)
    B.op("linear", [P("hid"), P("w2"), P("b2"), P("x1")], P("y"), nid=P("ffn2"), kin=1, out=[d], act="none",
         trans=0, swap=0, bias=1, res=1)
    return P("y")


def _prefix(layers: int, i: int) -> str:
    """Id prefix of block i in a stack of `layers` blocks (none for a single block)."""
    return f"L{i}_" if layers > 1 else ""


def transformer(N, d, h, f=0, causal=False, dtype="bf16", attn_only=False, name="transformer",
                eps=1e-5, layers=1, fused=False) -> Graph:
    """`layers` pre-LN blocks in sequence (NEXT f3 stacks; one block by default);
    fused: attention as one attn_fused node (NEXT f1)."""
    B = Builder(name, dtype)
    B.input("x", (N, d))
    x = "x"
    for i in range(max(1, layers)):
        x = _transformer_block(B, d, h, f, causal, attn_only, eps, _prefix(layers, i), x, fused)
    B.output(x)
    return B.build()


def _tri_weights(B: Builder, pre: str, cz: int, H: int, c: int):
    for nm, shp, role, fan in (("ln_g", (cz,), "ln_gamma", cz), ("ln_b", (cz,), "ln_beta", cz),
                               ("wb", (H, cz), "matrix", cz), ("wq", (H * c, cz), "matrix", cz),
                               ("wk", (H * c, cz), "matrix", cz), ("wv", (H * c, cz), "matrix", cz),
                               ("wg", (H * c, cz), "matrix", cz), ("bg", (H * c,), "bias", cz),
                               ("wo", (cz, H * c), "matrix", H * c), ("bo", (cz,), "bias", H * c)):
        B.weight(pre + nm, shp, role, fan)


def _tri_attention(B: Builder, z: str, pre: str, N: int, cz: int, H: int, c: int, ending: int,
                   out: str, eps=1e-5):
    zn, b, q, k, vt, g = (pre + s for s in ("zn", "bias", "q", "k", "vt", "g"))
    B.op("layernorm", [z, pre + "ln_g", pre + "ln_b"], zn, nid=pre + "ln", naxes=1, eps=eps)
    # ending node: the bias is used as b_ki (Alg. 14), written transposed (swap) so the
    # scores epilogue reads it contiguously along the key index
    B.op("linear", [zn, pre + "wb"], b, nid=pre + "proj_b", kin=1, out=[H], act="none", trans=1,
         swap=int(ending), bias=0, res=0)
    B.op("linear", [zn, pre + "wq"], q, nid=pre + "proj_q", kin=1, out=[H, c], act="none", trans=0,
         swap=0, bias=0, res=0)
    B.op("linear", [zn, pre + "wk"], k, nid=pre + "proj_k", kin=1, out=[H, c], act="none", trans=0,
         swap=0, bias=0, res=0)
    B.op("linear", [zn, pre + "wv"], vt, nid=pre + "proj_v", kin=1, out=[H, c], act="none", trans=1,
         swap=int(ending), bias=0, res=0)
    B.op("linear", [zn, pre + "wg", pre + "bg"], g, nid=pre + "proj_g", kin=1, out=[H, c],
         act="sigmoid", trans=0, swap=0, bias=1, res=0)
    B.op("tri_scores", [q, k, b], pre + "s", nid=pre + "scores", scale=1.0 / math.sqrt(c),
         ending=int(ending))
    B.op("softmax", [pre + "s"], pre + "p", nid=pre + "softmax", dim=3)
    B.op("tri_pv", [pre + "p", vt, g], pre + "o", nid=pre + "pv", ending=int(ending))
    B.op("linear", [pre + "o", pre + "wo", pre + "bo", z], out, nid=pre + "proj_o", kin=2, out=[cz],
         act="none", trans=0, swap=0, bias=1, res=1)


def tri_attn_pair(N, cz=128, H=4, c=32, dtype="bf16", name="af_pair", layers=1) -> Graph:
    """Triangle attention around the starting node (rows, Alg. 13) followed by
    the ending node (columns, Alg. 14), each with its residual add; `layers`
    such pairs in sequence."""
    B = Builder(name, dtype)
    B.input("z", (N, N, cz))
    z = "z"
    for i in range(max(1, layers)):
        p = _prefix(layers, i)
        _tri_weights(B, p + "row_", cz, H, c)
        _tri_weights(B, p + "col_", cz, H, c)
        _tri_attention(B, z, p + "row_", N, cz, H, c, 0, p + "z1")
        _tri_attention(B, p + "z1", p + "col_", N, cz, H, c, 1, p + "z2")
        z = p + "z2"
    B.output(z)
    return B.build()


def _tri_mul(B: Builder, z: str, pre: str, cz: int, cm: int, incoming: int, out: str, eps=1e-5):
    """Triangular multiplicative update, AF2 supplement Alg. 11 (outgoing edges,
    x_ij = sum_k a_ik b_jk) / Alg. 12 (incoming, x_ij = sum_k a_ki b_jk):
    zn = LN(z); a = sigmoid(Linear(zn)) * Linear(zn); b likewise; g = sigmoid(Linear(zn));
    z + g * Linear(LN(x)).  a and b are written channel-major [c, i, k] ([c, j, k])
    so the product is a batched K-major GEMM; the incoming edges read z transposed
    (`swap`), so both updates share one kind (tri_mul)."""
    P = (lambda s_: pre + s_)
    for nm, shp, role, fan in (("ln_g", (cz,), "ln_gamma", cz), ("ln_b", (cz,), "ln_beta", cz),
                               ("wag", (cm, cz), "matrix", cz), ("bag", (cm,), "bias", cz),
                               ("wa", (cm, cz), "matrix", cz), ("ba", (cm,), "bias", cz),
                               ("wbg", (cm, cz), "matrix", cz), ("bbg", (cm,), "bias", cz),
                               ("wb", (cm, cz), "matrix", cz), ("bb", (cm,), "bias", cz),
                               ("wg", (cz, cz), "matrix", cz), ("bg", (cz,), "bias", cz),
                               ("lnx_g", (cm,), "ln_gamma", cm), ("lnx_b", (cm,), "ln_beta", cm),
                               ("wo", (cz, cm), "matrix", cm), ("bo", (cz,), "bias", cm)):
        B.weight(P(nm), shp, role, fan)
    B.op("layernorm", [z, P("ln_g"), P("ln_b")], P("zn"), nid=P("ln"), naxes=1, eps=eps)
    sw = int(incoming)
    B.op("linear", [P("zn"), P("wag"), P("bag")], P("ag"), nid=P("proj_ag"), kin=1, out=[cm], act="sigmoid",
         trans=1, swap=sw, bias=1, res=0)
    B.op("linear", [P("zn"), P("wa"), P("ba"), P("ag")], P("a"), nid=P("proj_a"), kin=1, out=[cm], act="none",
         trans=1, swap=sw, bias=1, res=0, gate=1)
    B.op("linear", [P("zn"), P("wbg"), P("bbg")], P("bgt"), nid=P("proj_bg"), kin=1, out=[cm], act="sigmoid",
         trans=1, swap=sw, bias=1, res=0)
    B.op("linear", [P("zn"), P("wb"), P("bb"), P("bgt")], P("b"), nid=P("proj_b"), kin=1, out=[cm], act="none",
         trans=1, swap=sw, bias=1, res=0, gate=1)
    B.op("linear", [P("zn"), P("wg"), P("bg")], P("g"), nid=P("proj_g"), kin=1, out=[cz], act="sigmoid",
         trans=0, swap=0, bias=1, res=0)
    B.op("tri_mul", [P("a"), P("b")], P("x"), nid=P("mul"))
    B.op("ln_cfirst", [P("x"), P("lnx_g"), P("lnx_b")], P("xn"), nid=P("lnx"), eps=eps)
    B.op("linear", [P("xn"), P("wo"), P("bo"), P("g"), z], out, nid=P("proj_o"), kin=1, out=[cz], act="none",
         trans=0, swap=0, bias=1, res=1, gate=1)


def _transition(B: Builder, z: str, pre: str, cz: int, nf: int, out: str, eps=1e-5):
    """Pair transition, AF2 Alg. 15: z + Linear(relu(Linear(LN(z)))), hidden n * c_z."""
    P = (lambda s_: pre + s_)
    for nm, shp, role, fan in (("ln_g", (cz,), "ln_gamma", cz), ("ln_b", (cz,), "ln_beta", cz),
                               ("w1", (nf * cz, cz), "matrix", cz), ("b1", (nf * cz,), "bias", cz),
                               ("w2", (cz, nf * cz), "matrix", nf * cz), ("b2", (cz,), "bias", nf * cz)):
        B.weight(P(nm), shp, role, fan)
    B.op("layernorm", [z, P("ln_g"), P("ln_b")], P("zn"), nid=P("ln"), naxes=1, eps=eps)
    B.op("linear", [P("zn"), P("w1"), P("b1")], P("h"), nid=P("ffn1"), kin=1, out=[nf * cz], act="relu",
         trans=0, swap=0, bias=1, res=0)
    B.op("linear", [P("h"), P("w2"), P("b2"), z], out, nid=P("ffn2"), kin=1, out=[cz], act="none",
         trans=0, swap=0, bias=1, res=1)


def evoformer_pair(N, cz=128, H=4, c=32, dtype="bf16", name="evoformer_pair", layers=1, cm=128, nf=4) -> Graph:
    """The Evoformer pair stack (AF2 Alg. 6 lines 13-17, dropout at inference =
    identity): z += TriangleMultiplicationOutgoing(z); z += ...Incoming(z);
    z += TriangleAttentionStartingNode(z); z += ...EndingNode(z); z += PairTransition(z);
    `layers` such stacks in sequence."""
    B = Builder(name, dtype)
    B.input("z", (N, N, cz))
    z = "z"
    for i in range(max(1, layers)):
        p = _prefix(layers, i)
        _tri_mul(B, z, p + "mo_", cz, cm, 0, p + "z1")
        _tri_mul(B, p + "z1", p + "mi_", cz, cm, 1, p + "z2")
        _tri_weights(B, p + "row_", cz, H, c)
        _tri_weights(B, p + "col_", cz, H, c)
        _tri_attention(B, p + "z2", p + "row_", N, cz, H, c, 0, p + "z3")
        _tri_attention(B, p + "z3", p + "col_", N, cz, H, c, 1, p + "z4")
        _transition(B, p + "z4", p + "tr_", cz, nf, p + "z5")
        z = p + "z5"
    B.output(z)
    return B.build()


CONFIGS = {
    # BASELINE.json configs[0..4]
    "tiny": dict(kind="transformer", N=256, d=64, h=2, f=256, causal=False, dtype="f32"),
    "gpt": dict(kind="transformer", N=16384, d=1024, h=16, f=4096, causal=True, dtype="bf16"),
    "vit": dict(kind="transformer", N=65536, d=1024, h=16, f=4096, causal=False, dtype="bf16"),
    "af": dict(kind="evoformer_pair", N=1024, d=128, h=4, f=32, causal=False, dtype="bf16"),
    "af_attn": dict(kind="tri_attn_pair", N=1024, d=128, h=4, f=32, causal=False, dtype="bf16"),
    "unet": dict(kind="attn_only", N=16384, d=640, h=10, f=0, causal=False, dtype="bf16"),
    "unet_h8": dict(kind="attn_only", N=16384, d=640, h=8, f=0, causal=False, dtype="bf16"),
    # NEXT f1: the GPT block with a fused attention kernel (the paper's second regime)
    "gpt_fa": dict(kind="transformer_fa", N=16384, d=1024, h=16, f=4096, causal=True, dtype="bf16"),
}


def block(kind, N, d, h, f=0, causal=False, dtype="bf16", name=None, layers=1) -> Graph:
    if kind == "transformer":
        return transformer(N, d, h, f, causal, dtype, False, name or "transformer", layers=layers)
    if kind == "attn_only":
        return transformer(N, d, h, 0, causal, dtype, True, name or "attn_only", layers=layers)
    if kind == "transformer_fa":
        return transformer(N, d, h, f, causal, dtype, False, name or "transformer_fa", layers=layers, fused=True)
    if kind == "attn_only_fa":
        return transformer(N, d, h, 0, causal, dtype, True, name or "attn_only_fa", layers=layers, fused=True)
    if kind == "tri_attn_pair":
        return tri_attn_pair(N, d, h, f, dtype, name or "af_pair", layers=layers)
    if kind == "evoformer_pair":
        return evoformer_pair(N, d, h, f, dtype, name or "evoformer_pair", layers=layers)
    raise ValueError(kind)


def config(name: str, **over) -> Graph:
    c = dict(CONFIGS[name])
    c.update(over)
    return block(c["kind"], c["N"], c["d"], c["h"], c["f"], c["causal"], c["dtype"], name)


# ----------------------------------------------------------- SPEC corpus
def corpus(name: str, seq=64, d=32, dtype="f64") -> Graph:
    """Desk-scale graphs from SPEC's primitive op set (mlp, attention,
    transformer2, alphafold_like_2d)."""
    B = Builder(name, dtype)
    if name == "mlp":
        B.input("x", (seq, d))
        B.weight("w1", (d, 4 * d), "matrix", d)
        B.weight("w2", (4 * d, d), "matrix", 4 * d)
        B.op("matmul", ["x", "w1"], "h1")
        B.op("relu", ["h1"], "h2")
        B.op("matmul", ["h2", "w2"], "y")
        B.output("y")
    elif name == "attention":
        B.input("x", (seq, d))
        for w in ("wq", "wk", "wv", "wo"):
            B.weight(w, (d, d), "matrix", d)
        B.weight("scale", (1,), "bias", 1)
        _spec_attn(B, "x", "", "y")
        B.output("y")
    elif name == "transformer2":
        B.input("x", (seq, d))
        cur = "x"
        for blk in range(2):
            p = f"b{blk}_"
            B.weight(p + "g1", (d,), "ln_gamma", d)
            B.weight(p + "be1", (d,), "ln_beta", d)
            for w in ("wq", "wk", "wv", "wo"):
                B.weight(p + w, (d, d), "matrix", d)
            B.weight(p + "scale", (1,), "bias", 1)
            B.weight(p + "g2", (d,), "ln_gamma", d)
            B.weight(p + "be2", (d,), "ln_beta", d)
            B.weight(p + "w1", (d, 2 * d), "matrix", d)
            B.weight(p + "w2", (2 * d, d), "matrix", 2 * d)
            B.op("layernorm", [cur, p + "g1", p + "be1"], p + "a", naxes=1, eps=1e-5)
            _spec_attn(B, p + "a", p, p + "att")
            B.op("add", [cur, p + "att"], p + "x1")
            B.op("layernorm", [p + "x1", p + "g2", p + "be2"], p + "c", naxes=1, eps=1e-5)
            B.op("matmul", [p + "c", p + "w1"], p + "h")
            B.op("gelu", [p + "h"], p + "hg")
            B.op("matmul", [p + "hg", p + "w2"], p + "m")
            B.op("add", [p + "x1", p + "m"], p + "out")
            cur = p + "out"
        B.output(cur)
    elif name == "alphafold_like_2d":
        L = seq
        B.input("z", (L, L, d))
        B.weight("w1", (d, d), "matrix", d)
        B.weight("w2", (d, d), "matrix", d)
        B.op("matmul", ["z", "w1"], "u")
        B.op("softmax", ["u"], "r", dim=1)
        B.op("mul", ["r", "z"], "rz")
        B.op("add", ["z", "rz"], "z1")
        B.op("matmul", ["z1", "w2"], "w")
        B.op("softmax", ["w"], "cc", dim=0)
        B.op("mul", ["cc", "z1"], "cz")
        B.op("add", ["z1", "cz"], "z2")
        B.output("z2")
    else:
        raise ValueError(f"unknown corpus {name}")
    return B.build()


def _spec_attn(B: Builder, x, p, out):
    B.op("matmul", [x, p + "wq"], p + "q")
    B.op("matmul", [x, p + "wk"], p + "k")
    B.op("matmul", [x, p + "wv"], p + "v")
    B.op("transpose", [p + "k"], p + "kt", perm=[1, 0])
    B.op("matmul", [p + "q", p + "kt"], p + "s")
    B.op("mul", [p + "s", p + "scale"], p + "ss")
    B.op("softmax", [p + "ss"], p + "pr", dim=1)
    B.op("matmul", [p + "pr", p + "v"], p + "o")
    B.op("matmul", [p + "o", p + "wo"], out)
