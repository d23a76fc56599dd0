"""Per-node-kind definitions for the oracle (test infrastructure only).

For every IR kind this module gives
  * shape(attrs, in_shapes)           -> output shape
  * flops(attrs, in_shapes, out)      -> integer FLOPs (SPEC S:76 conventions,
                                         extended to the fused kinds)
  * propagate(attrs, in_shapes, out, d) -> per input: int dim | NC | BREAK
                                         (chunk-flow legality, Eq. 4)
  * evaluate(attrs, values, ctx)      -> float64 result (the block maths)

Reductions: in EXACT mode every sum runs sequentially over its index
(k = 0, 1, ..., K-1), so the value of each output element depends only on the
element's own operands — chunking can never change it (Eq. 5).  FAST
mode uses numpy/BLAS (`np.matmul`, `np.sum`) as library primitives; it is used
for large-size parity where the comparison is toleranced.
"""
from __future__ import annotations

import contextlib
import math

import numpy as np
from scipy.special import erf as _erf

NC = "nc"        # input is used whole (non-chunkable for this flow)
BREAK = "break"  # the flow cannot pass this node along this dim

_EXACT = False


@contextlib.contextmanager
def exact_order(on: bool = True):
    global _EXACT
    old = _EXACT
    _EXACT = on
    try:
        yield
    finally:
        _EXACT = old


def is_exact() -> bool:
    return _EXACT


# ---------------------------------------------------------------- primitives
def _bdot(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """a [..., M, K] , b [..., N, K] -> [..., M, N] = sum_k a[...,m,k] b[...,n,k]."""
    if not _EXACT:
        return np.matmul(a, np.swapaxes(b, -1, -2))
    K = a.shape[-1]
    acc = a[..., :, None, 0] * b[..., None, :, 0]
    for k in range(1, K):
        acc = acc + a[..., :, None, k] * b[..., None, :, k]
    return acc


def _sum_axis(x: np.ndarray, axis: int) -> np.ndarray:
    if not _EXACT:
        return np.sum(x, axis=axis)
    x = np.moveaxis(x, axis, -1)
    acc = x[..., 0].copy()
    for i in range(1, x.shape[-1]):
        acc = acc + x[..., i]
    return acc


def _gelu(x):
    # erf-GELU (SURVEY §8(c) reading 16): 1/2 x (1 + erf(x / sqrt 2))
    return 0.5 * x * (1.0 + _erf(x / math.sqrt(2.0)))


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def _softmax(x: np.ndarray, axis: int) -> np.ndarray:
    """Stable softmax: subtract the row max, exponentiate, divide by the sum."""
    m = np.max(x, axis=axis, keepdims=True)
    e = np.exp(x - m)
    s = np.expand_dims(_sum_axis(e, axis), axis)
    return e / s


def _layernorm(x, gamma, beta, naxes: int, eps: float):
    """gamma * (x - mu) / sqrt(var + eps) + beta over the trailing naxes dims,
    biased variance."""
    lead = x.shape[: x.ndim - naxes]
    cnt = int(np.prod(x.shape[x.ndim - naxes:]))
    x2 = x.reshape(lead + (cnt,))
    mu = _sum_axis(x2, -1) / cnt
    xc = x2 - mu[..., None]
    var = _sum_axis(xc * xc, -1) / cnt
    y = xc / np.sqrt(var + eps)[..., None]
    return (y.reshape(x.shape) * gamma) + beta


def _bcast_shape(a, b):
    ra, rb = len(a), len(b)
    r = max(ra, rb)
    out = []
    for i in range(r):
        da = a[i - (r - ra)] if i >= r - ra else 1
        db = b[i - (r - rb)] if i >= r - rb else 1
        if da != db and da != 1 and db != 1:
            raise ValueError(f"broadcast mismatch {a} vs {b}")
        out.append(max(da, db))
    return tuple(out)


def prod(xs) -> int:
    p = 1
    for x in xs:
        p *= int(x)
    return p


# ---------------------------------------------------------------- kinds
ELEMENTWISE2 = ("add", "sub", "mul", "div")
UNARY = ("relu", "gelu", "exp", "sigmoid")
REDUCE = ("reduce_sum", "reduce_mean", "reduce_max")
SOURCE = ("input", "weight")
ALL_KINDS = SOURCE + ("matmul",) + ELEMENTWISE2 + UNARY + ("softmax", "layernorm") + REDUCE + (
    "transpose", "reshape", "concat", "slice",
    "linear", "attn_scores", "attn_pv", "tri_scores", "tri_pv", "attn_fused", "tri_mul", "ln_cfirst")

# attribute schema: name -> type tag ("int", "float", "ints", "str", "ranges")
ATTR_SCHEMA = {
    "softmax": {"dim": "int"},
    "layernorm": {"naxes": "int", "eps": "float"},
    "reduce_sum": {"dim": "int"}, "reduce_mean": {"dim": "int"}, "reduce_max": {"dim": "int"},
    "transpose": {"perm": "ints"},
    "reshape": {"shape": "ints"},
    "concat": {"dim": "int"},
    "slice": {"ranges": "ranges"},
    "linear": {"kin": "int", "out": "ints", "act": "str", "trans": "int", "swap": "int",
               "bias": "int", "res": "int", "gate": "int"},
    "ln_cfirst": {"eps": "float"},
    "attn_scores": {"scale": "float", "causal": "int"},
    "attn_fused": {"scale": "float", "causal": "int"},
    "tri_scores": {"scale": "float", "ending": "int"},
    "tri_pv": {"ending": "int"},
}

ARITY = {"matmul": (2, 2), "softmax": (1, 1), "layernorm": (3, 3), "transpose": (1, 1),
         "reshape": (1, 1), "concat": (1, 64), "slice": (1, 1), "linear": (2, 5),
         "tri_mul": (2, 2), "ln_cfirst": (3, 3),
         "attn_scores": (2, 2), "attn_pv": (2, 2), "tri_scores": (3, 3), "tri_pv": (3, 3),
         "attn_fused": (3, 3)}
for _k in ELEMENTWISE2:
    ARITY[_k] = (2, 2)
for _k in UNARY + REDUCE:
    ARITY[_k] = (1, 1)


def linear_arity(attrs) -> int:
    return 2 + int(attrs.get("bias", 0)) + int(attrs.get("gate", 0)) + int(attrs.get("res", 0))


def _linear_rows(attrs, a_shape):
    kin = attrs["kin"]
    rows = list(a_shape[: len(a_shape) - kin])
    if attrs.get("swap", 0):
        if len(rows) < 2:
            raise ValueError("linear swap needs >= 2 row dims")
        rows[0], rows[1] = rows[1], rows[0]
    return tuple(rows)


def shape(kind: str, attrs: dict, ins) -> tuple:
    """Output shape; raises ValueError on mismatch."""
    ins = [tuple(s) for s in ins]
    if kind == "matmul":
        a, b = ins
        if len(a) < 2 or len(b) < 2:
            raise ValueError("matmul needs rank >= 2")
        if a[-1] != b[-2]:
            raise ValueError(f"inner dimension mismatch {a[-1]}!={b[-2]}")
        if len(b) == 2:
            return a[:-1] + (b[-1],)
        if a[:-2] != b[:-2]:
            raise ValueError("matmul batch mismatch")
        return a[:-1] + (b[-1],)
    if kind in ELEMENTWISE2:
        return _bcast_shape(ins[0], ins[1])
    if kind in UNARY:
        return ins[0]
    if kind == "softmax":
        if not 0 <= attrs["dim"] < len(ins[0]):
            raise ValueError("softmax dim out of range")
        return ins[0]
    if kind == "layernorm":
        x, g, b = ins
        na = attrs["naxes"]
        if not 1 <= na <= len(x) or g != x[len(x) - na:] or b != g:
            raise ValueError("layernorm parameter shape mismatch")
        return x
    if kind in REDUCE:
        d = attrs["dim"]
        if not 0 <= d < len(ins[0]) or len(ins[0]) < 2:
            raise ValueError("reduce dim out of range")
        return ins[0][:d] + ins[0][d + 1:]
    if kind == "transpose":
        p = list(attrs["perm"])
        if sorted(p) != list(range(len(ins[0]))):
            raise ValueError("permutation is not a bijection")
        return tuple(ins[0][i] for i in p)
    if kind == "reshape":
        t = tuple(attrs["shape"])
        if prod(t) != prod(ins[0]) or any(s < 1 for s in t):
            raise ValueError("reshape element-count mismatch")
        return t
    if kind == "concat":
        d = attrs["dim"]
        r = ins[0]
        if not 0 <= d < len(r):
            raise ValueError("concat dim out of range")
        tot = 0
        for s in ins:
            if len(s) != len(r) or any(s[i] != r[i] for i in range(len(r)) if i != d):
                raise ValueError("concat shape mismatch")
            tot += s[d]
        return r[:d] + (tot,) + r[d + 1:]
    if kind == "slice":
        rg = attrs["ranges"]
        if len(rg) != len(ins[0]):
            raise ValueError("slice rank mismatch")
        out = []
        for (s, e), n in zip(rg, ins[0]):
            if not 0 <= s < e <= n:
                raise ValueError("slice range out of bounds")
            out.append(e - s)
        return tuple(out)
    if kind == "linear":
        if len(ins) != linear_arity(attrs):
            raise ValueError("linear arity mismatch")
        a, w = ins[0], ins[1]
        kin = attrs["kin"]
        if not 1 <= kin < len(a) + 0 or len(w) != 2:
            raise ValueError("linear rank mismatch")
        K = prod(a[len(a) - kin:])
        out = tuple(attrs["out"])
        if w != (prod(out), K):
            raise ValueError(f"linear weight shape {w} != {(prod(out), K)}")
        rows = _linear_rows(attrs, a)
        res = out + rows if attrs.get("trans", 0) else rows + out
        i = 2
        if attrs.get("bias", 0):
            if ins[i] != (prod(out),):
                raise ValueError("linear bias shape mismatch")
            i += 1
        if attrs.get("gate", 0):   # elementwise gate in the output's layout
            if ins[i] != res:
                raise ValueError("linear gate shape mismatch")
            i += 1
        if attrs.get("res", 0):
            if ins[i] != res:
                raise ValueError("linear residual shape mismatch")
        if attrs.get("act", "none") not in ("none", "gelu", "sigmoid", "relu"):
            raise ValueError("linear act")
        return res
    if kind == "attn_scores":
        q, k = ins
        if len(q) != 3 or len(k) != 3 or q[1:] != k[1:]:
            raise ValueError("attn_scores shape mismatch")
        return (q[1], q[0], k[0])
    if kind == "attn_pv":
        p, vt = ins
        if len(p) != 3 or len(vt) != 3 or p[0] != vt[0] or p[2] != vt[2]:
            raise ValueError("attn_pv shape mismatch")
        return (p[1], p[0], vt[1])
    if kind == "attn_fused":
        # NEXT f1: attention as one memory-efficient kernel,
        # o = softmax(q k^T * scale) v with no N x N intermediate
        q, k, vt = ins
        if len(q) != 3 or len(k) != 3 or len(vt) != 3 or q[1:] != k[1:] or vt != (k[1], k[2], k[0]):
            raise ValueError("attn_fused shape mismatch")
        return q
    if kind == "tri_scores":
        q, k, b = ins
        if len(q) != 4 or len(k) != 4 or len(b) != 3:
            raise ValueError("tri_scores rank")
        I, J, H, c = q
        if attrs.get("ending", 0):
            # bias given as bT[h, i, k] = b_ki (the projection writes it transposed)
            if k[1:] != (J, H, c) or b != (H, I, k[0]):
                raise ValueError("tri_scores(ending) shape mismatch")
            return (J, H, I, k[0])
        if (k[0], k[2], k[3]) != (I, H, c) or b != (H, J, k[1]):
            raise ValueError("tri_scores shape mismatch")
        return (I, H, J, k[1])
    if kind == "tri_mul":
        # AF2 Alg. 11 / 12 line 4, channel-major: x[c, i, j] = sum_k a[c, i, k] b[c, j, k]
        a, b = ins
        if len(a) != 3 or len(b) != 3 or a[0] != b[0] or a[2] != b[2]:
            raise ValueError("tri_mul shape mismatch")
        return (a[0], a[1], b[1])
    if kind == "ln_cfirst":
        # LayerNorm over the leading (channel) dim, written channel-last:
        # y[i, j, :] = LN(x[:, i, j]) (AF2 Alg. 11 line 4, the LN of the product)
        x, gm, bt = ins
        if len(x) != 3 or gm != (x[0],) or bt != gm:
            raise ValueError("ln_cfirst shape mismatch")
        return (x[1], x[2], x[0])
    if kind == "tri_pv":
        p, vt, g = ins
        if len(p) != 4 or len(vt) != 4 or len(g) != 4:
            raise ValueError("tri_pv rank")
        I, J, H, c = g
        if attrs.get("ending", 0):
            if p[:3] != (J, H, I) or vt != (H, c, J, p[3]):
                raise ValueError("tri_pv(ending) shape mismatch")
        else:
            if p[:3] != (I, H, J) or vt != (H, c, I, p[3]):
                raise ValueError("tri_pv shape mismatch")
        return g
    raise ValueError(f"unknown op kind {kind!r}")


def flops(kind: str, attrs: dict, ins, out) -> int:
    """FLOP model: SPEC S:76 for primitives; a fused kind counts the sum over
    its SPEC-primitive decomposition (S:76 conventions, as SPEC's attention
    corpus writes the scale as a `mul` node): the contraction
    (2 per multiply-add) + one per output element for each elementwise
    epilogue op (scale, causal mask add, bias add, activation, gate, residual).
    Pinned by tests/test_oracle_flops.py, which builds each decomposition."""
    ne = prod(out)
    if kind in SOURCE or kind in ("transpose", "reshape", "concat", "slice"):
        return 0
    if kind == "matmul":
        a = ins[0]
        return 2 * prod(a[:-1]) * a[-1] * out[-1]
    if kind in ELEMENTWISE2 or kind in UNARY:
        return ne
    if kind == "softmax":
        return 5 * ne
    if kind == "layernorm":
        return 8 * ne
    if kind in REDUCE:
        return prod(ins[0])
    if kind == "linear":
        a = ins[0]
        kin = attrs["kin"]
        R = prod(a[: len(a) - kin])
        K = prod(a[len(a) - kin:])
        O = prod(attrs["out"])
        extra = (int(attrs.get("bias", 0)) + int(attrs.get("act", "none") != "none") + int(attrs.get("gate", 0))
                 + int(attrs.get("res", 0)))
        return 2 * R * K * O + R * O * extra
    if kind == "attn_scores":     # matmul + scale mul (+ causal mask add)
        q = ins[0]
        return 2 * ne * q[2] + ne * (1 + int(attrs.get("causal", 0)))
    if kind == "attn_pv":
        p = ins[0]
        return 2 * prod(p) * out[2]
    if kind == "attn_fused":      # the unfused chain: scores + softmax (5/elem) + PV
        q, k = ins[0], ins[1]
        ns = q[1] * q[0] * k[0]
        return 4 * ns * q[2] + ns * (1 + int(attrs.get("causal", 0))) + 5 * ns
    if kind == "tri_scores":      # matmul + scale mul + bias add
        return 2 * ne * ins[0][3] + 2 * ne
    if kind == "tri_pv":
        p = ins[0]
        return 2 * prod(p) * out[3] + ne
    if kind == "tri_mul":         # a batched matmul over channels
        a = ins[0]
        return 2 * prod(a) * out[2]
    if kind == "ln_cfirst":       # transpose (0) + layernorm (8 / element)
        return 8 * ne
    raise ValueError(kind)


def propagate(kind: str, attrs: dict, ins, out, d: int):
    """Chunk-flow map (Eq. 4; SPEC S:229-237 for primitives).
    Returns one entry per input: int dim on that input, NC (used whole) or BREAK."""
    n = len(ins)
    if not 0 <= d < len(out):
        raise ValueError("out_dim out of range")
    if kind == "matmul":
        a, b = ins
        r = len(out)
        if d == r - 2:
            return [len(a) - 2, NC]
        if d == r - 1:
            return [NC, len(b) - 1]
        # batch dim
        return [d, d if len(b) > 2 else NC]
    if kind in ELEMENTWISE2:
        res = []
        for s in ins:
            dd = d - (len(out) - len(s))
            if dd < 0 or (s[dd] == 1 and out[d] != 1):
                res.append(NC)
            else:
                res.append(dd)
        return res
    if kind in UNARY:
        return [d]
    if kind == "softmax":
        return [BREAK] if d == attrs["dim"] else [d]
    if kind == "layernorm":
        na = attrs["naxes"]
        if d >= len(out) - na:
            return [BREAK, BREAK, BREAK]
        return [d, NC, NC]
    if kind in REDUCE:
        return [d if d < attrs["dim"] else d + 1]
    if kind == "transpose":
        return [attrs["perm"][d]]
    if kind == "reshape":
        a = ins[0]
        if d < len(a) and all(a[i] == out[i] for i in range(d + 1)):
            return [d]
        return [BREAK]
    if kind == "concat":
        return [BREAK] * n if d == attrs["dim"] else [d] * n
    if kind == "slice":
        s, e = attrs["ranges"][d]
        return [d] if (s == 0 and e == ins[0][d]) else [BREAK]
    if kind == "linear":
        a = ins[0]
        kin = attrs["kin"]
        nrows = len(a) - kin
        nout = len(attrs["out"])
        rd = d - nout if attrs.get("trans", 0) else d
        if not 0 <= rd < nrows:
            return [BREAK] * n
        ad = rd
        if attrs.get("swap", 0) and rd < 2:
            ad = 1 - rd
        res = [ad, NC]
        if attrs.get("bias", 0):
            res.append(NC)
        if attrs.get("gate", 0):
            res.append(d)
        if attrs.get("res", 0):
            res.append(d)
        return res
    if kind == "attn_scores":
        return [[1, 1], [0, NC], [NC, 0]][d]
    if kind == "attn_pv":
        return [[1, NC], [0, 0], [NC, 1]][d]
    if kind == "attn_fused":
        return [[0, NC, NC], [1, 1, 0], [NC, NC, 1]][d]
    if kind == "tri_mul":
        return [[0, 0], [1, NC], [NC, 1]][d]
    if kind == "ln_cfirst":
        return [[1, NC, NC], [2, NC, NC], [BREAK, BREAK, BREAK]][d]
    if kind == "tri_scores":
        if attrs.get("ending", 0):
            return [[1, 1, NC], [2, 2, 0], [0, NC, 1], [NC, 0, 2]][d]
        return [[0, 0, NC], [2, 2, 0], [1, NC, 1], [NC, 1, 2]][d]
    if kind == "tri_pv":
        if attrs.get("ending", 0):
            return [[2, NC, 0], [0, 2, 1], [1, 0, 2], [NC, 1, 3]][d]
        return [[0, 2, 0], [2, NC, 1], [1, 0, 2], [NC, 1, 3]][d]
    raise ValueError(kind)


def evaluate(kind: str, attrs: dict, vals, ctx=None) -> np.ndarray:
    """float64 value of one node.  ctx = {"dim": chunk dim of the output,
    "offset": global index of the slice's first element along it} — only the
    causal mask reads it (global positions)."""
    ctx = ctx or {}
    if kind == "matmul":
        a, b = vals
        if b.ndim == 2:
            return _bdot(a, np.swapaxes(b, -1, -2)[(None,) * (a.ndim - 2)])
        return _bdot(a, np.swapaxes(b, -1, -2))
    if kind == "add":
        return vals[0] + vals[1]
    if kind == "sub":
        return vals[0] - vals[1]
    if kind == "mul":
        return vals[0] * vals[1]
    if kind == "div":
        return vals[0] / vals[1]
    if kind == "relu":
        return np.maximum(vals[0], 0.0)
    if kind == "gelu":
        return _gelu(vals[0])
    if kind == "exp":
        return np.exp(vals[0])
    if kind == "sigmoid":
        return _sigmoid(vals[0])
    if kind == "softmax":
        return _softmax(vals[0], attrs["dim"])
    if kind == "layernorm":
        return _layernorm(vals[0], vals[1], vals[2], attrs["naxes"], attrs["eps"])
    if kind == "reduce_sum":
        return _sum_axis(vals[0], attrs["dim"])
    if kind == "reduce_mean":
        return _sum_axis(vals[0], attrs["dim"]) / vals[0].shape[attrs["dim"]]
    if kind == "reduce_max":
        return np.max(vals[0], axis=attrs["dim"])
    if kind == "transpose":
        return np.ascontiguousarray(np.transpose(vals[0], attrs["perm"]))
    if kind == "reshape":
        t = list(attrs["shape"])
        if "dim" in ctx:          # a chunk of the flow dim (leading dims preserved)
            t[ctx["dim"]] = vals[0].shape[ctx["dim"]]
        return np.reshape(vals[0], tuple(t))
    if kind == "concat":
        return np.concatenate(vals, axis=attrs["dim"])
    if kind == "slice":
        rg = [slice(s, e) for s, e in attrs["ranges"]]
        if "dim" in ctx:          # the flow dim is never sliced (propagate), keep the chunk
            rg[ctx["dim"]] = slice(None)
        return vals[0][tuple(rg)].copy()
    if kind == "linear":
        return _linear(attrs, vals)
    if kind == "attn_scores":
        q, k = vals
        s = _bdot(np.transpose(q, (1, 0, 2)), np.transpose(k, (1, 0, 2))) * attrs["scale"]
        if attrs.get("causal", 0):
            roff = ctx.get("offset", 0) if ctx.get("dim") == 1 else 0
            coff = ctx.get("offset", 0) if ctx.get("dim") == 2 else 0
            i = np.arange(s.shape[1])[:, None] + roff
            j = np.arange(s.shape[2])[None, :] + coff
            s = np.where((j > i)[None], -np.inf, s)
        return s
    if kind == "attn_pv":
        p, vt = vals
        o = _bdot(p, vt)              # [h, N, dh]
        return np.ascontiguousarray(np.transpose(o, (1, 0, 2)))
    if kind == "attn_fused":
        # the unfused chain written out: scores (row offset of a row chunk in ctx,
        # as for attn_scores' dim 1), softmax over keys, PV
        q, k, vt = vals
        c2 = dict(ctx or {})
        if c2.get("dim") == 0:
            c2["dim"] = 1        # o's row dim is the scores' row dim
        elif "dim" in c2:
            c2.pop("dim")
        s = evaluate("attn_scores", {"scale": attrs["scale"], "causal": attrs.get("causal", 0)}, [q, k], c2)
        p = _softmax(s, 2)
        return evaluate("attn_pv", {}, [p, vt])
    if kind == "tri_scores":
        q, k, b = vals
        sc = attrs["scale"]
        if attrs.get("ending", 0):
            Q = np.transpose(q, (1, 2, 0, 3))   # [J,H,I,c]
            Kk = np.transpose(k, (1, 2, 0, 3))  # [J,H,K,c]
            return _bdot(Q, Kk) * sc + b[None]            # b = bT[h, i, k] = b_ki
        Q = np.transpose(q, (0, 2, 1, 3))       # [I,H,J,c]
        Kk = np.transpose(k, (0, 2, 1, 3))      # [I,H,K,c]
        return _bdot(Q, Kk) * sc + b[None]
    if kind == "tri_mul":
        a, b = vals
        return _bdot(a, b)                       # [C, I, K] x [C, J, K] -> [C, I, J]
    if kind == "ln_cfirst":
        x, gm, bt = vals
        return _layernorm(np.moveaxis(x, 0, -1), gm, bt, 1, attrs["eps"])
    if kind == "tri_pv":
        p, vt, g = vals
        V = np.transpose(vt, (2, 0, 1, 3))      # [I|J, H, c, K]
        o = _bdot(p, V)                          # ending=0: [I,H,J,c]; ending=1: [J,H,I,c]
        if attrs.get("ending", 0):
            o = np.transpose(o, (2, 0, 1, 3))
        else:
            o = np.transpose(o, (0, 2, 1, 3))
        return o * g
    raise ValueError(kind)


def _linear(attrs, vals):
    a, w = vals[0], vals[1]
    kin = attrs["kin"]
    if attrs.get("swap", 0):
        a = np.swapaxes(a, 0, 1)
    rows = a.shape[: a.ndim - kin]
    K = prod(a.shape[a.ndim - kin:])
    a2 = np.ascontiguousarray(a).reshape((prod(rows), K))
    acc = _bdot(a2, w)                           # [R, O]
    i = 2
    if attrs.get("bias", 0):
        acc = acc + vals[i][None, :]
        i += 1
    act = attrs.get("act", "none")
    if act == "gelu":
        acc = _gelu(acc)
    elif act == "sigmoid":
        acc = _sigmoid(acc)
    elif act == "relu":
        acc = np.maximum(acc, 0.0)
    out = tuple(attrs["out"])
    y = acc.reshape(tuple(rows) + out)
    if attrs.get("trans", 0):
        nr = len(rows)
        y = np.ascontiguousarray(np.transpose(y, tuple(range(nr, nr + len(out))) + tuple(range(nr))))
    if attrs.get("gate", 0):
        y = y * vals[i]
        i += 1
    if attrs.get("res", 0):
        y = y + vals[i]
    return y
