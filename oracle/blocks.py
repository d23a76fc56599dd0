"""Sampled-row oracle for the transformer blocks at full size (test infrastructure only).

Every op of the pre-LN block except attention is row-wise in the token index,
and attention row i needs only q_i plus the full K and V (SURVEY §8(c) c.3,
"Sampled-row parity").  So output row i is a plain definition of its own:
    a = LN1(x); k = a Wk + bk; v = a Wv + bv            (all rows)
    q_i = a_i Wq + bq; s_i = q_i k^T / sqrt(dh) (causal: j > i -> -inf)
    o_i = softmax(s_i) v; x1_i = x_i + o_i Wo + bo; y_i = x1_i + GELU(LN2(x1_i) W1 + b1) W2 + b2
It evaluates the same node definitions as executor.run (oracle.ops), restricted
to the requested rows.
"""
from __future__ import annotations

import numpy as np

from . import ops
from .graph import Graph


def transformer_rows(g: Graph, v: dict, rows) -> dict:
    """Values of the region output o and block output (x1 or y) at `rows`."""
    rows = np.asarray(rows, dtype=np.int64)
    nd = {n.id: n for n in g.nodes}
    ev = lambda nid, vals: ops.evaluate(nd[nid].kind, nd[nid].attrs, vals)  # noqa: E731
    a = ev("ln1", [v["x"], v["ln1_g"], v["ln1_b"]])
    k = ev("proj_k", [a, v["wk"], v["bk"]])
    vt = ev("proj_v", [a, v["wv"], v["bv"]])
    q = ev("proj_q", [a[rows], v["wq"], v["bq"]])
    sc = nd["scores"].attrs
    s = ops.evaluate("attn_scores", {"scale": sc["scale"], "causal": 0}, [q, k])
    if sc.get("causal", 0):
        j = np.arange(k.shape[0])[None, :]
        s = np.where((j > rows[:, None])[None], -np.inf, s)
    p = ev("softmax", [s])
    o = ev("pv", [p, vt])
    x1 = ev("proj_o", [o, v["wo"], v["bo"], v["x"][rows]])
    out = {"o": o, "x1": x1}
    if "ffn2" in nd:
        c = ev("ln2", [x1, v["ln2_g"], v["ln2_b"]])
        hid = ev("ffn1", [c, v["w1"], v["b1"]])
        out["y"] = ev("ffn2", [hid, v["w2"], v["b2"], x1])
    return out


def sample_rows(N: int, chunk_len: int, n_random: int = 64, seed: int = 0):
    """First, last, every chunk boundary +-1, plus random rows."""
    rng = np.random.default_rng(seed)
    s = {0, N - 1}
    for b in range(chunk_len, N, chunk_len):
        s.update({b - 1, b})
    s.update(int(x) for x in rng.integers(0, N, n_random))
    return np.array(sorted(x for x in s if 0 <= x < N), dtype=np.int64)


def tri_attention_pairs(g: Graph, v: dict, pre: str, pairs, ending: bool) -> np.ndarray:
    """Outputs z_out[i, j] of one triangle attention (AF2 Alg. 13 starting node, or
    Alg. 14 ending node) at the sampled (i, j) pairs, from the same node definitions
    as executor.run restricted to what each pair reads:
      starting node: q[i, j], k[i, :], v[i, :], g[i, j], bias b[h, j, :] (zn row j)
      ending node:   q[i, j], k[:, j], v[:, j], g[i, j], bias b_ki = (zn[:, i] W_b)"""
    nd = {n.id: n for n in g.nodes}
    ev = lambda nid, vals: ops.evaluate(nd[nid].kind, nd[nid].attrs, vals)  # noqa: E731
    z = v["z"] if "z" in v else None
    zin = [n for n in g.nodes if n.id == pre + "ln"][0].inputs[0]
    z = v[zin] if zin in v else z
    ln = lambda t: ev(pre + "ln", [t, v[pre + "ln_g"], v[pre + "ln_b"]])  # noqa: E731
    wq, wk, wv, wg, wb = (v[pre + w] for w in ("wq", "wk", "wv", "wg", "wb"))
    H = wb.shape[0]
    c = wq.shape[0] // H
    scale = nd[pre + "scores"].attrs["scale"]
    out = []
    for i, j in pairs:
        zn_ij = ln(z[i, j][None])[0]
        q = (zn_ij @ wq.T).reshape(H, c)
        gt = 1.0 / (1.0 + np.exp(-(zn_ij @ wg.T + v[pre + "bg"]))).reshape(H, c)
        if not ending:
            zr = ln(z[i])                       # row i: keys / values k[i, :], v[i, :]
            kk = (zr @ wk.T).reshape(-1, H, c)
            vv = (zr @ wv.T).reshape(-1, H, c)
            b = ln(z[j]) @ wb.T                 # b[j, k, h] = zn[j, k] . w_b
        else:
            zc = ln(z[:, j])                    # column j: k[:, j], v[:, j]
            kk = (zc @ wk.T).reshape(-1, H, c)
            vv = (zc @ wv.T).reshape(-1, H, c)
            b = ln(z[:, i]) @ wb.T              # b_ki = zn[k, i] . w_b
        s = np.einsum("hc,khc->hk", q, kk) * scale + b.T
        s = s - s.max(-1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(-1, keepdims=True)
        o = gt * np.einsum("hk,khc->hc", p, vv)
        out.append(z[i, j] + o.reshape(-1) @ v[pre + "wo"].T + v[pre + "bo"])
    return np.stack(out)
