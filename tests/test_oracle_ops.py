"""Pins for the oracle's block maths (SURVEY §8(c) c.3 "O1 block forward").

Each pin comes from outside the oracle: torch.nn.functional in fp64 (library
routines), closed forms and the paper's/SPEC's worked examples."""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import executor, graph, ops, workloads
from oracle.graph import Builder, GraphError
import synth


def _values(g, seed=0):
    return {t: s.value for t, s in synth.make_inputs(g.input_specs(), seed).items()}


def _torch_transformer(v, N, d, h, causal, attn_only):
    """Same block through torch.nn.functional (fp64 CPU): layer_norm, linear,
    scaled_dot_product_attention, gelu(approximate='none')."""
    T = {k: torch.from_numpy(np.asarray(a, dtype=np.float64)) for k, a in v.items()}
    dh = d // h
    x = T["x"]
    a = F.layer_norm(x, (d,), T["ln1_g"], T["ln1_b"], eps=1e-5)
    q = F.linear(a, T["wq"], T["bq"]).view(N, h, dh).transpose(0, 1)
    k = F.linear(a, T["wk"], T["bk"]).view(N, h, dh).transpose(0, 1)
    vv = F.linear(a, T["wv"], T["bv"]).view(N, h, dh).transpose(0, 1)
    with torch.nn.attention.sdpa_kernel(torch.nn.attention.SDPBackend.MATH):
        o = F.scaled_dot_product_attention(q[None], k[None], vv[None], is_causal=causal)[0]
    o = o.transpose(0, 1).reshape(N, d)
    x1 = x + F.linear(o, T["wo"], T["bo"])
    if attn_only:
        return x1.numpy()
    c = F.layer_norm(x1, (d,), T["ln2_g"], T["ln2_b"], eps=1e-5)
    hid = F.gelu(F.linear(c, T["w1"], T["b1"]), approximate="none")
    return (x1 + F.linear(hid, T["w2"], T["b2"])).numpy()


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("attn_only", [False, True])
def test_transformer_matches_torch_functional(causal, attn_only):
    N, d, h, f = 48, 32, 4, 64
    g = workloads.block("attn_only" if attn_only else "transformer", N, d, h, f, causal, "f64")
    v = _values(g)
    ours = executor.run(g, v)[g.outputs[0]]
    ref = _torch_transformer(v, N, d, h, causal, attn_only)
    np.testing.assert_allclose(ours, ref, rtol=0, atol=1e-12)


def _torch_tri_attention(z, W, ending):
    """AF2 Alg. 13 (starting node) / Alg. 14 (ending node) via torch einsum."""
    T = {k: torch.from_numpy(np.asarray(a, dtype=np.float64)) for k, a in W.items()}
    z = torch.from_numpy(z)
    N, _, cz = z.shape
    H = T["wb"].shape[0]
    c = T["wq"].shape[0] // H
    zn = F.layer_norm(z, (cz,), T["ln_g"], T["ln_b"], eps=1e-5)
    q = (zn @ T["wq"].T).view(N, N, H, c)
    k = (zn @ T["wk"].T).view(N, N, H, c)
    v = (zn @ T["wv"].T).view(N, N, H, c)
    b = zn @ T["wb"].T                                   # [N, N, H] : b[j,k,h]
    g = torch.sigmoid(zn @ T["wg"].T + T["bg"]).view(N, N, H, c)
    if not ending:   # a_ijk = softmax_k(q_ij . k_ik / sqrt c + b_jk)
        logits = torch.einsum("ijhc,ikhc->ihjk", q, k) / math.sqrt(c) + b.permute(2, 0, 1)[None]
        a = torch.softmax(logits, dim=-1)
        o = torch.einsum("ihjk,ikhc->ijhc", a, v)
    else:            # a_ijk = softmax_k(q_ij . k_kj / sqrt c + b_ki)
        logits = torch.einsum("ijhc,kjhc->jhik", q, k) / math.sqrt(c) + b.permute(2, 1, 0)[None]
        a = torch.softmax(logits, dim=-1)
        o = torch.einsum("jhik,kjhc->ijhc", a, v)
    o = g * o
    return (z + o.reshape(N, N, H * c) @ T["wo"].T + T["bo"]).numpy()


def test_triangle_attention_matches_af2_algorithms():
    N, cz, H, c = 12, 16, 2, 8
    g = workloads.tri_attn_pair(N, cz, H, c, "f64")
    v = _values(g, 3)
    env = executor.run(g, v, keep_all=True)
    rw = {k[4:]: v[k] for k in v if k.startswith("row_")}
    cw = {k[4:]: v[k] for k in v if k.startswith("col_")}
    z1 = _torch_tri_attention(v["z"], rw, ending=False)
    np.testing.assert_allclose(env["z1"], z1, rtol=0, atol=1e-12)
    z2 = _torch_tri_attention(z1, cw, ending=True)
    np.testing.assert_allclose(env["z2"], z2, rtol=0, atol=1e-12)


def test_ending_node_is_starting_node_on_transpose():
    """Alg. 14 on z equals Alg. 13 on z^T, transposed back (AF2 construction)."""
    N, cz, H, c = 10, 8, 2, 4
    g = workloads.tri_attn_pair(N, cz, H, c, "f64")
    v = _values(g, 5)
    env = executor.run(g, v, keep_all=True)
    # run the row block with the column weights on z1^T
    gr = workloads.tri_attn_pair(N, cz, H, c, "f64")
    v2 = dict(v)
    v2["z"] = np.ascontiguousarray(np.transpose(env["z1"], (1, 0, 2)))
    for k in list(v):
        if k.startswith("col_"):
            v2["row_" + k[4:]] = v[k]
    env2 = executor.run(gr, v2, keep_all=True)
    np.testing.assert_allclose(np.transpose(env2["z1"], (1, 0, 2)), env["z2"], rtol=0, atol=1e-12)


def _attn_graph(N, h, dh, causal):
    B = Builder("a", "f64")
    B.input("q", (N, h, dh))
    B.input("k", (N, h, dh))
    B.input("vt", (h, dh, N))
    B.op("attn_scores", ["q", "k"], "s", scale=1.0 / math.sqrt(dh), causal=int(causal))
    B.op("softmax", ["s"], "p", dim=2)
    B.op("attn_pv", ["p", "vt"], "o")
    B.output("o")
    return B.build()


def test_closed_forms_attention():
    N, h, dh = 7, 2, 3
    rng = np.random.default_rng(0)
    vt = rng.standard_normal((h, dh, N))
    g = _attn_graph(N, h, dh, False)
    z = np.zeros((N, h, dh))
    o = executor.run(g, {"q": z, "k": z, "vt": vt})["o"]     # uniform softmax -> mean of v
    np.testing.assert_allclose(o, np.broadcast_to(vt.mean(axis=2)[None], (N, h, dh)), atol=1e-15)
    gc = _attn_graph(N, h, dh, True)
    q = rng.standard_normal((N, h, dh))
    k = rng.standard_normal((N, h, dh))
    o = executor.run(gc, {"q": q, "k": k, "vt": vt})["o"]
    np.testing.assert_allclose(o[0], vt[:, :, 0], atol=1e-15)  # causal row 0 attends to key 0 only
    g1 = _attn_graph(1, h, dh, False)                          # single key -> o = v
    o = executor.run(g1, {"q": q[:1], "k": k[:1], "vt": vt[:, :, :1]})["o"]
    np.testing.assert_allclose(o[0], vt[:, :, 0], atol=1e-15)


def test_closed_forms_elementwise():
    assert ops.evaluate("relu", {}, [np.array([-1.0, 2.0])]).tolist() == [0.0, 2.0]
    assert ops.evaluate("softmax", {"dim": 0}, [np.array([0.0, 0.0])]).tolist() == [0.5, 0.5]
    m = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert ops.evaluate("matmul", {}, [m, np.eye(2)]).tolist() == m.tolist()
    assert ops.evaluate("gelu", {}, [np.array([0.0])])[0] == 0.0
    beta = np.array([0.3, -0.2, 0.1])
    y = ops.evaluate("layernorm", {"naxes": 1, "eps": 1e-5},
                     [np.full((2, 3), 7.0), np.array([2.0, 3.0, 4.0]), beta])
    np.testing.assert_array_equal(y, np.broadcast_to(beta, (2, 3)))   # LN of a constant row -> beta
    # GELU(x) -> x for large x, -> 0 for very negative x; GELU(1) = Phi(1)
    assert abs(ops.evaluate("gelu", {}, [np.array([1.0])])[0] - 0.8413447460685429) < 1e-15


def test_exact_mode_equals_fast_mode():
    g = workloads.block("transformer", 32, 16, 2, 32, True, "f64")
    v = _values(g, 7)
    a = executor.run(g, v)["y"]
    with ops.exact_order():
        b = executor.run(g, v)["y"]
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)


def test_mirror_rounding_is_bf16():
    x = np.array([1.0 + 2 ** -9, 1.0 + 3 * 2 ** -9, -3.14159, 65504.0])
    r = executor.round_bf16(x)
    # ties to even at 1 + 2^-8 spacing
    assert r[0] == 1.0 and r[1] == 1.0 + 2 ** -7
    assert abs(r[2] - -3.140625) == 0


# ---------------------------------------------------------------- SPEC graph_ir examples
def test_spec_infer_shapes_and_flops():
    assert ops.shape("matmul", {}, [(2, 3), (3, 4)]) == (2, 4)
    assert ops.flops("matmul", {}, [(2, 3), (3, 4)], (2, 4)) == 48
    assert ops.shape("reshape", {"shape": [3, 4]}, [(2, 6)]) == (3, 4)
    with pytest.raises(ValueError, match="inner dimension mismatch"):
        ops.shape("matmul", {}, [(2, 3), (4, 5)])
    assert ops.flops("relu", {}, [(4, 4)], (4, 4)) == 16
    assert ops.flops("transpose", {"perm": [1, 0]}, [(3, 5)], (5, 3)) == 0
    assert graph.TensorMeta("t", "f32", (3, 4)).strides == (4, 1)


def test_spec_load_graph_examples():
    doc = "autochunk-graph 1\ntensor x f32 2,3\ntensor y f32 2,3\ninput x\nnode r relu x y\noutput y\n"
    g = graph.load_graph(doc)
    assert len([n for n in g.nodes if n.kind == "relu"]) == 1 and len(g.tensors) == 2
    with pytest.raises(GraphError, match="unknown tensor id"):
        graph.load_graph(doc.replace("node r relu x y", "node r relu t9 y"))
    cyc = ("autochunk-graph 1\ntensor x f32 2\ntensor a f32 2\ntensor b f32 2\ninput x\n"
           "node A add x,b a\nnode B relu a b\noutput b\n")
    with pytest.raises(GraphError, match="cycle|order"):
        graph.load_graph(cyc)
    bad = doc.replace("node r relu x y", "node r transpose x y perm=0,0")
    with pytest.raises(GraphError, match="bijection"):
        graph.load_graph(bad)


@pytest.mark.parametrize("name", ["tiny", "gpt", "vit", "af", "unet", "unet_h8"])
def test_document_round_trip(name):
    g = workloads.config(name)
    doc = graph.serialize(g)
    g2 = graph.load_graph(doc)
    assert graph.serialize(g2) == doc
    graph.infer_shapes(g2)
    assert graph.serialize(g2) == doc


def test_sampled_rows_equal_full_run():
    """oracle.blocks.transformer_rows (full-size parity helper) == executor.run rows."""
    from oracle import blocks
    for causal, kind in ((True, "transformer"), (False, "attn_only")):
        g = workloads.block(kind, 64, 32, 4, 64, causal, "f64")
        v = _values(g, 9)
        env = executor.run(g, v, keep_all=True)
        rows = blocks.sample_rows(64, 16, 8)
        got = blocks.transformer_rows(g, v, rows)
        out = "y" if kind == "transformer" else "x1"
        np.testing.assert_allclose(got[out], env[out][rows], rtol=0, atol=1e-12)
        np.testing.assert_allclose(got["o"], env["o"][rows], rtol=0, atol=1e-12)


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("attn_only", [False, True])
def test_fused_attention_block_matches_torch_functional(causal, attn_only):
    """NEXT f1: the attn_fused node (one kernel, no N x N tensor) is pinned by the
    same torch.nn.functional block (SDPA math path) as the unfused chain."""
    N, d, h, f = 48, 32, 4, 64
    g = workloads.block("attn_only_fa" if attn_only else "transformer_fa", N, d, h, f, causal, "f64")
    assert not any(n.kind in ("attn_scores", "softmax", "attn_pv") for n in g.nodes)
    v = _values(g)
    ours = executor.run(g, v)[g.outputs[0]]
    ref = _torch_transformer(v, N, d, h, causal, attn_only)
    np.testing.assert_allclose(ours, ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("causal", [False, True])
def test_fused_attention_chunked_is_exact(causal):
    """attn_fused chunked along query rows (offset-aware causal mask) or heads
    reproduces the unchunked node bitwise in exact-order fp64 (Eq. 5)."""
    from oracle import select
    g = workloads.block("transformer_fa", 40, 16, 2, 32, causal, "f64")
    v = _values(g, 3)
    with ops.exact_order():
        base = executor.run(g, v)
        for spec in ([("attn", "attn", 3, [0])], [("attn", "ffn2", 4, [0])], [("attn", "attn", 2, [1])]):
            plan = select.user_plan(g, spec)
            got = executor.run_chunked(g, v, plan.regions)
            np.testing.assert_array_equal(got[g.outputs[0]], base[g.outputs[0]])


@pytest.mark.parametrize("ending", [0, 1])
def test_tri_attention_pair_sampler_equals_full_run(ending):
    """The sampled-pair oracle for one triangle attention equals the full executor
    run at those pairs (fp64), so it can check full-size GPU runs."""
    from oracle import blocks
    from oracle.graph import Builder
    N, cz, H, c = 12, 8, 2, 4
    B = Builder("tri1", "f64")
    B.input("z", (N, N, cz))
    workloads._tri_weights(B, "t_", cz, H, c)
    workloads._tri_attention(B, "z", "t_", N, cz, H, c, ending, "zo")
    B.output("zo")
    g = B.build()
    v = _values(g, 2)
    full = executor.run(g, v)["zo"]
    pairs = [(0, 0), (3, 7), (11, 2), (5, 11)]
    got = blocks.tri_attention_pairs(g, v, "t_", pairs, bool(ending))
    np.testing.assert_allclose(got, np.stack([full[i, j] for i, j in pairs]), rtol=0, atol=1e-12)


# ----------------------------------------- Evoformer pair stack (NEXT f3), AF2 Alg. 6/11/12/15
def _torch_tri_mul(z, W, incoming):
    """AF2 Alg. 11 (outgoing) / Alg. 12 (incoming) via torch einsum, fp64."""
    T = {k: torch.from_numpy(np.asarray(a, dtype=np.float64)) for k, a in W.items()}
    z = torch.from_numpy(z)
    cz = z.shape[-1]
    zn = F.layer_norm(z, (cz,), T["ln_g"], T["ln_b"], eps=1e-5)
    a = torch.sigmoid(F.linear(zn, T["wag"], T["bag"])) * F.linear(zn, T["wa"], T["ba"])
    b = torch.sigmoid(F.linear(zn, T["wbg"], T["bbg"])) * F.linear(zn, T["wb"], T["bb"])
    g = torch.sigmoid(F.linear(zn, T["wg"], T["bg"]))
    x = torch.einsum("kic,kjc->ijc", a, b) if incoming else torch.einsum("ikc,jkc->ijc", a, b)
    xn = F.layer_norm(x, (x.shape[-1],), T["lnx_g"], T["lnx_b"], eps=1e-5)
    return (z + g * F.linear(xn, T["wo"], T["bo"])).numpy()


def _torch_transition(z, W):
    """AF2 Alg. 15 (pair transition, n = 4): z + Linear(relu(Linear(LN(z))))."""
    T = {k: torch.from_numpy(np.asarray(a, dtype=np.float64)) for k, a in W.items()}
    z = torch.from_numpy(z)
    zn = F.layer_norm(z, (z.shape[-1],), T["ln_g"], T["ln_b"], eps=1e-5)
    return (z + F.linear(torch.relu(F.linear(zn, T["w1"], T["b1"])), T["w2"], T["b2"])).numpy()


def test_evoformer_pair_stack_matches_af2_algorithms():
    """Every update of the pair stack (AF2 Alg. 6 lines 13-17) against its algorithm
    written with torch (einsum / nn.functional), on the previous update's output."""
    N, cz, H, c, cm = 10, 16, 2, 8, 12
    g = workloads.evoformer_pair(N, cz, H, c, "f64", cm=cm)
    v = _values(g, 4)
    env = executor.run(g, v, keep_all=True)
    pick = lambda pre: {k[len(pre):]: v[k] for k in v if k.startswith(pre)}  # noqa: E731
    z1 = _torch_tri_mul(v["z"], pick("mo_"), incoming=False)
    np.testing.assert_allclose(env["z1"], z1, rtol=0, atol=1e-12)
    z2 = _torch_tri_mul(env["z1"], pick("mi_"), incoming=True)
    np.testing.assert_allclose(env["z2"], z2, rtol=0, atol=1e-12)
    z3 = _torch_tri_attention(env["z2"], pick("row_"), ending=False)
    np.testing.assert_allclose(env["z3"], z3, rtol=0, atol=1e-12)
    z4 = _torch_tri_attention(env["z3"], pick("col_"), ending=True)
    np.testing.assert_allclose(env["z4"], z4, rtol=0, atol=1e-12)
    z5 = _torch_transition(env["z4"], pick("tr_"))
    np.testing.assert_allclose(env["z5"], z5, rtol=0, atol=1e-12)
