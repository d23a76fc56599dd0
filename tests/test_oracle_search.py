"""Pins for the oracle chunk search (SURVEY §8(c) c.3 "O4 search"): SPEC examples,
the node-pair count closed form, and a brute-force execution-equivalence oracle
that decides legality by running chunks (no propagate tables involved)."""
import itertools

import numpy as np
import pytest

from oracle import memory, ops, search, workloads
from oracle.graph import Builder
import synth


def _values(g, seed=0):
    return {t: s.value for t, s in synth.make_inputs(g.input_specs(), seed).items()}


def test_node_pairs_examples():
    assert search.get_node_pairs(5, 2, 2) == [(2, 2), (1, 2), (2, 3)]
    assert search.get_node_pairs(5, 2, 1) == [(2, 2)]
    for N in range(1, 9):
        for p in range(N):
            assert len(search.get_node_pairs(N, p, N)) == (p + 1) * (N - p)


def test_propagate_examples():
    assert ops.propagate("matmul", {}, [(2, 3), (3, 4)], (2, 4), 0) == [0, ops.NC]
    assert ops.propagate("softmax", {"dim": 1}, [(4, 8)], (4, 8), 1) == [ops.BREAK]
    assert ops.propagate("softmax", {"dim": 1}, [(4, 8)], (4, 8), 0) == [0]


def _single_relu():
    B = Builder("r", "f64")
    B.input("x", (4, 6))
    B.op("relu", ["x"], "y")
    B.output("y")
    return B.build()


def test_filter_examples():
    g = _single_relu()
    assert search.two_stage_filter(g, 1, 1, ["y"], (0,), g.producer_index())
    B = Builder("rs", "f64")
    B.input("x", (2, 6))
    B.op("reshape", ["x"], "y", shape=[3, 4])
    B.output("y")
    g = B.build()
    for d in (0, 1):
        assert not search.two_stage_filter(g, 1, 1, ["y"], (d,), g.producer_index())


def test_attention_finds_query_dim_not_softmax_dim():
    """candidate on the query-sequence dim exists, none on the softmax dim."""
    g = workloads.corpus("attention", 16, 8)
    names = [n.id for n in g.nodes]
    s, e = names.index("n_s"), names.index("n_o")
    assert search.candidate_for(g, s, e, (0,)) is not None
    sm = names.index("n_pr")
    assert search.candidate_for(g, sm, sm, (1,)) is None


# ----------------------------------------------------------- brute force (AC-5)
def _bf_legal(g, s, e, outs, assign, vals, full):
    """Is there a slicing of the region inputs (one dim per input, each consumer
    edge taking the slice or the whole tensor) whose two chunks concatenate to the
    unchunked outputs exactly (fp64, exact reduction order)?

    Position-dependent kinds (the causal mask of attn_scores / attn_fused) need the
    global index of a slice: for each such node every hypothesis "output dim d of
    this chunk starts at the chunk's offset" (or none) is tried, so legality is
    decided by execution alone, never by the propagate tables under test."""
    E = g.tensors[outs[0]].shape[assign[0]]
    if any(g.tensors[y].shape[d] != E for y, d in zip(outs, assign)) or E < 2:
        return False
    pos = [i for i in range(s, e + 1) if g.nodes[i].attrs.get("causal", 0)]
    ctx_opts = [[None] + [d for d, x in enumerate(g.tensors[g.nodes[i].output].shape) if x == E] for i in pos]
    for csel in itertools.product(*ctx_opts):
        if _bf_legal_ctx(g, s, e, outs, assign, vals, full, E, dict(zip(pos, csel))):
            return True
    return False


def _bf_legal_ctx(g, s, e, outs, assign, vals, full, E, ctxdim):
    produced = {g.nodes[i].output for i in range(s, e + 1)}
    ins = [t for t in memory.region_io(g, s, e)[0] if t not in g.weights]
    dim_opts = [[None] + [d for d, x in enumerate(g.tensors[t].shape) if x == E] for t in ins]
    L = -(-E // 2)
    for dsel in itertools.product(*dim_opts):
        dmap = dict(zip(ins, dsel))
        edges = [(i, j) for i in range(s, e + 1) for j, t in enumerate(g.nodes[i].inputs)
                 if dmap.get(t) is not None]
        for esel in itertools.product((True, False), repeat=len(edges)):
            take = dict(zip(edges, esel))
            chunks = []
            ok = True
            for c in range(2):
                off, ln = c * L, min(L, E - c * L)
                loc = {}
                try:
                    for i in range(s, e + 1):
                        nd = g.nodes[i]
                        vv = []
                        for j, t in enumerate(nd.inputs):
                            if t in produced:
                                vv.append(loc[t])
                            elif take.get((i, j)):
                                idx = [slice(None)] * vals[t].ndim
                                idx[dmap[t]] = slice(off, off + ln)
                                vv.append(vals[t][tuple(idx)])
                            else:
                                vv.append(vals[t])
                        cd = ctxdim.get(i)
                        ctx = None if cd is None else {"dim": cd, "offset": off}
                        loc[nd.output] = ops.evaluate(nd.kind, nd.attrs, vv, ctx)
                except (ValueError, IndexError):
                    ok = False
                    break
                chunks.append(loc)
            if not ok:
                continue
            good = True
            for y, d in zip(outs, assign):
                try:
                    cat = np.concatenate([chunks[0][y], chunks[1][y]], axis=d)
                except ValueError:
                    good = False
                    break
                if cat.shape != full[y].shape or not np.array_equal(cat, full[y]):
                    good = False
                    break
            if good:
                return True
    return False


CORPUS = [("mlp", 8, 4), ("attention", 8, 4), ("transformer2", 6, 4), ("alphafold_like_2d", 4, 3)]

# every fused kind: linear with bias / act / residual / trans (vᵀ) and
# swap (ending-node bias, vᵀ), attn_scores causal and not, attn_pv, attn_fused (f1),
# tri_scores / tri_pv for the starting and the ending node; extents chosen distinct
# where the block allows (N=5 gives a ragged 3+2 split)
FUSED = {
    "gpt": lambda: workloads.block("transformer", 5, 4, 2, 8, True, "f64"),
    "vit": lambda: workloads.block("transformer", 5, 4, 2, 8, False, "f64"),
    "fa_causal": lambda: workloads.block("transformer_fa", 5, 4, 2, 8, True, "f64"),
    "fa": lambda: workloads.block("attn_only_fa", 5, 4, 2, 0, False, "f64"),
    "af": lambda: workloads.tri_attn_pair(4, 3, 2, 5, "f64"),
    "evo_mul": lambda: _evo_mul_graph(),
}


def _evo_mul_graph():
    """Triangle multiplication outgoing + incoming + pair transition (the f3 kinds:
    gated channel-major linear, tri_mul, ln_cfirst, relu FFN) on a 4 x 4 pair rep."""
    B = Builder("evo_mul", "f64")
    B.input("z", (4, 4, 3))
    workloads._tri_mul(B, "z", "mo_", 3, 5, 0, "z1")
    workloads._tri_mul(B, "z1", "mi_", 3, 5, 1, "z2")
    workloads._transition(B, "z2", "tr_", 3, 2, "z3")
    B.output("z3")
    return B.build()


@pytest.mark.parametrize("name,seq,d", CORPUS + [(k, 0, 0) for k in FUSED])
def test_search_complete_and_sound_vs_brute_force(name, seq, d):
    g = FUSED[name]() if name in FUSED else workloads.corpus(name, seq, d, "f64")
    vals = _values(g, 11)
    from oracle import executor
    with ops.exact_order():
        full = executor.run(g, vals, keep_all=True)
        prod = g.producer_index()
        sources = [i for i, n in enumerate(g.nodes) if n.kind in ("input", "weight")]
        W = 4
        npass = nfilt = nlegal = 0
        for p in range(len(g.nodes)):
            if p in sources:
                continue
            for s, e in search.get_node_pairs(len(g.nodes), p, W, sources):
                if s != p and e != p:
                    continue   # each interval once (as the left- or right-most pair of some p)
                ins, outs = memory.region_io(g, s, e)
                if not outs or len(outs) > 2:
                    continue
                for assign in itertools.product(*[range(len(g.tensors[y].shape)) for y in outs]):
                    got = search.bfs_region(g, s, e, ins, outs, assign, prod) is not None
                    want = _bf_legal(g, s, e, outs, assign, full, full)
                    assert got == want, (name, s, e, assign, got, want)
                    f = search.two_stage_filter(g, s, e, outs, assign, prod)
                    nfilt += f
                    npass += 1
                    if got:
                        assert f                              # no false negatives (AC-8)
                        # the flow map the search emits (propagate rows, X^c dims, the
                        # causal offsets it implies) executed chunk by chunk must give
                        # the unchunked graph outputs bit for bit (Eq. 5)
                        for hz in (False, True):
                            r = search.candidate_for(g, s, e, assign, hoist=hz)
                            assert r is not None
                            ch = executor.run_chunked(g, vals, [r.with_n(2)])
                            for o in g.outputs:
                                assert np.array_equal(ch[o], full[o]), (name, s, e, assign, hz, o)
                        nlegal += 1
        assert npass > 0 and nfilt <= npass
        assert nlegal > 0


def test_rule4_holds_and_window_monotone():
    g = workloads.corpus("transformer2", 8, 4, "f64")
    p = memory.profile(g)
    prev = None
    for k in (2, 4, 8, 16, 32):
        cands = search.search(g, p.peak_step, [], p.peak_bytes, window=k)
        sigs = {c.signature() for c in cands}
        for c in cands:
            assert len(set(c.dims)) == len(c.dims)                                     # Rule 4
            assert set(t for t, _ in c.xc) | set(c.xnc) == set(memory.region_io(g, c.start, c.end)[0])
        if prev is not None:
            assert prev <= sigs
        prev = sigs


def test_hoisting_moves_kv_projections_out():
    """Graph optimisation: in the region [q-proj .. pv] the K/V projections
    are off the flow and get hoisted; the region keeps q-proj, scores, softmax, pv."""
    g = workloads.block("transformer", 64, 16, 2, 32, False, "f32")
    names = [n.id for n in g.nodes]
    r = search.candidate_for(g, names.index("proj_q"), names.index("pv"), (0,))
    assert [names[i] for i in r.hoisted] == ["proj_k", "proj_v"]
    assert (names[r.start], names[r.end]) == ("proj_q", "pv")
    r2 = search.candidate_for(g, names.index("proj_k"), names.index("pv"), (0,))
    assert (names[r2.start], names[r2.end]) == ("scores", "pv") and r2.hoisted == []
    r3 = search.candidate_for(g, names.index("proj_q"), names.index("pv"), (0,), hoist=False)
    assert r3.hoisted == [] and (names[r3.start], names[r3.end]) == ("proj_q", "pv")
