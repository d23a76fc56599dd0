"""Pins for the oracle estimator (SURVEY §8(c) c.3 "O3 estimator"): SPEC's worked
examples, the Eq. 2 closed form, and brute force — tracked_run measures live
bytes from the buffers that actually exist and must equal the estimate exactly."""
import numpy as np
import pytest

from oracle import executor, memory, ops, search, workloads
from oracle.graph import Builder
import synth


def _values(g, seed=0):
    return {t: s.value for t, s in synth.make_inputs(g.input_specs(), seed).items()}


def test_spec_profile_examples():
    B = Builder("c", "f32")
    B.input("x", (4, 4))
    B.op("relu", ["x"], "y")
    B.output("y")
    p = memory.profile(B.build())
    assert p.per_step == [64, 128] and p.peak_bytes == 128 and p.peak_node == "n_y"
    lv = memory.liveness(B.build())
    assert lv["x"] == (0, 1) and lv["y"] == (1, 1)

    # 100 B -> 1000 B -> 100 B chain
    g = Builder("c", "f32")
    g.input("x", (1, 25))
    g.weight("w", (25, 250), "matrix", 25)
    g.weight("w2", (250, 25), "matrix", 250)
    g.op("matmul", ["x", "w"], "m")
    g.op("matmul", ["m", "w2"], "y")
    g.output("y")
    p = memory.profile(g.build())
    assert p.peak_bytes == 1100 and p.per_step[p.peak_step] == 1100
    assert p.peak_node == "n_m"                                                         # first on ties

    e = Builder("e", "f32")                   # empty graph: inputs = outputs
    e.input("x", (3, 5))
    e.output("x")
    assert memory.profile(e.build()).peak_bytes == 60


def test_spec_liveness_diamond_and_unused_weight():
    B = Builder("d", "f32")
    B.input("x", (2, 2))
    B.weight("w", (2, 2), "matrix", 2)
    B.op("relu", ["x"], "a")
    B.op("exp", ["x"], "b")
    B.op("add", ["a", "b"], "y")
    B.output("y")
    g = B.build()
    lv = memory.liveness(g)
    assert lv["x"][1] == max(2, 3)
    assert lv["w"] == (0, 0)


def test_eq2_closed_form_single_region():
    """mem(X)=100 B, mem(Y)=100 B, interior mem(A)=1000 B, n=10 -> 300 B."""
    h = Builder("eq2", "bf16")
    h.input("x", (10, 5))                     # 100 B
    h.weight("w", (5, 50), "matrix", 5)
    h.weight("w2", (50, 5), "matrix", 50)
    h.op("matmul", ["x", "w"], "a")           # 1000 B interior
    h.op("matmul", ["a", "w2"], "y")          # 100 B output
    h.output("y")
    g = h.build()
    r = search.candidate_for(g, 3, 4, (0,))
    assert r is not None and r.xc == [("x", 0)] and r.yc == [("y", 0)]
    est = memory.estimate_with_plan(g, [r.with_n(10)])
    assert est.per_step[3] == 300 and est.per_step[4] == 300 and est.peak_bytes == 300
    # n = extent -> one slice row each: same here since E = 10
    assert memory.estimate_with_plan(g, [r.with_n(5)]).peak_bytes == 100 + 100 + 200
    # empty plan -> profile; n = 1 -> the step is dropped (reading R7)
    assert memory.estimate_with_plan(g, []).per_step == memory.profile(g).per_step
    assert memory.estimate_with_plan(g, [r.with_n(1)]).per_step == memory.profile(g).per_step


def test_contiguity_cost_examples():
    assert memory.contiguity_cost((8, 16), 4, 0, 4) == 0
    assert memory.contiguity_cost((8, 16), 4, 1, 4) == 128
    assert memory.contiguity_cost((7,), 4, 0, 3) == 0
    assert memory.contiguity_cost((1, 6, 5), 2, 1, 4) == 0


GRAPHS = [
    lambda: workloads.corpus("mlp", 16, 8),
    lambda: workloads.corpus("attention", 16, 8),
    lambda: workloads.corpus("transformer2", 16, 8),
    lambda: workloads.corpus("alphafold_like_2d", 6, 4),
    lambda: workloads.block("transformer", 32, 16, 2, 32, True, "bf16"),
    lambda: workloads.block("attn_only", 24, 16, 4, 0, False, "f32"),
    lambda: workloads.tri_attn_pair(6, 8, 2, 4, "bf16"),
]


@pytest.mark.parametrize("mk", GRAPHS)
def test_profile_equals_tracked_run(mk):
    g = mk()
    _, per = executor.tracked_run(g, _values(g))
    assert per == memory.profile(g).per_step                                            # AC-3


@pytest.mark.parametrize("mk", GRAPHS)
@pytest.mark.parametrize("contig", [False, True])
def test_estimate_equals_tracked_chunked_run(mk, contig):
    """Every legal single-region candidate around every node, n in {2, 3, E}:
    predicted per-step bytes == measured per-step bytes, exactly."""
    g = mk()
    v = _values(g, 1)
    prod = g.producer_index()
    sources = [i for i, n in enumerate(g.nodes) if n.kind in ("input", "weight")]
    checked = 0
    for p in range(len(g.nodes)):
        if p in sources:
            continue
        for s, e in search.get_node_pairs(len(g.nodes), p, 4, sources):
            ins, outs = memory.region_io(g, s, e)
            if len(outs) != 1:
                continue
            for d in range(len(g.tensors[outs[0]].shape)):
                for hz in (True, False):   # graph optimisation on / off (Table 1)
                    r = search.candidate_for(g, s, e, (d,), prod=prod, hoist=hz)
                    if r is None:
                        continue
                    for n in sorted({2, 3, r.extent}):
                        if n > r.extent:
                            continue
                        rr = r.with_n(n)
                        _, per = executor.tracked_run(g, v, [rr], contiguity=contig)
                        est = memory.estimate_with_plan(g, [rr], contiguity=contig)
                        assert per == est.per_step, (s, e, d, n, hz)
                        checked += 1
        if checked > 60:
            break
    assert checked > 0


def test_monotone_in_n():
    g = workloads.block("transformer", 64, 16, 2, 32, False, "f32")
    names = [n.id for n in g.nodes]
    r = search.candidate_for(g, names.index("scores"), names.index("pv"), (0,))
    peaks = [memory.estimate_with_plan(g, [r.with_n(n)]).peak_bytes for n in (2, 4, 8, 16, 32, 64)]
    assert all(a >= b for a, b in zip(peaks, peaks[1:]))


def test_gpt_closed_form_peaks():
    """SURVEY App. A, plain Eq. 1 / Eq. 2 (fp32 GPT: no fused chain): unchunked softmax
    step = 2 N d b + 2 h N^2 b; minimal attention region at n chunks =
    5 N d b + 2 h N ceil(N/n) b."""
    N, d, h, b = 16384, 1024, 16, 4
    g = workloads.config("gpt", dtype="f32")
    assert memory.f2_chains(g) == []
    p = memory.profile(g)
    assert p.peak_bytes == 2 * N * d * b + 2 * h * N * N * b and p.peak_node == "softmax"
    names = [n.id for n in g.nodes]
    r = search.candidate_for(g, names.index("scores"), names.index("pv"), (0,))
    for n in (4, 8, 16):
        est = memory.estimate_with_plan(g, [r.with_n(n)])
        assert est.peak_bytes == 5 * N * d * b + 2 * h * N * (-(-N // n)) * b


def test_gpt_f2_closed_form_peaks():
    """R25 on the bf16 GPT block: the chain is fused, S is its e-tiles (N, N multiples
    of 128 / 64: exactly h N^2 bf16), P its slab statistics h N (N/64) 8 B written by
    the scores step.  Unchunked peak at the scores step = x + q + k + v^T + S + P =
    4 N d 2 + 2 h N^2 + 8 h N N/64; the attention region at n chunks holds x, q, k,
    v^T and o whole plus one chunk of S and P: 5 N d 2 + (2 h N + 8 h N/64) ceil(N/n)."""
    N, d, h = 16384, 1024, 16
    g = workloads.config("gpt")
    names = [n.id for n in g.nodes]
    assert memory.f2_chains(g) == [(names.index("scores"), names.index("softmax"), names.index("pv"))]
    p = memory.profile(g)
    assert p.peak_bytes == 4 * N * d * 2 + 2 * h * N * N + 8 * h * N * (N // 64) and p.peak_node == "scores"
    r = search.candidate_for(g, names.index("scores"), names.index("pv"), (0,))
    for n in (4, 8, 16):
        est = memory.estimate_with_plan(g, [r.with_n(n)])
        L = -(-N // n)
        assert est.peak_bytes == 5 * N * d * 2 + (2 * h * N + 8 * h * (N // 64)) * L
    # a chunk of 32 rows pads its e-tiles to 128 rows: charged so
    est = memory.estimate_with_plan(g, [r.with_n(N // 32)])
    assert est.peak_bytes == 5 * N * d * 2 + 2 * h * 128 * N + 8 * h * 32 * (N // 64)
