"""Pins for the oracle selection (SURVEY §8(c) c.3 "O4 selection", "Expected plans")
and the chunked == unchunked equivalence of Eq. 5."""
import numpy as np
import pytest

from oracle import executor, memory, ops, plan, select, workloads
import synth

GiB = 2 ** 30


def _values(g, seed=0):
    return {t: s.value for t, s in synth.make_inputs(g.input_specs(), seed).items()}


def test_cost_arithmetic_examples():
    p = select.CostParams(alpha=1.0, beta=1e-9)
    assert select.macro_cost(5, 2_000_000, p) == pytest.approx(5.002, abs=1e-12)
    q = select.CostParams(gamma=-1e-5, lam=0.01)
    assert select.micro_cost(1e5, 16, q) == pytest.approx(-0.84, abs=1e-12)
    z = select.CostParams(alpha=0.0, beta=0.0, gamma=0.0, lam=0.0)
    assert select.macro_cost(7, 10 ** 9, z) == 0.0 and select.micro_cost(3.0, 9, z) == 0.0


def test_budget_edge_cases():
    g = workloads.corpus("transformer2", 16, 8, "f64")
    base = memory.profile(g).peak_bytes
    p = select.select(g, base + 1)
    assert p.feasible and p.regions == [] and p.cost == 0.0
    io = sum(g.tensors[t].bytes for t in g.inputs + g.outputs)
    p = select.select(g, io)
    assert not p.feasible


@pytest.mark.parametrize("name,seq,d,frac", [("mlp", 32, 8, 0.5), ("attention", 32, 8, 0.4),
                                             ("transformer2", 24, 8, 0.5),
                                             ("alphafold_like_2d", 8, 4, 0.6),
                                             ("attention", 32, 8, 0.25)])
def test_dp_beam_equals_exhaustive(name, seq, d, frac):
    """AC-6: beam >= 16 gives the exhaustive minimum-cost feasible plan."""
    g = workloads.corpus(name, seq, d, "f64")
    budget = int(frac * memory.profile(g).peak_bytes)
    prm = select.CostParams(beam=64)
    p = select.select(g, budget, prm)
    ex = select.exhaustive(g, budget, prm, max_passes=3)
    if ex is None:
        assert not p.feasible
        return
    assert p.feasible and p.cost == ex[0]
    assert sorted((r.start, r.end, r.n) for r in p.regions) == sorted((r.start, r.end, r.n) for r in ex[1])


@pytest.mark.parametrize("name,seq,d", [("mlp", 32, 8), ("attention", 32, 8), ("transformer2", 24, 8),
                                        ("alphafold_like_2d", 8, 4)])
@pytest.mark.parametrize("frac", [0.5, 0.4, 0.2])
def test_chunked_equals_unchunked_bitwise(name, seq, d, frac):
    """AC-1: every produced plan, >= 20 seeds, run_chunked == run bitwise."""
    g = workloads.corpus(name, seq, d, "f64")
    p = select.select(g, int(frac * memory.profile(g).peak_bytes))
    with ops.exact_order():
        for seed in range(20):
            v = _values(g, seed)
            a = executor.run(g, v)
            b = executor.run_chunked(g, v, p.regions)
            for o in g.outputs:
                assert np.array_equal(a[o], b[o])


def test_feasible_plans_meet_budget_and_measure():
    for name, seq, d in [("attention", 256, 16), ("transformer2", 256, 16)]:
        g = workloads.corpus(name, seq, d, "f32")
        base = memory.profile(g).peak_bytes
        p = select.select(g, int(0.2 * base))                                          # AC-2
        assert p.feasible and p.peak < 0.2 * base
        _, per = executor.tracked_run(g, _values(g), p.regions)
        assert max(per) == p.peak


def test_determinism_and_scale_invariance():
    g = workloads.corpus("transformer2", 24, 8, "f64")
    b = int(0.3 * memory.profile(g).peak_bytes)
    t1 = plan.serialize(select.select(g, b), g)
    assert t1 == plan.serialize(select.select(g, b), g)
    s = select.CostParams(alpha=2.0, beta=2e-9, gamma=-2e-5, lam=0.02)
    p2 = select.select(g, b, s)
    p1 = select.select(g, b)
    assert [(r.start, r.end, r.n, tuple(r.dims.items())) for r in p1.regions] == \
           [(r.start, r.end, r.n, tuple(r.dims.items())) for r in p2.regions]          # S:364 argmin


# ------------------------------------------------------------- expected plans (§8(a))
def _plan(name):
    g = workloads.config(name)
    base = memory.profile(g)
    return g, base, select.select(g, int(0.2 * base.peak_bytes))


def test_expected_plan_gpt():
    """Under R25 (fused chain: e-tile S, statistics P) the unchunked peak is the scores
    step, 4 N d 2 + 2 h N^2 + 8 h N N/64; 20 % of it leaves the attention region at
    n = 8 (n = 4 would hold 2.2 GB)."""
    g, base, p = _plan("gpt")
    names = [n.id for n in g.nodes]
    assert base.peak_bytes == 9261023232                        # 8.625 GiB at the scores step
    assert p.feasible and len(p.regions) == 1
    r = p.regions[0]
    assert (names[r.start], names[r.end], r.n, r.chunk_len) == ("scores", "pv", 8, 2048)
    assert r.yc == [("o", 0)] and r.xc == [("q", 0)] and r.xnc == ["k", "vt"]
    assert p.peak == 1308622848                                 # 1.219 GiB = 14.1 %


def test_expected_plan_vit_unet():
    g, base, p = _plan("vit")
    assert base.peak_bytes == 146565758976 and p.regions[0].n == 8   # 136.5 GiB: fits one B200
    assert p.peak == 18924699648
    for nm in ("unet", "unet_h8"):   # (h8: head dim 80 > 64, chain not fused, P materialised)
        g, base, p = _plan(nm)
        assert p.feasible and p.regions[0].n == 8 and p.regions[0].yc == [("o", 0)]
    assert memory.f2_chains(workloads.config("unet_h8")) == []


def test_expected_plan_af_two_regions():
    """AlphaFold under R25: query-dim chunks of fewer than 128 rows would pad their
    e-tiles to 128 rows, so the planner cuts the batch dim of each attention (i for
    the starting node, j for the ending node), 32 chunks each."""
    g, base, p = _plan("af")
    names = [n.id for n in g.nodes]
    assert base.peak_bytes == 10477371392
    assert p.feasible and [(names[r.start], names[r.end], r.n) for r in p.regions] == \
        [("row_scores", "row_pv", 32), ("col_scores", "col_pv", 32)]
    assert p.regions[0].yc == [("row_o", 0)] and p.regions[1].yc == [("col_o", 1)]
    assert p.peak == 1904214016


def test_expected_plan_tiny_infeasible():
    g, base, p = _plan("tiny")
    assert not p.feasible and p.regions                         # AC_ERR_BUDGET + best effort
    assert 0.25 < p.peak / base.peak_bytes < 0.3                # floor ~28 %


def test_normalized_features_closed_forms():
    """R27 normalised features (AC_FLAG_NORMALIZE, SURVEY c.2 #10): a region holding
    every compute node of the graph (nothing hoisted) has N_node / S_g = 1,
    N_flop / F_g = 1 and N_density / (F_g / S_g) = 1 exactly, and a row-chunked
    [N, *] flow tensor has N_stride / numel = 1 / N."""
    g = workloads.corpus("mlp", 32, 8, "f32")
    spec = [("n_h1", "n_y", 4, (0,), False)]
    def cost(**kw):
        p = select.CostParams(normalize=True, **kw)
        (r,) = select.user_plan(g, spec, p).regions
        assert r.hoisted == [] or list(r.hoisted) == []
        return r.cost
    assert cost(alpha=1.0, beta=0.0, gamma=0.0, lam=0.0).macro == 1.0
    assert cost(alpha=0.0, beta=1.0, gamma=0.0, lam=0.0).macro == 1.0
    assert cost(alpha=0.0, beta=0.0, gamma=-1.0, lam=0.0).micro == -1.0
    assert cost(alpha=0.0, beta=0.0, gamma=0.0, lam=1.0).micro == 1.0 / 32
    # the raw features are the same numbers either way
    raw = select.user_plan(g, spec).regions[0].cost
    nrm = cost(alpha=1.0, beta=1.0, gamma=-1.0, lam=1.0)
    assert (raw.n_node, raw.n_flop, raw.density, raw.stride) == (nrm.n_node, nrm.n_flop, nrm.density, nrm.stride)
    # Table-1 toggles still zero their terms
    p = select.CostParams(normalize=True, alpha=1.0, beta=1.0, gamma=-1.0, lam=1.0, use_node=False,
                          use_flop=False, use_density=False, use_stride=False)
    assert select.user_plan(g, spec, p).regions[0].cost.total == 0.0


def test_normalized_features_pick_the_ffn_region_for_fused_attention():
    """GPT with fused attention (NEXT f1) at 90 % of its unchunked peak: the raw SPEC
    features choose the attention-including region (the density term, ~1e6, swamps
    the others); normalised features with unit weights choose an FFN-only region."""
    g = workloads.config("gpt_fa")
    budget = int(0.9 * memory.profile(g).peak_bytes)
    raw = select.select(g, budget)
    assert [g.nodes[r.start].id for r in raw.regions] == ["attn"]
    nrm = select.select(g, budget, select.CostParams(normalize=True, alpha=1.0, beta=1.0, gamma=-1.0, lam=1.0))
    assert nrm.feasible and all(g.nodes[r.start].id in ("ln2", "ffn1") for r in nrm.regions)
