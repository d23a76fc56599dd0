"""The C-ABI host library (ac_graph_*, ac_estimate_memory, ac_plan, ac_plan_parse)
against the oracle: byte-identical documents, per-step estimates and plan texts
(SURVEY §7 step 2).  CPU only — no compute calls."""
import ctypes
import random
import re

import pytest

from oracle import graph as og
from oracle import memory, plan as oplan, select, workloads
from oracle.graph import Builder

api = pytest.importorskip("paper_2401_10652_b200.api")
from paper_2401_10652_b200 import _lib  # noqa: E402


def test_library_exports_every_declared_symbol(root):
    import os
    L = _lib.lib()
    declared = set()
    for h in ("ac.h", "ac_kernels.h"):
        txt = open(os.path.join(root, "include", h)).read()
        declared |= set(re.findall(r"\b(ac_[a-z0-9_]+)\s*\(", txt))
    declared -= {"ac_plan_workspace_bytes(plan"}  # (none: regex only matches identifiers)
    for name in sorted(declared):
        assert hasattr(L, name), name
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert declared <= bound, declared - bound


CONFIGS = ["tiny", "gpt", "vit", "af", "af_attn", "unet", "unet_h8", "gpt_fa"]


def _c_graph(name):
    c = workloads.CONFIGS[name]
    return api.graph_block(c["kind"], c["N"], c["d"], c["h"], c["f"], c["causal"], c["dtype"], name=name)


@pytest.mark.parametrize("name", CONFIGS)
def test_block_documents_identical(name):
    assert _c_graph(name).serialize() == og.serialize(workloads.config(name))


@pytest.mark.parametrize("name", CONFIGS)
def test_parse_round_trip_and_profile(name):
    doc = og.serialize(workloads.config(name))
    g = api.graph_parse(doc)
    assert g.serialize() == doc
    prof, per = api.estimate_memory(g)
    ref = memory.profile(workloads.config(name))
    assert per == ref.per_step and prof.peak_bytes == ref.peak_bytes and prof.peak_step == ref.peak_step
    assert (prof.x_bytes, prof.y_bytes, prof.a_bytes) == (ref.x_bytes, ref.y_bytes, ref.a_bytes)


@pytest.mark.parametrize("name", CONFIGS)
@pytest.mark.parametrize("frac", [0.5, 0.2])
def test_plans_bit_exact(name, frac):
    og_g = workloads.config(name)
    budget = int(frac * memory.profile(og_g).peak_bytes)
    ref = select.select(og_g, budget)
    g = _c_graph(name)
    p = api.ac_plan(g, budget)
    assert p.serialize() == oplan.serialize(ref, og_g)
    assert p.feasible == ref.feasible
    prof, per = api.estimate_memory(g, p)
    assert per == memory.estimate_with_plan(og_g, ref.regions).per_step


def _corpus():
    for name, seq, d in [("mlp", 32, 8), ("attention", 32, 8), ("transformer2", 24, 8),
                         ("alphafold_like_2d", 8, 4)]:
        yield name, workloads.corpus(name, seq, d, "f32")


@pytest.mark.parametrize("frac", [0.6, 0.4, 0.25])
def test_corpus_plans_bit_exact(frac):
    for name, g in _corpus():
        doc = og.serialize(g)
        cg = api.graph_parse(doc)
        budget = int(frac * memory.profile(g).peak_bytes)
        for kw, prm in [({}, select.CostParams()), ({"beam": 16}, select.CostParams(beam=16)),
                        ({"flags": _lib.AC_FLAG_NO_HOIST}, select.CostParams(hoist=False)),
                        ({"flags": _lib.AC_FLAG_CONTIGUITY}, select.CostParams(contiguity=True)),
                        ({"flags": _lib.AC_FLAG_NORMALIZE, "alpha": 1.0, "beta": 1.0, "gamma": -1.0, "lam": 1.0},
                         select.CostParams(normalize=True, alpha=1.0, beta=1.0, gamma=-1.0, lam=1.0))]:
            ref = select.select(g, budget, prm)
            got = api.ac_plan(cg, budget, api.cost_params(**kw))
            assert got.serialize() == oplan.serialize(ref, g), (name, kw)


def _random_graph(rng: random.Random, i: int):
    """Fuzzed tiny graphs over the primitive and fused kinds."""
    B = Builder(f"fz{i}", rng.choice(["f32", "bf16", "f64"]))
    N, d = rng.choice([4, 6, 8]), rng.choice([2, 4])
    B.input("x", (N, d))
    B.weight("w", (d, d), "matrix", d)
    B.weight("w2", (d, 2 * d), "matrix", d)
    B.weight("g", (d,), "ln_gamma", d)
    B.weight("b", (d,), "ln_beta", d)
    B.weight("lw", (d, d), "matrix", d)
    live = ["x"]
    shapes = {"x": (N, d)}
    for k in range(rng.randint(3, 9)):
        src = rng.choice(live)
        out = f"t{k}"
        kind = rng.choice(["relu", "gelu", "exp", "add", "mul", "softmax0", "softmax1", "ln", "matmul",
                           "transpose", "linear", "reduce"])
        s = shapes[src]
        try:
            if kind in ("relu", "gelu", "exp"):
                B.op(kind, [src], out)
            elif kind in ("add", "mul"):
                other = rng.choice([t for t in live if shapes[t] == s] or [src])
                B.op(kind, [src, other], out)
            elif kind.startswith("softmax"):
                B.op("softmax", [src], out, dim=int(kind[-1]) % len(s))
            elif kind == "ln" and s[-1] == d and len(s) == 2:
                B.op("layernorm", [src, "g", "b"], out, naxes=1, eps=1e-5)
            elif kind == "matmul" and s[-1] == d:
                B.op("matmul", [src, rng.choice(["w", "w2"])], out)
            elif kind == "transpose" and len(s) == 2:
                B.op("transpose", [src], out, perm=[1, 0])
            elif kind == "linear" and s[-1] == d and len(s) == 2:
                B.op("linear", [src, "lw"], out, kin=1, out=[d], act=rng.choice(["none", "gelu"]),
                     trans=rng.choice([0, 1]), swap=0, bias=0, res=0)
            elif kind == "reduce" and len(s) == 2:
                B.op("reduce_sum", [src], out, dim=rng.choice([0, 1]))
            else:
                continue
        except ValueError:
            continue
        live.append(out)
        shapes[out] = B.g.tensors[out].shape
    B.output(live[-1])
    if len(live) > 3 and rng.random() < 0.5:
        B.output(live[-2])
    return B.build()


def test_fuzzed_graphs_plans_and_estimates_bit_exact():
    rng = random.Random(1234)
    n_checked = 0
    for i in range(60):
        g = _random_graph(rng, i)
        doc = og.serialize(g)
        cg = api.graph_parse(doc)
        assert cg.serialize() == doc
        base = memory.profile(g)
        _, per = api.estimate_memory(cg)
        assert per == base.per_step
        for frac in (0.7, 0.4):
            budget = int(frac * base.peak_bytes)
            ref = select.select(g, budget, select.CostParams(window=8))
            got = api.ac_plan(cg, budget, api.cost_params(window=8))
            assert got.serialize() == oplan.serialize(ref, g), doc
            n_checked += len(ref.regions)
    assert n_checked > 10


def test_user_plan_parse_matches_oracle():
    g = workloads.config("gpt")
    cg = _c_graph("gpt")
    txt = "autochunk-plan 1\nregion s=scores e=pv n=8 dims=0\n"
    p = api.plan_parse(cg, txt)
    ref = select.user_plan(g, [("scores", "pv", 8, (0,))])
    assert p.serialize() == oplan.serialize(ref, g)
    whole = "autochunk-plan 1\nregion s=proj_q e=ffn2 n=8 dims=0\n"
    p = api.plan_parse(cg, whole)
    ref = select.user_plan(g, [("proj_q", "ffn2", 8, (0,))])
    assert p.serialize() == oplan.serialize(ref, g)
    # opt=0: graph optimisation off for the region (K / V projections recomputed per chunk)
    for txt in ("autochunk-plan 1\nregion s=proj_q e=pv n=8 dims=0 opt=0\n",
                "autochunk-plan 1\nregion s=proj_q e=ffn2 n=4 dims=0 opt=0\n"):
        p = api.plan_parse(cg, txt)
        ref = select.user_plan(g, oplan.parse_user_regions(txt))
        assert p.serialize() == oplan.serialize(ref, g)
        assert "hoist=- " in p.serialize()
    # the canonical text of an ac_plan result parses back to the same plan
    full = api.ac_plan(cg, int(0.2 * memory.profile(g).peak_bytes))
    again = api.plan_parse(cg, full.serialize())
    assert re.sub(r"budget \d+\n", "", again.serialize().replace("budget 0\n", "")).split("peak")[1] == \
        re.sub(r"budget \d+\n", "", full.serialize()).split("peak")[1]


def test_error_codes():
    with pytest.raises(_lib.ACError) as e:
        api.graph_parse("autochunk-graph 1\ntensor x f32 2,3\ninput x\nnode r relu t9 y\n")
    assert e.value.status == _lib.AC_ERR_GRAPH
    cg = _c_graph("tiny")
    for bad in ["autochunk-plan 1\nregion s=softmax e=softmax n=2 dims=2\n",     # softmax dim: BREAK
                "autochunk-plan 1\nregion s=scores e=pv n=99999 dims=0\n",       # n > extent
                "autochunk-plan 1\nregion s=nope e=pv n=2 dims=0\n",
                "autochunk-plan 1\nregion s=scores e=pv n=2 dims=0\nregion s=softmax e=proj_o n=2 dims=0\n"]:
        with pytest.raises(_lib.ACError) as e:
            api.plan_parse(cg, bad)
        assert e.value.status == _lib.AC_ERR_PLAN
    p = api.ac_plan(cg, int(0.2 * memory.profile(workloads.config("tiny")).peak_bytes))
    assert p.status == _lib.AC_ERR_BUDGET and p.num_regions > 0


# NEXT f3: stacked blocks (multi-block plans; the DP runs one pass per region as the
# peak moves from block to block)
STACKS = [("transformer", 512, 64, 4, 256, True, 3), ("attn_only", 512, 64, 4, 0, False, 2),
          ("tri_attn_pair", 48, 16, 2, 8, False, 2)]


@pytest.mark.parametrize("kind,N,d,h,f,causal,L", STACKS)
def test_stack_documents_identical(kind, N, d, h, f, causal, L):
    a = api.graph_block(kind, N, d, h, f, causal, "bf16", name="stack", layers=L).serialize()
    assert a == og.serialize(workloads.block(kind, N, d, h, f, causal, "bf16", name="stack", layers=L))


@pytest.mark.parametrize("kind,N,d,h,f,causal,L", STACKS)
@pytest.mark.parametrize("frac", [0.5, 0.2, 0.1])
def test_stack_plans_bit_exact(kind, N, d, h, f, causal, L, frac):
    og_g = workloads.block(kind, N, d, h, f, causal, "bf16", name="stack", layers=L)
    budget = int(frac * memory.profile(og_g).peak_bytes)
    ref = select.select(og_g, budget)
    g = api.graph_block(kind, N, d, h, f, causal, "bf16", name="stack", layers=L)
    p = api.ac_plan(g, budget)
    assert p.serialize() == oplan.serialize(ref, og_g)
    assert p.feasible == ref.feasible
    _, per = api.estimate_memory(g, p)
    assert per == memory.estimate_with_plan(og_g, ref.regions).per_step
    if ref.feasible and frac <= 0.2:
        # every block's attention peak had to be chunked: one region per block at least
        assert p.num_regions >= L


# NEXT f3: max inference length under a budget (SPEC cmd_maxlen S:478-486)
@pytest.mark.parametrize("kind,d,h,f,causal,L,budget,step,cap", [
    ("transformer", 64, 4, 256, True, 1, 64 << 20, 128, 1 << 20),
    ("transformer", 64, 4, 256, False, 2, 32 << 20, 128, 1 << 20),
    ("tri_attn_pair", 16, 2, 8, False, 1, 64 << 20, 8, 1 << 12),
])
def test_max_length_matches_oracle(kind, d, h, f, causal, L, budget, step, cap):
    from oracle import maxlen
    got = api.max_length(kind, d, h, f, causal, "bf16", budget, layers=L, step=step, cap=cap)
    ref = maxlen.max_length(kind, d, h, f, causal, "bf16", budget, layers=L, step=step, cap=cap)
    assert (got["unchunked"], got["chunked"]) == (ref["unchunked"], ref["chunked"])
    # SPEC AC-4 floors: >= 3x for the 1D attention family, >= 2x for the 2D family
    assert got["ratio"] >= (2.0 if kind == "tri_attn_pair" else 3.0)
    # the lengths are maxima: one step more no longer fits
    g = api.graph_block(kind, got["chunked"] + step, d, h, f, causal, "bf16", name="maxlen", layers=L)
    assert not api.ac_plan(g, budget).feasible
    g = api.graph_block(kind, got["unchunked"] + step, d, h, f, causal, "bf16", name="maxlen", layers=L)
    assert api.estimate_memory(g)[0].peak_bytes >= budget


def test_max_length_unbounded_budget_hits_cap():
    """budget -> infinity: both lengths reach the search cap, ratio 1."""
    got = api.max_length("transformer", 64, 4, 256, True, "bf16", 1 << 60, step=128, cap=1 << 14)
    assert got["unchunked"] == got["chunked"] == 1 << 14 and got["ratio"] == 1.0


# ------------------------------------------------ R25: planned == arena + caller (no GPU)
def _arena_cases():
    from oracle import workloads
    return [
        (workloads.config("gpt"), None),
        (workloads.config("unet"), None),
        (workloads.config("af"), None),
        (workloads.block("transformer", 1024, 256, 4, 512, True, "bf16", name="m"),
         "region s=scores e=pv n=32 dims=0"),
        (workloads.block("transformer", 1024, 256, 4, 512, True, "bf16", name="m"),
         "region s=proj_q e=ffn2 n=4 dims=0"),
        (workloads.block("attn_only", 4096, 256, 4, 0, False, "bf16", name="h"), "region s=scores e=pv n=4 dims=1"),
        (workloads.tri_attn_pair(64, 128, 4, 32, "bf16", name="t"),
         "region s=row_scores e=row_pv n=4 dims=0\nregion s=col_scores e=col_pv n=4 dims=1"),
        (workloads.tri_attn_pair(64, 128, 4, 32, "bf16", name="t"),
         "region s=row_scores e=row_pv n=2 dims=1\nregion s=col_scores e=col_pv n=2 dims=0"),
        (workloads.transformer(512, 256, 4, 512, True, "bf16", name="st", layers=2), None),
    ]


@pytest.mark.parametrize("case", range(9))
def test_arena_equals_planned_per_step(case):
    """ac_plan_arena_profile (the arena ac_exec_create lays out) + the caller-held
    inputs / outputs the oracle's Eq. 2 model has live at each step == the per-step
    estimate, at EVERY step, for planned (ac_plan at 20 %) and user plans; and the
    arena has no fragmentation at its peak."""
    from oracle import graph as og_graph, memory, select
    og, txt = _arena_cases()[case]
    cg = api.graph_parse(og_graph.serialize(og))
    if txt is None:
        plan = api.ac_plan(cg, int(0.2 * memory.profile(og).peak_bytes))
        regions = select.select(og, int(0.2 * memory.profile(og).peak_bytes)).regions
    else:
        plan = api.plan_parse(cg, "autochunk-plan 1\n" + txt + "\n")
        from oracle import search
        names = [n.id for n in og.nodes]
        regions = [search.candidate_for(og, names.index(a), names.index(b), d).with_n(n)
                   for a, b, n, d in oplan.parse_user_regions("autochunk-plan 1\n" + txt + "\n")]
    live, peak, ctl = api.arena_profile(plan)
    est = memory.estimate_with_plan(og, regions)
    prof, per = api.estimate_memory(cg, plan)
    assert per == est.per_step
    callers = set(og.inputs) | set(og.outputs)
    tot = []
    for s_ in range(len(og.nodes)):
        caller = sum(b for t, b in est.live_sets[s_].items() if t in callers)
        assert live[s_] + caller == est.per_step[s_], (s_, og.nodes[s_].id, live[s_], caller, est.per_step[s_])
        tot.append(live[s_] + caller)
    assert max(tot) == prof.peak_bytes and max(live) == peak
    assert plan.workspace_bytes() - ctl == peak   # size-ordered first fit: no holes at the peak


@pytest.mark.parametrize("name,frac", [("gpt_fa", 0.9), ("gpt", 0.2), ("af", 0.2), ("tiny", 0.5)])
def test_normalized_plans_bit_exact(name, frac):
    """AC_FLAG_NORMALIZE (R27): the C++ planner and the oracle agree byte for byte
    (plan text incl. every cost term) at the configs' sizes."""
    og_g = workloads.config(name)
    budget = int(frac * memory.profile(og_g).peak_bytes)
    ref = select.select(og_g, budget, select.CostParams(normalize=True, alpha=1.0, beta=1.0, gamma=-1.0, lam=1.0))
    got = api.ac_plan(_c_graph(name), budget, api.cost_params(flags=_lib.AC_FLAG_NORMALIZE, alpha=1.0, beta=1.0,
                                                               gamma=-1.0, lam=1.0))
    assert got.serialize() == oplan.serialize(ref, og_g)


def test_chunk_pipeline_schedule(monkeypatch):
    """ac_plan_chunk_pipeline (host only): the fused-attention block's region
    [attn ... ffn2] is pipelined and chunk k's attention waits only for chunk k-1's
    out-projection (the arena gives the attention output the LN2 output's bytes, not
    the FFN hidden's); an f2 region run with the chunk-loop overlap is not pipelined;
    waits stay inside their region; AC_PIPELINE=0 / AC_OVERLAP=0 turn it off."""
    from oracle import graph as og_graph
    def sched(name, txt):
        g = workloads.config(name)
        cg = api.graph_parse(og_graph.serialize(g))
        plan = api.plan_parse(cg, "autochunk-plan 1\n" + txt)
        w, p = plan.chunk_pipeline()
        ids = [n.id for n in g.nodes]
        return {ids[i]: ids[w[i]] for i in range(len(ids)) if w[i] >= 0}, p, ids
    waits, p, ids = sched("gpt_fa", "region s=attn e=ffn2 n=16 dims=0\n")
    assert p == [1] and waits["attn"] == "proj_o"
    assert set(waits) <= set(ids[ids.index("attn"): ids.index("ffn2") + 1])
    waits, p, _ = sched("gpt", "region s=scores e=pv n=8 dims=0\n")
    assert p == [0]
    waits, p, _ = sched("gpt_fa", "region s=ln2 e=ffn2 n=2 dims=0\n")
    assert p == [1] and waits["ln2"] == "ffn1"
    monkeypatch.setenv("AC_PIPELINE", "0")
    assert sched("gpt_fa", "region s=attn e=ffn2 n=16 dims=0\n")[1] == [0]
    monkeypatch.delenv("AC_PIPELINE")
    monkeypatch.setenv("AC_OVERLAP", "0")
    assert sched("gpt_fa", "region s=attn e=ffn2 n=16 dims=0\n")[1] == [0]
