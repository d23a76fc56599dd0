"""GPU path (ac_run through the C ABI) vs the fp64 oracle, element by element.
Tolerances (north_star): fp32 path 1e-4, bf16 path 2e-2, normwise max relative
error per output tensor (R18)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import blocks, executor, memory, select, workloads  # noqa: E402

TOL = {"f32": 1e-4, "bf16": 2e-2}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _gu():
    import gpu_util
    return gpu_util


def _unfused_base(cg, og, dev):
    import os
    gu = _gu()
    old = os.environ.get("AC_FUSE_SOFTMAX")
    os.environ["AC_FUSE_SOFTMAX"] = "0"
    try:
        base, _ = gu.run(cg, gu.empty_plan(cg), og, dev)
        torch.cuda.synchronize()
    finally:
        if old is None:
            del os.environ["AC_FUSE_SOFTMAX"]
        else:
            os.environ["AC_FUSE_SOFTMAX"] = old
    return base


def _check_all_plans(og, plans, seed=0):
    gu = _gu()
    from paper_2401_10652_b200 import api
    cg = gu.c_graph(og)
    vals, dev = gu.make_values(og, seed)
    ref = executor.run(og, vals)
    base, _ = gu.run(cg, gu.empty_plan(cg), og, dev)
    dt = og.tensors[og.outputs[0]].dtype
    for o in og.outputs:
        assert gu.rel_err(base[o], ref[o]) < TOL[dt], ("unchunked", o)
    for txt in plans:
        plan = api.plan_parse(cg, txt) if isinstance(txt, str) else txt
        got, ex = gu.run(cg, plan, og, dev)
        torch.cuda.synchronize()
        for o in og.outputs:
            err = gu.rel_err(got[o], ref[o])
            assert err < TOL[dt], (txt, o, err)
            # chunked == unchunked bitwise: tiles never depend on the chunking.
            # A plan that cuts a scores -> softmax -> PV chain across regions runs that
            # chain unfused, so it is compared with the unfused unchunked run.
            if not torch.equal(got[o], base[o]):
                assert torch.equal(got[o], _unfused_base(cg, og, dev)[o]), (txt, o)
        st = ex.stats()
        assert st.launches > 0 and st.chunks_run >= 1
    return cg


def test_tiny_fp32_forced_chunk32():
    og = workloads.config("tiny")
    _check_all_plans(og, [
        "autochunk-plan 1\nregion s=scores e=pv n=8 dims=0\n",      # attention region, chunk_len 32
        "autochunk-plan 1\nregion s=proj_q e=ffn2 n=8 dims=0\n",    # whole block on rows
        "autochunk-plan 1\nregion s=scores e=pv n=32 dims=0\n",     # reading R1 alternative (len 8)
        "autochunk-plan 1\nregion s=scores e=pv n=2 dims=1\n",      # heads
        "autochunk-plan 1\nregion s=ln2 e=ffn2 n=7 dims=0\n",       # ragged FFN chunks
    ])


def test_tiny_fp32_ac_plan_best_effort():
    gu = _gu()
    from paper_2401_10652_b200 import api
    og = workloads.config("tiny")
    cg = gu.c_graph(og)
    plan = api.ac_plan(cg, int(0.2 * memory.profile(og).peak_bytes))
    assert not plan.feasible
    _check_all_plans(og, [plan])


@pytest.mark.parametrize("N,causal", [(1024, True), (1024 + 96, True), (768, False)])
def test_small_gpt_bf16(N, causal):
    og = workloads.block("transformer", N, 256, 4, 1024, causal, "bf16", name="gpt_small")
    _check_all_plans(og, [
        "autochunk-plan 1\nregion s=scores e=pv n=4 dims=0\n",
        "autochunk-plan 1\nregion s=scores e=pv n=3 dims=0\n",      # ragged chunks (unaligned: masked path)
        "autochunk-plan 1\nregion s=proj_q e=ffn2 n=4 dims=0\n",
    ])


@pytest.mark.parametrize("kind,N,plan", [
    ("transformer", 1024, "region s=scores e=pv n=4 dims=0"),
    ("transformer", 1024, "region s=scores e=pv n=32 dims=0"),          # 32-row chunks: padded e-tiles
    ("transformer", 1024, "region s=proj_q e=ffn2 n=4 dims=0"),
    ("transformer", 1024, ""),
    ("attn_only", 4096, "region s=scores e=pv n=4 dims=1"),
    ("tri", 64, "region s=row_scores e=row_pv n=4 dims=0\nregion s=col_scores e=col_pv n=4 dims=1"),
    ("tri", 64, "region s=row_scores e=row_pv n=2 dims=1\nregion s=col_scores e=col_pv n=2 dims=0"),
])
def test_planned_peak_equals_arena(kind, N, plan):
    """R25 exactness at small sizes: ac_estimate_memory(plan).peak == the arena's
    activation high-water + the caller-held inputs / outputs live at the peak step
    (the fused chains' e-tiles padded to 128 rows and their statistics included)."""
    gu = _gu()
    from paper_2401_10652_b200 import api
    if kind == "tri":
        og = workloads.tri_attn_pair(N, 128, 4, 32, "bf16", name="af_m")
    else:
        og = workloads.block(kind, N, 256, 4, 512, kind == "transformer", "bf16", name="m")
    cg = gu.c_graph(og)
    p = api.plan_parse(cg, "autochunk-plan 1\n" + plan + ("\n" if plan else ""))
    vals, dev = gu.make_values(og, 0)
    _, ex = gu.run(cg, p, og, dev)
    st = ex.stats()
    prof, per = api.estimate_memory(cg, p)
    live, peak, ctl = api.arena_profile(p)
    assert st.planned_peak == prof.peak_bytes and st.arena_live_peak == peak and st.control_bytes == ctl
    # the executor's arena is the one ac_plan_arena_profile lays out: its per-step live
    # slot bytes + the caller tensors live at that step are the per-step estimate (the
    # CPU test checks that per step); here: the run allocated exactly that workspace
    assert st.workspace_high_water == p.workspace_bytes() and max(live) == peak


def test_small_unet_bf16():
    og = workloads.block("attn_only", 512, 640, 10, 0, False, "bf16", name="unet_small")
    _check_all_plans(og, ["autochunk-plan 1\nregion s=scores e=pv n=4 dims=0\n",
                          "autochunk-plan 1\nregion s=scores e=pv n=8 dims=0\n"])


@pytest.mark.parametrize("plan", ["region s=scores e=pv n=4 dims=1", "region s=scores e=pv n=2 dims=1",
                                  "region s=scores e=pv n=4 dims=0"])
def test_heads_cut_splitk_overlap_bf16(plan):
    """Non-causal rows of >= 4096 keys: the f2 PV runs split-K and the chunk loop
    overlaps (both default); a heads cut shrinks each launch's batch count, which
    the overlap control block's split-K counters must follow.
    The gpu_util canary checks the run stays inside its workspace."""
    og = workloads.block("attn_only", 4096, 256, 4, 0, False, "bf16", name="unet_heads")
    _check_all_plans(og, ["autochunk-plan 1\n" + plan + "\n"])


def test_small_af_bf16():
    # (at 64 residues the held z / q / k / v / g floor the R25 peak near 39 %: 40 % budget)
    og = workloads.tri_attn_pair(64, 128, 4, 32, "bf16", name="af_small")
    plan = select.select(og, int(0.4 * memory.profile(og).peak_bytes))
    gu = _gu()
    from paper_2401_10652_b200 import api
    cg = gu.c_graph(og)
    p = api.ac_plan(cg, int(0.4 * memory.profile(og).peak_bytes))
    assert p.feasible
    assert p.num_regions == len(plan.regions)
    _check_all_plans(og, [p,
                          "autochunk-plan 1\nregion s=row_scores e=row_pv n=4 dims=0\n"
                          "region s=col_scores e=col_pv n=4 dims=1\n"])


def test_gpt_full_size_sampled_rows():
    """BASELINE configs[1] at full size, the plan ac_plan picks at 20 %, in the
    launch configuration bench.py times; sampled rows vs the oracle."""
    gu = _gu()
    from paper_2401_10652_b200 import api
    og = workloads.config("gpt")
    cg = gu.c_graph(og)
    budget = int(0.2 * memory.profile(og).peak_bytes)
    plan = api.ac_plan(cg, budget)
    vals, dev = gu.make_values(og, 0)
    got, ex = gu.run(cg, plan, og, dev)
    torch.cuda.synchronize()
    rows = blocks.sample_rows(16384, 2048, 48)
    ref = blocks.transformer_rows(og, vals, rows)
    err = gu.rel_err(got["y"][torch.from_numpy(rows).cuda()], ref["y"])
    assert err < 2e-2, err
    st = ex.stats()
    assert st.planned_peak < budget
    # the IR describes what runs (R25): the planned peak (Eq. 2 with the fused chain's
    # e-tiles and statistics) equals the activation high-water of the arena plus the
    # caller-held tensors live at the peak step, exactly; no fragmentation
    prof, per = api.estimate_memory(cg, plan)
    live, peak, ctl = api.arena_profile(plan)
    assert st.planned_peak == prof.peak_bytes and st.arena_live_peak == peak and st.control_bytes == ctl
    assert st.planned_peak == max(live[s] + (per[s] - live[s]) for s in range(len(per)))
    assert st.planned_peak - st.arena_live_peak == 2 * 16384 * 1024 * 2 - 16384 * 1024 * 2  # x only at the peak
    assert st.workspace_high_water - st.control_bytes == st.arena_live_peak
    assert st.control_bytes < 1 << 20


def test_gpt_full_size_whole_block_plan():
    """The forced whole-block plan at the full GPT size ([proj_q ... ffn2]
    on 2048-row chunks, K / V hoisted, the N x 4d FFN hidden never exists): sampled rows
    vs the oracle, and the same bits as the planner's attention-region plan (tiles and
    row kernels never depend on the chunking)."""
    gu = _gu()
    from paper_2401_10652_b200 import api
    og = workloads.config("gpt")
    cg = gu.c_graph(og)
    vals, dev = gu.make_values(og, 0)
    got, ex = gu.run(cg, api.plan_parse(cg, "autochunk-plan 1\nregion s=proj_q e=ffn2 n=8 dims=0\n"), og, dev)
    torch.cuda.synchronize()
    rows = blocks.sample_rows(16384, 2048, 24)
    ref = blocks.transformer_rows(og, vals, rows)
    assert gu.rel_err(got["y"][torch.from_numpy(rows).cuda()], ref["y"]) < 2e-2
    other, _ = gu.run(cg, api.plan_parse(cg, "autochunk-plan 1\nregion s=scores e=pv n=8 dims=0\n"), og, dev)
    torch.cuda.synchronize()
    assert torch.equal(got["y"], other["y"])


@pytest.mark.parametrize("causal", [True, False])
def test_fused_softmax_pv_vs_unfused(monkeypatch, causal):
    """NEXT f2: scores -> softmax -> PV with the normalisation folded into the PV
    operand path (AC_FUSE_SOFTMAX=1, default) against the three-kernel path
    (AC_FUSE_SOFTMAX=0): both within the bf16 tolerance of the oracle, smaller
    workspace, one launch fewer per chunk (the PV folds each row's (M, 1/L) itself)."""
    gu = _gu()
    from paper_2401_10652_b200 import api
    og = workloads.block("transformer", 1024 + 96, 256, 4, 1024, causal, "bf16", name="gpt_small")
    cg = gu.c_graph(og)
    vals, dev = gu.make_values(og, 3)
    ref = executor.run(og, vals)
    txt = "autochunk-plan 1\nregion s=scores e=pv n=4 dims=0\n"
    res = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("AC_FUSE_SOFTMAX", flag)
        plan = api.plan_parse(cg, txt)
        got, ex = gu.run(cg, plan, og, dev)
        torch.cuda.synchronize()
        res[flag] = (got["y"], ex.stats(), plan.workspace_bytes())
        assert gu.rel_err(got["y"], ref["y"]) < TOL["bf16"], flag
    (y0, s0, w0), (y1, s1, w1) = res["0"], res["1"]
    assert s1.launches == s0.launches - 4
    assert w1 < w0
    # same bf16 P rounding point, different exp/sum order: close, not bitwise
    assert gu.rel_err(y1, y0.double().cpu().numpy()) < 1e-2


@pytest.mark.parametrize("split", ["0", "1"])
def test_fused_pv_split_k_chunk_invariant(monkeypatch, split):
    """Fixed split-K of the fused PV (AC_PV_SPLITK=1 forces it on, 0 off; keys cut
    into 4 granules at fixed positions): bf16 tolerance vs the oracle and chunked ==
    unchunked bitwise, causal and not; each granule folds its own (max, sum) and the
    tile's last unit (a finish warp group) merges them in granule order."""
    monkeypatch.setenv("AC_PV_SPLITK", split)
    for causal in (True, False):
        og = workloads.block("attn_only", 2048 + 320, 256, 4, 0, causal, "bf16", name="pv_split")
        _check_all_plans(og, ["autochunk-plan 1\nregion s=scores e=pv n=4 dims=0\n",
                              "autochunk-plan 1\nregion s=scores e=pv n=3 dims=0\n"], seed=5)


@pytest.mark.parametrize("nres", [64, 192])
def test_af_fused_softmax_vs_unfused(monkeypatch, nres):
    """NEXT f2 on the AlphaFold triangle chains (tri_scores + bias -> softmax ->
    gated tri_pv, row and column attention): fused (default) and three-kernel
    paths both within the bf16 tolerance of the oracle, chunked == unchunked
    bitwise for each, one launch fewer per chunk of each region.
    nres = 192 leaves a ragged 128-row tile and a ragged key slab."""
    gu = _gu()
    from paper_2401_10652_b200 import api
    og = workloads.tri_attn_pair(nres, 128, 4, 32, "bf16", name="af_f2")
    cg = gu.c_graph(og)
    plans = ["autochunk-plan 1\nregion s=row_scores e=row_pv n=4 dims=0\n"
             "region s=col_scores e=col_pv n=4 dims=1\n",
             "autochunk-plan 1\nregion s=row_scores e=row_pv n=3 dims=0\n"]
    res = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("AC_FUSE_SOFTMAX", flag)
        _check_all_plans(og, plans, seed=7)
        plan = api.plan_parse(cg, plans[0])
        vals, dev = gu.make_values(og, 7)
        got, ex = gu.run(cg, plan, og, dev)
        torch.cuda.synchronize()
        res[flag] = (got[og.outputs[0]], ex.stats(), plan.workspace_bytes())
    (y0, s0, w0), (y1, s1, w1) = res["0"], res["1"]
    assert s1.launches == s0.launches - 8  # no combine launch: the PV folds (M, 1/L) per chunk
    # (no workspace claim at these sizes: e-tiles pad the rows to 128-row tiles)
    assert gu.rel_err(y1, y0.double().cpu().numpy()) < 1e-2


def test_stacked_blocks_multi_region_plan():
    """NEXT f3: a stack of 3 causal blocks; ac_plan at 25 % and 20 % chunks every
    block's attention (one region per block, multi-pass DP); vs the oracle and
    chunked == unchunked bitwise; plus a user plan whose 96-row chunks take the
    unaligned masked causal path."""
    gu = _gu()
    from paper_2401_10652_b200 import api
    og = workloads.transformer(2048, 256, 4, 512, True, "bf16", name="stack", layers=3)
    cg = gu.c_graph(og)
    plans = [api.ac_plan(cg, int(fr * memory.profile(og).peak_bytes)) for fr in (0.25, 0.2)]
    for p in plans:
        assert p.feasible and p.num_regions >= 3
    plans.append("autochunk-plan 1\nregion s=L0_scores e=L0_pv n=22 dims=0\nregion s=L2_scores e=L2_pv n=3 dims=0\n")
    _check_all_plans(og, plans, seed=11)


def test_long_sequence_beyond_unchunked_capacity():
    """NEXT f3: a GPT block at 131072 tokens, whose unchunked activations (> 1 TB)
    exceed B200 HBM, runs under the plan ac_plan picks for a 96 GiB budget; sampled
    output rows vs the fp64 oracle."""
    gu = _gu()
    from paper_2401_10652_b200 import api
    N = 131072
    og = workloads.block("transformer", N, 1024, 16, 4096, True, "bf16", name="gpt_long")
    assert memory.profile(og).peak_bytes > 200 << 30
    cg = gu.c_graph(og)
    plan = api.ac_plan(cg, 96 << 30)
    assert plan.feasible
    vals, dev = gu.make_values(og, 0)
    got, ex = gu.run(cg, plan, og, dev)
    torch.cuda.synchronize()
    rows = np.array([0, 1, 4095, 65536, N - 129, N - 1])
    ref = blocks.transformer_rows(og, vals, rows)
    err = gu.rel_err(got["y"][torch.from_numpy(rows).cuda()], ref["y"])
    assert err < 2e-2, err
    assert ex.stats().planned_peak < 96 << 30


@pytest.mark.parametrize("N,causal", [(1024, True), (1024 + 96, True), (768, False), (200, True)])
def test_fused_attention_block(N, causal):
    """NEXT f1: the transformer block with attention as one fused kernel (no N x N
    tensor) vs the fp64 oracle; row-chunked plans (attention and FFN
    regions, ragged) equal the unchunked run bitwise."""
    og = workloads.block("transformer_fa", N, 256, 4, 1024, causal, "bf16", name="gpt_fa")
    _check_all_plans(og, [
        "autochunk-plan 1\nregion s=attn e=ffn2 n=4 dims=0\n",
        "autochunk-plan 1\nregion s=ln2 e=ffn2 n=3 dims=0\n",
        "autochunk-plan 1\nregion s=proj_q e=proj_o n=5 dims=0\n",
    ], seed=4)


def test_fused_attention_two_tile_units():
    """The fused attention's two-tile units (NT = 2, >= 296 tiles: 16 heads x 32 row
    tiles unchunked) and one-tile units (NT = 1: a 1024-row chunk is 128 tiles) compute
    every row with the same job order and arithmetic: chunked == unchunked bitwise, and
    both vs the fp64 oracle."""
    og = workloads.block("transformer_fa", 4096, 1024, 16, 1024, True, "bf16", name="fa_nt2")
    _check_all_plans(og, ["autochunk-plan 1\nregion s=attn e=ffn2 n=4 dims=0\n"], seed=6)


def test_fused_attention_regime_plan():
    """NEXT f1 at the GPT config: ac_plan under a budget below the fused block's
    unchunked peak chunks the FFN-side intermediates; sampled rows vs the oracle."""
    gu = _gu()
    from paper_2401_10652_b200 import api
    og = workloads.config("gpt_fa")
    cg = gu.c_graph(og)
    pk = memory.profile(og).peak_bytes
    plan = api.ac_plan(cg, int(0.95 * pk))
    assert plan.feasible and plan.num_regions >= 1
    vals, dev = gu.make_values(og, 0)
    got, ex = gu.run(cg, plan, og, dev)
    torch.cuda.synchronize()
    rows = blocks.sample_rows(16384, 1024, 24)
    ref = blocks.transformer_rows(workloads.config("gpt"), vals, rows)
    assert gu.rel_err(got["y"][torch.from_numpy(rows).cuda()], ref["y"]) < 2e-2


PIPE_CASES = {
    # f1 region: chunk k's attention runs beside chunk k-1's FFN (only the o / h
    # scratch orders them)
    "gpt_fa": (lambda: workloads.block("transformer_fa", 2048, 256, 4, 1024, True, "bf16", name="pipe_fa"),
               "autochunk-plan 1\nregion s=attn e=ffn2 n=4 dims=0\n", True),
    # whole block with its causal f2 chain run without the chunk-loop overlap
    "gpt_block": (lambda: workloads.transformer(1024, 256, 4, 512, True, "bf16", name="pipe_blk"),
                  "autochunk-plan 1\nregion s=proj_q e=ffn2 n=4 dims=0\n", None),
    # triangle attention pair (the triangle chains run without the overlap by default)
    "af": (lambda: workloads.tri_attn_pair(192, 128, 4, 32, "bf16", name="pipe_af"),
           "autochunk-plan 1\nregion s=row_scores e=row_pv n=4 dims=1\nregion s=col_scores e=col_pv n=6 dims=0\n",
           None),
    # ragged FFN region, odd chunk count
    "ffn_ragged": (lambda: workloads.block("transformer_fa", 1024 + 96, 256, 4, 1024, True, "bf16", name="pipe_rag"),
                   "autochunk-plan 1\nregion s=ln2 e=ffn2 n=5 dims=0\n", True),
}


@pytest.mark.parametrize("name", list(PIPE_CASES))
def test_chunk_pipelining(monkeypatch, name):
    """Chunk pipelining over two streams (chunk k waits only for the launches of chunk
    k-1 that touch the same workspace bytes): bitwise equal to the same plan run on
    one stream (AC_PIPELINE=0), to the unchunked run, also under CUDA graph capture,
    and the f1 / FFN regions really run their odd chunks on the second stream."""
    gu = _gu()
    from paper_2401_10652_b200 import api
    mk, txt, expect = PIPE_CASES[name]
    og = mk()
    cg = gu.c_graph(og)
    plan = api.plan_parse(cg, txt)
    _, dev = gu.make_values(og, 11)
    base, _ = gu.run(cg, gu.empty_plan(cg), og, dev)
    got, ex = gu.run(cg, plan, og, dev)
    torch.cuda.synchronize()
    st = ex.stats()
    if expect:
        assert st.pipelined_chunks > 0
    monkeypatch.setenv("AC_PIPELINE", "0")
    one, ex1 = gu.run(cg, plan, og, dev)
    torch.cuda.synchronize()
    assert ex1.stats().pipelined_chunks == 0
    monkeypatch.delenv("AC_PIPELINE")
    for o in og.outputs:
        assert torch.equal(got[o], one[o]), (name, o)
        if not torch.equal(got[o], base[o]):
            assert torch.equal(got[o], _unfused_base(cg, og, dev)[o]), (name, o)
    # captured: the side stream joins the capture through the fork event
    ws = torch.empty(max(plan.workspace_bytes(), 16), dtype=torch.uint8, device="cuda")
    exg = api.Exec(plan, ws)
    outs = {o: torch.full_like(got[o], float("nan")) for o in og.outputs}
    ins = {t: dev[t] for t in og.inputs + og.weights}
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    exg.run(ins, outs, s)                     # warm-up (module loads) outside the capture
    s.synchronize()
    for o in outs:
        outs[o].fill_(float("nan"))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        exg.run(ins, outs, s)
    graph.replay()
    torch.cuda.synchronize()
    for o in og.outputs:
        assert torch.equal(outs[o], got[o]), (name, "graph", o)


def test_af_chunk_overlap_opt_in(monkeypatch):
    """The chunk-loop overlap on the triangle chains (AC_OVERLAP_TRI=1: paired
    short-chunk scores with dynamic tiles waiting on per-batch epochs of the previous
    chunk's PV) keeps the results: vs the oracle and bitwise equal to unchunked."""
    monkeypatch.setenv("AC_OVERLAP_TRI", "1")
    og = workloads.tri_attn_pair(192, 128, 4, 32, "bf16", name="af_ov")
    _check_all_plans(og, ["autochunk-plan 1\nregion s=row_scores e=row_pv n=4 dims=1\n"
                          "region s=col_scores e=col_pv n=6 dims=0\n"], seed=9)


def test_ac_run_cuda_graph_capture():
    """ac_run is stream-ordered with no host synchronisation, so a chunked run can be
    captured into a CUDA graph and replayed: the replay reproduces the direct run
    bitwise (f2 chain with the chunk-loop overlap on a non-causal block, and a causal
    block in stream order)."""
    gu = _gu()
    from paper_2401_10652_b200 import api
    for causal in (False, True):
        og = workloads.block("attn_only", 2048 + 320, 256, 4, 0, causal, "bf16", name="cg")
        cg = gu.c_graph(og)
        vals, dev = gu.make_values(og, 19)
        plan = api.plan_parse(cg, "autochunk-plan 1\nregion s=scores e=pv n=4 dims=0\n")
        got, ex = gu.run(cg, plan, og, dev)
        torch.cuda.synchronize()
        ws = torch.empty(max(plan.workspace_bytes(), 16), dtype=torch.uint8, device="cuda")
        ex2 = api.Exec(plan, ws)
        ins = {t: dev[t] for t in og.inputs + og.weights}
        outs = {o: torch.empty_like(got[o]) for o in og.outputs}
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ex2.run(ins, outs, stream=s)  # warm-up (function attributes, tensor maps)
        s.synchronize()
        for o in outs:
            outs[o].zero_()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ex2.run(ins, outs, stream=s)
        g.replay()
        torch.cuda.synchronize()
        for o in og.outputs:
            assert torch.equal(outs[o], got[o]), (causal, o)


@pytest.mark.parametrize("ov", ["0", "1"])
def test_causal_chunk_overlap(monkeypatch, ov):
    """The chunk-loop overlap on causal attention chains (dynamic scores tiles of chunk
    k+1 waiting on per-head epochs of chunk k's PV, PDL launches; on by default,
    AC_OVERLAP_CAUSAL=0 off) keeps the results: vs the oracle and bitwise equal to
    unchunked, also on a 2-block stack."""
    monkeypatch.setenv("AC_OVERLAP_CAUSAL", ov)
    og = workloads.block("attn_only", 2048 + 320, 256, 4, 0, True, "bf16", name="ovc")
    _check_all_plans(og, ["autochunk-plan 1\nregion s=scores e=pv n=4 dims=0\n",
                          "autochunk-plan 1\nregion s=scores e=pv n=3 dims=0\n"], seed=17)
    og = workloads.transformer(512, 256, 4, 512, True, "bf16", name="ovs", layers=2)
    _check_all_plans(og, ["autochunk-plan 1\nregion s=L0_scores e=L0_pv n=4 dims=0\n"
                          "region s=L1_scores e=L1_pv n=2 dims=0\n"], seed=17)


@pytest.mark.parametrize("kind", ["transformer", "transformer_fa"])
def test_degenerate_sizes(kind):
    """Degenerate cases: the smallest aligned bf16 sequence (8 tokens)
    with chunk_len 1 (n = extent) on the attention region and on the whole block (K / V
    projections hoisted), and a ragged n = 3 FFN region; sequences that break the
    16-byte row alignment of the bf16 tensor-core operands (9 tokens) are refused with
    AC_ERR_UNSUPPORTED, never run wrong."""
    from paper_2401_10652_b200 import api, _lib
    gu = _gu()
    og = workloads.block(kind, 8, 256, 4, 512, True, "bf16", name="deg")
    attn = ("scores", "pv") if kind == "transformer" else ("attn", "proj_o")
    _check_all_plans(og, ["autochunk-plan 1\nregion s=%s e=%s n=8 dims=0\n" % attn,
                          "autochunk-plan 1\nregion s=proj_q e=ffn2 n=8 dims=0\n",
                          "autochunk-plan 1\nregion s=ln2 e=ffn2 n=3 dims=0\n"], seed=2)
    og9 = workloads.block(kind, 9, 256, 4, 512, True, "bf16", name="deg9")
    cg = gu.c_graph(og9)
    vals, dev = gu.make_values(og9, 2)
    with pytest.raises(_lib.ACError) as ei:
        gu.run(cg, gu.empty_plan(cg), og9, dev)
    assert ei.value.status == _lib.AC_ERR_UNSUPPORTED


@pytest.mark.parametrize("N", [1, 9])
def test_degenerate_sizes_fp32(N):
    """fp32 (SIMT) path at 1 and 9 tokens, chunk_len 1 plans: vs the oracle (1e-4) and
    chunked == unchunked bitwise."""
    og = workloads.block("transformer", N, 64, 2, 128, True, "f32", name="deg32")
    plans = [] if N == 1 else ["autochunk-plan 1\nregion s=scores e=pv n=9 dims=0\n",
                               "autochunk-plan 1\nregion s=proj_q e=ffn2 n=9 dims=0\n"]
    _check_all_plans(og, plans, seed=2)


def test_single_key_attention_is_v():
    """Closed form: with one token the attention output is v itself,
    so the block output is x + (a Wv + bv) Wo + bo."""
    gu = _gu()
    og = workloads.block("attn_only", 1, 64, 2, 0, True, "f32", name="one")
    cg = gu.c_graph(og)
    vals, dev = gu.make_values(og, 1)
    got, _ = gu.run(cg, gu.empty_plan(cg), og, dev)
    torch.cuda.synchronize()
    x = vals["x"]
    mu, var = x.mean(-1, keepdims=True), x.var(-1, keepdims=True)
    a = (x - mu) / np.sqrt(var + 1e-5) * vals["ln1_g"] + vals["ln1_b"]
    v = a @ vals["wv"].T + vals["bv"]
    ref = x + v @ vals["wo"].T + vals["bo"]
    assert gu.rel_err(got["x1"], ref) < 1e-4


@pytest.mark.parametrize("causal", [True, False])
def test_f2_large_logit_range(causal):
    """f2 scores take each 64-key slab's first score as its exponent reference and
    redo a row against the slab max when the max exceeds it by more than 96 (log2
    units).  Wq scaled by 64 (exact in bf16) spreads the logits over hundreds of units
    so both paths run: vs the oracle on the same values, chunked == unchunked bitwise.
    At this logit scale the bf16 rounding of q and k alone moves logits by whole
    units and decides near-ties, so the reference takes q, k, vT and o rounded where
    the GPU stores them (the oracle's mirror mode, reading R17) while S stays exact,
    as in the fused chain (reading R19)."""
    gu = _gu()
    og = workloads.block("attn_only", 640, 256, 4, 0, causal, "bf16", name="wide")
    vals, dev = gu.make_values(og, 4)
    vals["wq"] = vals["wq"] * 64.0
    dev["wq"] = (dev["wq"].float() * 64.0).bfloat16()
    cg = gu.c_graph(og)
    from paper_2401_10652_b200 import api
    mir = executor.run(og, vals, mirror=True, keep_all=True)
    q, k, vt = mir["q"], mir["k"], mir["vt"]                     # [N,h,dh], [N,h,dh], [h,dh,N]
    sc = np.einsum("ihd,jhd->hij", q, k) / 8.0
    if causal:
        sc = np.where(np.triu(np.ones(sc.shape[1:], bool), 1)[None], -np.inf, sc)
    p = np.exp(sc - sc.max(-1, keepdims=True))
    p /= p.sum(-1, keepdims=True)
    o = np.einsum("hij,hdj->ihd", p, vt).reshape(q.shape[0], -1)
    o = torch.from_numpy(o).bfloat16().double().numpy()          # O stored in bf16
    ref = vals["x"] + o @ vals["wo"].T + vals["bo"]
    base, _ = gu.run(cg, gu.empty_plan(cg), og, dev)
    torch.cuda.synchronize()
    assert gu.rel_err(base["x1"], ref) < 2e-2
    for n in (5, 2):
        got, _ = gu.run(cg, api.plan_parse(cg, "autochunk-plan 1\nregion s=scores e=pv n=%d dims=0\n" % n), og, dev)
        torch.cuda.synchronize()
        assert torch.equal(got["x1"], base["x1"]), n


def test_af_large_logit_range():
    """The triangle chains take the same one-pass reference as the plain chains (R19: the
    slab's first score x = (q.k scale + b) log2 e, a row redone against its max when the
    slab sum exceeds 2^96, the bias of the redo read from global memory because the staging
    box already holds e).  Wq and the bias projection scaled by 64 (exact in bf16) spread
    the logits over hundreds of log2 units so the redo path runs in every launch: the
    128-row kernel (unchunked, batch-dim chunks) and the paired 64-row kernel (query-dim
    chunks of 48 rows) must give the same bits, and every output is finite."""
    gu = _gu()
    from paper_2401_10652_b200 import api
    og = workloads.tri_attn_pair(192, 128, 4, 32, "bf16", name="af_wide")
    cg = gu.c_graph(og)
    vals, dev = gu.make_values(og, 5)
    for w in ("row_wq", "col_wq", "row_wb", "col_wb"):
        dev[w] = (dev[w].float() * 64.0).bfloat16()
    base, _ = gu.run(cg, gu.empty_plan(cg), og, dev)
    torch.cuda.synchronize()
    out = og.outputs[0]
    assert torch.isfinite(base[out].float()).all()
    for txt in ("region s=row_scores e=row_pv n=4 dims=1\nregion s=col_scores e=col_pv n=4 dims=0\n",
                "region s=row_scores e=row_pv n=3 dims=0\nregion s=col_scores e=col_pv n=2 dims=1\n"):
        got, _ = gu.run(cg, api.plan_parse(cg, "autochunk-plan 1\n" + txt), og, dev)
        torch.cuda.synchronize()
        assert torch.equal(got[out], base[out]), txt


@pytest.mark.parametrize("name,rows_per_chunk", [("unet", 2048), ("vit", 8192)])
def test_full_size_sampled_rows(name, rows_per_chunk):
    """BASELINE configs at full size (UNet 16384 tokens h=10, ViT-L 65536 tokens) under
    the plan ac_plan picks at 20 % - the launch configuration bench.py times - sampled
    rows (first, last, every chunk boundary +-1, random) vs the fp64 oracle."""
    gu = _gu()
    from paper_2401_10652_b200 import api
    og = workloads.config(name)
    cg = gu.c_graph(og)
    budget = int(0.2 * memory.profile(og).peak_bytes)
    plan = api.ac_plan(cg, budget)
    assert plan.feasible
    vals, dev = gu.make_values(og, 0)
    got, ex = gu.run(cg, plan, og, dev)
    torch.cuda.synchronize()
    N = og.tensors["x"].shape[0]
    rows = blocks.sample_rows(N, rows_per_chunk, 16)
    ref = blocks.transformer_rows(og, vals, rows)
    out = og.outputs[0]
    assert gu.rel_err(got[out][torch.from_numpy(rows).cuda()], ref[out]) < 2e-2
    assert ex.stats().planned_peak < budget


@pytest.mark.parametrize("ending", [0, 1])
def test_af_full_size_sampled_pairs(ending):
    """One AlphaFold triangle attention (starting node, Alg. 13, or ending node,
    Alg. 14) at N_res = 1024, c_z = 128, H = 4, c = 32 under ac_plan at 20 % (the
    short query-dim chunks of the bench's AF config: paired 64-row kernels), sampled
    (i, j) pairs incl. chunk boundaries vs the fp64 oracle."""
    gu = _gu()
    from oracle.graph import Builder
    from paper_2401_10652_b200 import api
    N, cz, H, c = 1024, 128, 4, 32
    B = Builder("af_one", "bf16")
    B.input("z", (N, N, cz))
    workloads._tri_weights(B, "t_", cz, H, c)
    workloads._tri_attention(B, "z", "t_", N, cz, H, c, ending, "zo")
    B.output("zo")
    og = B.build()
    cg = gu.c_graph(og)
    budget = int(0.2 * memory.profile(og).peak_bytes)
    plan = api.ac_plan(cg, budget)
    assert plan.feasible and plan.num_regions >= 1
    vals, dev = gu.make_values(og, 0)
    got, _ = gu.run(cg, plan, og, dev)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    pairs = [(0, 0), (N - 1, N - 1), (63, 64), (64, 63), (511, 512)] + \
        [tuple(int(x) for x in rng.integers(0, N, 2)) for _ in range(11)]
    ref = blocks.tri_attention_pairs(og, vals, "t_", pairs, bool(ending))
    g_pairs = torch.stack([got["zo"][i, j] for i, j in pairs])
    assert gu.rel_err(g_pairs, ref) < 2e-2


def test_rank_above_six_refused():
    """ac_tensor / the executor's views carry at most 6 dims (ac.h): a rank-7 graph
    is refused at ac_exec_create with AC_ERR_UNSUPPORTED."""
    from oracle.graph import Builder
    from paper_2401_10652_b200 import _lib
    gu = _gu()
    B = Builder("rank7", "bf16")
    B.input("x", (1, 1, 1, 1, 1, 2, 64))
    B.weight("g", (64,), "ln_gamma", 64)
    B.weight("b", (64,), "ln_beta", 64)
    B.op("layernorm", ["x", "g", "b"], "y", naxes=1, eps=1e-5)
    B.output("y")
    og = B.build()
    cg = gu.c_graph(og)
    vals, dev = gu.make_values(og, 0)
    with pytest.raises(_lib.ACError) as ei:
        gu.run(cg, gu.empty_plan(cg), og, dev)
    assert ei.value.status == _lib.AC_ERR_UNSUPPORTED


def test_evoformer_pair_stack_bf16():
    """NEXT f3: the full Evoformer pair stack (triangle multiplication outgoing /
    incoming: gated channel-major projections, the tri_mul GEMM over channels, the
    channel LayerNorm written channel-last, the gated output projection; triangle
    attention starting / ending node; pair transition) vs the fp64 oracle, chunked
    == unchunked bitwise, with regions cutting each kind of node along rows (i) and
    columns (j)."""
    og = workloads.evoformer_pair(64, 128, 4, 32, "bf16", name="evo_small")
    _check_all_plans(og, [
        "autochunk-plan 1\nregion s=mo_mul e=mo_proj_o n=4 dims=0\n",
        "autochunk-plan 1\nregion s=mo_proj_ag e=mo_proj_o n=2 dims=0\n",
        "autochunk-plan 1\nregion s=mi_proj_bg e=mi_proj_o n=2 dims=1\n",
        "autochunk-plan 1\nregion s=mi_mul e=mi_lnx n=4 dims=1\n",
        "autochunk-plan 1\nregion s=tr_ln e=tr_ffn2 n=4 dims=0\n",
        "autochunk-plan 1\nregion s=row_scores e=row_pv n=4 dims=0\nregion s=col_scores e=col_pv n=4 dims=1\n"
        "region s=tr_ln e=tr_ffn2 n=2 dims=1\n",
        # channel-major projections on chunks of the second row dim (batched over the
        # first), including chunks of length 1 (the Table 1 ablation's best-effort plans)
        "autochunk-plan 1\nregion s=mo_proj_bg e=mo_proj_b n=4 dims=2\n",
        "autochunk-plan 1\nregion s=mo_proj_bg e=mo_proj_b n=64 dims=2\n",
        # both triangle chains cut across regions (the ablation's best-effort shape): both
        # run unfused, so the result equals the unfused unchunked run bitwise
        "autochunk-plan 1\nregion s=row_scores e=row_scores n=64 dims=0\nregion s=row_softmax e=row_pv n=64 dims=0\n"
        "region s=col_scores e=col_scores n=4 dims=0\nregion s=col_softmax e=col_pv n=4 dims=0\n",
    ], seed=9)
