"""The N>1 path on CPU (world_size 2, gloo): every rank asks libautochunk which
chunks it owns (ac_plan_rank_chunks, the arithmetic ac_run uses), computes only
those chunks of the region with the oracle, and the Y^c slabs are exchanged by
broadcast from their owners (the collective pattern of comm_gather_slabs).  The
gathered result must equal the unchunked single-process output bitwise
(fp64, exact reduction order)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import executor, graph as og_graph, ops, select
from oracle.graph import Builder
import synth


def _attn_graph(N=96, d=32, h=2):
    B = Builder("mr", "f64")
    B.input("x", (N, d))
    B.weight("g", (d,), "ln_gamma", d)
    B.weight("b", (d,), "ln_beta", d)
    for w in ("wq", "wk", "wv"):
        B.weight(w, (d, d), "matrix", d)
    B.op("layernorm", ["x", "g", "b"], "a", nid="ln", naxes=1, eps=1e-5)
    B.op("linear", ["a", "wq"], "q", nid="proj_q", kin=1, out=[h, d // h], act="none", trans=0, swap=0, bias=0, res=0)
    B.op("linear", ["a", "wk"], "k", nid="proj_k", kin=1, out=[h, d // h], act="none", trans=0, swap=0, bias=0, res=0)
    B.op("linear", ["a", "wv"], "vt", nid="proj_v", kin=1, out=[h, d // h], act="none", trans=1, swap=0, bias=0,
         res=0)
    B.op("attn_scores", ["q", "k"], "s", nid="scores", scale=0.25, causal=1)
    B.op("softmax", ["s"], "p", nid="softmax", dim=2)
    B.op("attn_pv", ["p", "vt"], "o", nid="pv")
    B.output("o")
    return B.build()


def _worker(rank, world, port, n_chunks, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_10652_b200 import api
    g = _attn_graph()
    spec = [("scores", "pv", n_chunks, (0,))]
    regions = select.user_plan(g, spec).regions
    cplan = api.plan_parse(api.graph_parse(og_graph.serialize(g)),
                           f"autochunk-plan 1\nregion s=scores e=pv n={n_chunks} dims=0\n")
    vals = {t: s.value for t, s in synth.make_inputs(g.input_specs(), 3).items()}
    ranges = [cplan.rank_chunks(0, q, world) for q in range(world)]
    c0, c1, L, E = ranges[rank]
    with ops.exact_order():
        mine = executor.run_chunked(g, vals, regions, chunk_ranges={0: (c0, c1)})["o"]
    y = torch.from_numpy(np.ascontiguousarray(mine))
    for q, (a, b, _, _) in enumerate(ranges):          # owner broadcasts its slab
        lo, hi = min(E, a * L), min(E, b * L)
        if hi > lo:
            slab = y[lo:hi].clone()
            dist.broadcast(slab, src=q)
            y[lo:hi] = slab
    result_q.put((rank, y.numpy(), [(a, b) for a, b, _, _ in ranges]))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_chunks", [4, 3, 8])
def test_two_rank_chunk_split_equals_single_rank(n_chunks):
    pytest.importorskip("paper_2401_10652_b200.api")
    world = 2
    port = 29500 + n_chunks + (os.getpid() % 1000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = _attn_graph()
    vals = {t: s.value for t, s in synth.make_inputs(g.input_specs(), 3).items()}
    with ops.exact_order():
        ref = executor.run(g, vals)["o"]
    ranges = res[0][2]
    assert ranges[0][0] == 0 and ranges[-1][1] == n_chunks                     # full coverage
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(len(ranges) - 1))  # no gap/overlap
    for rank, y, _ in res:
        assert np.array_equal(y, ref), rank


def _tri_row_graph(N=12, cz=8, H=2, c=4):
    """Triangle attention around the starting node up to its gated output o[i, j, h, c]
    (the region output whose chunks run along dim 1, j)."""
    from oracle import workloads
    B = Builder("mr_af", "f64")
    B.input("z", (N, N, cz))
    workloads._tri_weights(B, "row_", cz, H, c)
    B.op("layernorm", ["z", "row_ln_g", "row_ln_b"], "zn", nid="ln", naxes=1, eps=1e-5)
    B.op("linear", ["zn", "row_wb"], "bias", nid="proj_b", kin=1, out=[H], act="none", trans=1, swap=0, bias=0, res=0)
    for nm, w, tr in (("q", "row_wq", 0), ("k", "row_wk", 0), ("vt", "row_wv", 1)):
        B.op("linear", ["zn", w], nm, nid="proj_" + nm, kin=1, out=[H, c], act="none", trans=tr, swap=0, bias=0,
             res=0)
    B.op("linear", ["zn", "row_wg", "row_bg"], "g", nid="proj_g", kin=1, out=[H, c], act="sigmoid", trans=0, swap=0,
         bias=1, res=0)
    B.op("tri_scores", ["q", "k", "bias"], "s", nid="scores", scale=0.5, ending=0)
    B.op("softmax", ["s"], "p", nid="softmax", dim=3)
    B.op("tri_pv", ["p", "vt", "g"], "o", nid="pv", ending=0)
    B.output("o")
    return B.build()


def _worker_dim1(rank, world, port, n_chunks, result_q):
    """AlphaFold pattern: the region output o[i, j, h, c] is chunked along dim 1 (j);
    owners broadcast one run per outer index i (comm_gather_slabs for d > 0)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_10652_b200 import api
    g = _tri_row_graph()
    cplan = api.plan_parse(api.graph_parse(og_graph.serialize(g)),
                           f"autochunk-plan 1\nregion s=scores e=pv n={n_chunks} dims=1\n")
    regions = select.user_plan(g, [("scores", "pv", n_chunks, (1,))]).regions
    vals = {t: s.value for t, s in synth.make_inputs(g.input_specs(), 5).items()}
    ranges = [cplan.rank_chunks(0, q, world) for q in range(world)]
    c0, c1, L, E = ranges[rank]
    with ops.exact_order():
        mine = executor.run_chunked(g, vals, regions, chunk_ranges={0: (c0, c1)})["o"]
    y = torch.from_numpy(np.ascontiguousarray(mine))
    for o in range(y.shape[0]):                         # one run per outer index
        for q, (a, b, _, _) in enumerate(ranges):
            lo, hi = min(E, a * L), min(E, b * L)
            if hi > lo:
                run = y[o, lo:hi].clone()
                dist.broadcast(run, src=q)
                y[o, lo:hi] = run
    result_q.put((rank, y.numpy(), None))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_chunks", [4, 3])
def test_two_rank_dim1_chunks_equal_single_rank(n_chunks):
    """SURVEY §8(e) AlphaFold: chunks along dim 1 exchanged per outer index."""
    pytest.importorskip("paper_2401_10652_b200.api")
    world = 2
    port = 29700 + n_chunks + (os.getpid() % 1000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_dim1, args=(r, world, port, n_chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = _tri_row_graph()
    vals = {t: s.value for t, s in synth.make_inputs(g.input_specs(), 5).items()}
    with ops.exact_order():
        ref = executor.run(g, vals)["o"]
    for rank, y, _ in res:
        assert np.array_equal(y, ref), rank
