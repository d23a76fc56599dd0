"""The N>1 path on CPU (gloo, world sizes 2 and 4): every rank asks libautochunk for its
schedule (ac_plan_rank_chunks: its chunks of every region; ac_plan_rank_schedule: the
nodes it runs on its rows only and the exchanges), executes exactly that with the
oracle's node maths (tests/rank_replay.py) and the exchanges as gloo collectives.
Every rank's outputs must equal the unchunked single-process output bitwise (fp64,
exact reduction order) - chunks are independent (Eq. 4)."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import executor, graph as og_graph, ops, select, workloads
import synth

CASES = {
    # causal GPT-like block, attention region: zigzag ownership, post-region rows
    "gpt": (lambda: workloads.transformer(96, 32, 2, 64, True, "f64", name="mr_gpt"),
            [("scores", "pv", 4, (0,))]),
    # non-causal attention-only block (UNet): round-robin ownership
    "unet": (lambda: workloads.transformer(64, 32, 2, 0, False, "f64", attn_only=True, name="mr_unet"),
             [("scores", "pv", 4, (0,))]),
    # whole transformer block as the region (forced whole-block plan, K/V hoisted)
    "gpt_block": (lambda: workloads.transformer(96, 32, 2, 64, True, "f64", name="mr_blk"),
                  [("proj_q", "ffn2", 4, (0,))]),
    # extent not divisible into whole groups: contiguous shares, owner broadcasts
    "ragged": (lambda: workloads.transformer(90, 32, 2, 64, False, "f64", name="mr_rag"),
               [("scores", "pv", 3, (0,))]),
    # Evoformer pair stack: row attention along i, column attention along j (chunk dim
    # not outermost: packed all-gathers), partitions handed across nodes
    "evo": (lambda: workloads.evoformer_pair(16, 8, 2, 4, "f64", name="mr_evo", cm=8, nf=2),
            [("row_scores", "row_pv", 4, (0,)), ("col_scores", "col_pv", 4, (1,))]),
}


def _plan(name):
    mk, spec = CASES[name]
    g = mk()
    text = "autochunk-plan 1\n" + "".join(
        f"region s={s} e={e} n={n} dims={','.join(map(str, d))}\n" for s, e, n, d in spec)
    return g, spec, text


def _worker(rank, world, port, name, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2401_10652_b200 import api
        from rank_replay import run_rank
        g, spec, text = _plan(name)
        cplan = api.plan_parse(api.graph_parse(og_graph.serialize(g)), text)
        regions = select.user_plan(g, spec).regions
        vals = {t: s.value for t, s in synth.make_inputs(g.input_specs(), 3).items()}
        with ops.exact_order():
            outs, log = run_rank(g, vals, regions, cplan, rank, world)
        result_q.put((rank, outs, log, None))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        result_q.put((rank, None, None, traceback.format_exc()))
    dist.destroy_process_group()


def _spawn(name, world):
    port = 29500 + (hash((name, world)) % 2000) + (os.getpid() % 1000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for _, _, _, err in res:
        assert err is None, err
    for p in procs:
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name", list(CASES))
def test_rank_schedule_replay_equals_single_rank(name, world):
    pytest.importorskip("paper_2401_10652_b200.api")
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    res = _spawn(name, world)
    g, _, _ = _plan(name)
    vals = {t: s.value for t, s in synth.make_inputs(g.input_specs(), 3).items()}
    with ops.exact_order():
        ref = executor.run(g, vals)
    logs = [r[2] for r in res]
    assert all(lg == logs[0] for lg in logs)          # every rank issues the same collectives
    for rank, outs, _, _ in res:
        for o in g.outputs:
            assert np.array_equal(outs[o], ref[o]), (name, world, rank, o)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_chunk_shares_partition_the_range(world):
    """Every chunk is owned by exactly one rank; causal regions are zigzag-balanced."""
    from paper_2401_10652_b200 import api
    for name in CASES:
        g, _, text = _plan(name)
        cplan = api.plan_parse(api.graph_parse(og_graph.serialize(g)), text)
        for k in range(cplan.num_regions):
            shares = [cplan.rank_chunks(k, r, world) for r in range(world)]
            n_eff, L, E = shares[0][1:]
            allc = sorted(c for s in shares for c in s[0])
            assert allc == [c for c in range(n_eff) if c * L < E], (name, k)
    # GPT configs[1] on 8 ranks: n = 8 refined to 16 zigzag chunks, equal causal work
    cg = api.graph_block("transformer", 16384, 1024, 16, 4096, True, "bf16", name="gpt")
    plan = api.plan_parse(cg, "autochunk-plan 1\nregion s=scores e=pv n=8 dims=0\n")
    work = []
    for r in range(8):
        chunks, n_eff, L, E = plan.rank_chunks(0, r, 8)
        assert n_eff == 16 and L == 1024
        work.append(sum(sum(i + 1 for i in range(c * L, (c + 1) * L)) for c in chunks))
    assert max(work) == min(work)


def test_gpt_schedule_partitions_rows_beyond_the_region():
    """GPT block at W = 8: Q projection, out-projection, LN2, FFN1, FFN2 run on the
    rank's rows only (LN1, K and V stay replicated); the block output is gathered once
    at the end with in-place all-gathers (one per zigzag half)."""
    from paper_2401_10652_b200 import api
    cg = api.graph_block("transformer", 16384, 1024, 16, 4096, True, "bf16", name="gpt")
    plan = api.plan_parse(cg, "autochunk-plan 1\nregion s=scores e=pv n=8 dims=0\n")
    ids = [n.id for n in workloads.transformer(16384, 1024, 16, 4096, True, "bf16", name="gpt").nodes]
    nr, nd, xops = plan.rank_schedule(3, 8)
    part = {ids[i] for i in range(len(ids)) if nr[i] >= 0}
    assert part == {"proj_q", "proj_o", "ln2", "ffn1", "ffn2"}, part
    assert [(o["kind"], o["tensor"], o["before_node"]) for o in xops] == [(0, "y", len(ids)), (1, "y", len(ids))]
