"""The multi-rank executor on ONE GPU: W ranks of an in-process communicator
(ac_comm_init_local), each driven by its own host thread, stream, workspace and
outputs, run their shares of the plan (ac_plan_rank_chunks / ac_plan_rank_schedule,
SURVEY §8(e)) through ac_run - the same kernels, partitioned launches, packed
staging and communication-stream overlap as with NCCL; only the transport is
emulated (device-to-device copies ordered by events).  Every rank's outputs must
equal the single-rank run bitwise, and the run must issue exactly the schedule's
exchanges."""
import threading

import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import workloads  # noqa: E402

CASES = {
    "gpt": (lambda: workloads.transformer(1024, 256, 4, 512, True, "bf16", name="mg_gpt"),
            "region s=scores e=pv n=4 dims=0\n"),
    "unet": (lambda: workloads.transformer(1024, 256, 4, 0, False, "bf16", attn_only=True, name="mg_unet"),
             "region s=scores e=pv n=4 dims=0\n"),
    "gpt_block": (lambda: workloads.transformer(1024, 256, 4, 512, True, "bf16", name="mg_blk"),
                  "region s=proj_q e=ffn2 n=4 dims=0\n"),
    "evo": (lambda: workloads.evoformer_pair(128, 64, 2, 32, "bf16", name="mg_evo", cm=64, nf=2),
            "region s=row_scores e=row_pv n=4 dims=0\nregion s=col_scores e=col_pv n=4 dims=1\n"),
    # f1 region: chunks pipelined over two streams, region outputs gathered eagerly
    "gpt_fa": (lambda: workloads.block("transformer_fa", 2048, 256, 4, 1024, True, "bf16", name="mg_fa"),
               "region s=attn e=ffn2 n=8 dims=0\n"),
    "ragged": (lambda: workloads.transformer(896, 256, 4, 512, False, "bf16", name="mg_rag"),
               "region s=scores e=pv n=3 dims=0\n"),
}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name", list(CASES))
def test_local_ranks_equal_single_rank(name, world):
    import gpu_util as gu
    from paper_2401_10652_b200 import api
    mk, regions = CASES[name]
    og = mk()
    cg = gu.c_graph(og)
    plan = api.plan_parse(cg, "autochunk-plan 1\n" + regions)
    _, dev = gu.make_values(og, 0)
    ref, _ = gu.run(cg, plan, og, dev)
    torch.cuda.synchronize()
    comms = api.Comm.local(world)
    ins = {t: dev[t] for t in og.inputs + og.weights}
    outs, execs, errs, streams = [], [], [None] * world, []
    for r in range(world):
        ws = torch.empty(max(plan.workspace_bytes(r, world), 16), dtype=torch.uint8, device="cuda")
        outs.append({o: torch.full_like(ref[o], float("nan")) for o in og.outputs})
        execs.append(api.Exec(plan, ws, comms[r]))
        streams.append(torch.cuda.Stream())

    def work(r):
        try:
            for _ in range(2):          # twice: the exchange slots and events are reused
                execs[r].run(ins, outs[r], streams[r])
        except Exception as e:  # pragma: no cover
            errs[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    torch.cuda.synchronize()
    assert errs == [None] * world, errs
    for r in range(world):
        _, _, xops = plan.rank_schedule(r, world)
        assert execs[r].stats().exchanges == len(xops)
        assert execs[r].stats().chunks_run == sum(len(plan.rank_chunks(k, r, world)[0])
                                                  for k in range(plan.num_regions))
        for o in og.outputs:
            assert torch.equal(outs[r][o], ref[o]), (name, world, r, o)


def test_nccl_communicator_world1():
    """The NCCL binding itself on this one-GPU box: unique id, ncclCommInitRank, the
    rank-reversed ncclCommSplit, ncclCommGetAsyncError (ac_comm_check) and an ac_run
    through a world-1 communicator (no exchanges) equal to the run without one."""
    import gpu_util as gu
    from paper_2401_10652_b200 import api
    og = workloads.transformer(512, 256, 4, 512, True, "bf16", name="nccl1")
    cg = gu.c_graph(og)
    plan = api.plan_parse(cg, "autochunk-plan 1\nregion s=scores e=pv n=4 dims=0\n")
    _, dev = gu.make_values(og, 0)
    ref, _ = gu.run(cg, plan, og, dev)
    comm = api.Comm(api.Comm.unique_id(), 0, 1, torch.cuda.current_device())
    comm.check()
    ws = torch.empty(plan.workspace_bytes(0, 1), dtype=torch.uint8, device="cuda")
    outs = {o: torch.empty_like(ref[o]) for o in og.outputs}
    ex = api.Exec(plan, ws, comm)
    ex.run({t: dev[t] for t in og.inputs + og.weights}, outs)
    torch.cuda.synchronize()
    comm.check()
    assert ex.stats().exchanges == 0
    for o in og.outputs:
        assert torch.equal(outs[o], ref[o])
