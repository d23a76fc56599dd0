"""Which split-chain region of the Evoformer triangle attention breaks chunked == unchunked
(unfused path)?"""
import os, sys
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
os.environ["AC_FUSE_SOFTMAX"] = "0"
import torch
import gpu_util as gu
from oracle import workloads
from paper_2401_10652_b200 import api
og = workloads.evoformer_pair(64, 128, 4, 32, "bf16", name="evo_small")
cg = gu.c_graph(og)
_, dev = gu.make_values(og, 9)
base, _ = gu.run(cg, gu.empty_plan(cg), og, dev)
torch.cuda.synchronize()
for txt in ["region s=row_scores e=row_scores n=64 dims=0", "region s=row_softmax e=row_softmax n=64 dims=0",
            "region s=row_pv e=row_pv n=64 dims=0", "region s=row_scores e=row_scores n=2 dims=0",
            "region s=row_pv e=row_pv n=2 dims=0", "region s=row_pv e=row_pv n=32 dims=0",
            "region s=row_scores e=row_pv n=64 dims=0", "region s=row_scores e=row_pv n=4 dims=0"]:
    got, _ = gu.run(cg, api.plan_parse(cg, "autochunk-plan 1\n" + txt + "\n"), og, dev)
    torch.cuda.synchronize()
    o = og.outputs[0]
    d = (got[o].float() - base[o].float()).abs()
    print(f"{txt:50s} equal={torch.equal(got[o], base[o])} maxdiff={d.max().item():.3e} ndiff={(d > 0).sum().item()}")
