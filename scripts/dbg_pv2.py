"""Chunked vs unchunked bitwise check of the fused PV under env variants (debug)."""
import os, sys, itertools
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import gpu_util as gu
from oracle import workloads
from paper_2401_10652_b200 import api

for ov, causal, n in itertools.product(["0", "1"], [True, False], [3, 4]):
    os.environ["AC_OVERLAP_CAUSAL"] = ov
    os.environ["AC_OVERLAP"] = ov
    os.environ["AC_PV_SPLITK"] = "0"
    og = workloads.block("attn_only", 2048 + 320, 256, 4, 0, causal, "bf16", name="pv_split")
    cg = gu.c_graph(og)
    vals, dev = gu.make_values(og, 5)
    base, _ = gu.run(cg, gu.empty_plan(cg), og, dev)
    got, _ = gu.run(cg, api.plan_parse(cg, f"autochunk-plan 1\nregion s=scores e=pv n={n} dims=0\n"), og, dev)
    torch.cuda.synchronize()
    a, b = got["x1"].float(), base["x1"].float()
    bad = (a != b).any(dim=1).nonzero().flatten().tolist()
    print(f"ov={ov} causal={causal} n={n}: bad rows {len(bad)} first {bad[:10]} maxdiff {(a-b).abs().max().item():.3g}")
    # repeat the chunked run: deterministic?
    got2, _ = gu.run(cg, api.plan_parse(cg, f"autochunk-plan 1\nregion s=scores e=pv n={n} dims=0\n"), og, dev)
    base2, _ = gu.run(cg, gu.empty_plan(cg), og, dev)
    torch.cuda.synchronize()
    print("   chunked rerun equal:", torch.equal(got2["x1"], got["x1"]), " unchunked rerun equal:", torch.equal(base2["x1"], base["x1"]))
