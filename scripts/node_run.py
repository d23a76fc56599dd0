"""Exactly one ac_run of a bench config (for ncu captures: every kernel of one
step, nothing else of ours).  Usage: python scripts/node_run.py CONFIG [unchunked | n=N]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2401_10652_b200 import api  # noqa: E402

cfg = sys.argv[1]
cg, doc = bench.c_graph(cfg)
prof0, _ = api.estimate_memory(cg)
budget = int(bench.DEFAULT_BUDGET.get(cfg, 0.2) * prof0.peak_bytes)
if len(sys.argv) > 2 and sys.argv[2] == "unchunked":
    plan = api.plan_parse(cg, "autochunk-plan 1\n")
elif len(sys.argv) > 2 and sys.argv[2].startswith("n="):  # forced region chunk count
    plan = api.plan_parse(cg, f"autochunk-plan 1\nregion s=scores e=pv {sys.argv[2]} dims=0\n")
elif cfg == "tiny":
    plan = api.plan_parse(cg, "autochunk-plan 1\nregion s=scores e=pv n=8 dims=0\n")
else:
    plan = api.ac_plan(cg, budget)
_, dev = bench.device_inputs(doc, torch)
TD = {"bf16": torch.bfloat16, "f32": torch.float32}
outs = {o: torch.empty(doc.tensors[o][1], dtype=TD[doc.tensors[o][0]], device="cuda") for o in doc.outputs}
ws = torch.empty(max(plan.workspace_bytes(), 16), dtype=torch.uint8, device="cuda")
ex = api.Exec(plan, ws)
ex.run({t: dev[t] for t in doc.order}, outs)
torch.cuda.synchronize()
print("launches", ex.stats().launches)
