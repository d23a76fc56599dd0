"""Debug: run attn_only blocks chunked / unchunked and synchronise after each."""
import sys
import torch
sys.path[:0] = [".", "tests"]
import gpu_util as gu
from oracle import workloads, memory
from paper_2401_10652_b200 import api

for N in [int(a) for a in sys.argv[1:]]:
    og = workloads.block("attn_only", N, 640, 10, 0, False, "bf16", name="u")
    cg = gu.c_graph(og)
    vals, dev = gu.make_values(og, 0)
    for txt in ["autochunk-plan 1\nregion s=scores e=pv n=8 dims=0\n", "autochunk-plan 1\n"]:
        plan = api.plan_parse(cg, txt)
        try:
            got, ex = gu.run(cg, plan, og, dev)
            torch.cuda.synchronize()
            print(N, repr(txt[-30:]), "ok", {o: float(v.float().abs().max()) for o, v in got.items()}, flush=True)
        except Exception as e:
            print(N, repr(txt[-30:]), "FAIL", e, flush=True)
            sys.exit(1)
