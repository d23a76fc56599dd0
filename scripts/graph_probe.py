"""Probe: one GPT step (ac_run) captured into a CUDA graph and replayed vs launched
directly; L2 flushed between steps in both (as in bench.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2401_10652_b200 import api  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "gpt"
cg, doc = bench.c_graph(cfg)
prof0, _ = api.estimate_memory(cg)
plan = api.ac_plan(cg, int(bench.DEFAULT_BUDGET.get(cfg, 0.2) * prof0.peak_bytes))
_, dev = bench.device_inputs(doc, torch)
TD = {"bf16": torch.bfloat16, "f32": torch.float32}
outs = {o: torch.empty(doc.tensors[o][1], dtype=TD[doc.tensors[o][0]], device="cuda") for o in doc.outputs}
ws = torch.empty(max(plan.workspace_bytes(), 16), dtype=torch.uint8, device="cuda")
ex = api.Exec(plan, ws)
ins = {t: dev[t] for t in doc.order}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        ex.run(ins, outs, stream=s)
s.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    ex.run(ins, outs, stream=s)
torch.cuda.synchronize()


def timed(fn, k=20):
    ts = []
    for _ in range(k):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


for rep in range(2):
    d = timed(lambda: ex.run(ins, outs))
    gg = timed(lambda: g.replay())
    print(f"{cfg}: direct {d:.4f} ms  graph {gg:.4f} ms")
ref = {o: outs[o].clone() for o in outs}
g.replay()
torch.cuda.synchronize()
print("graph output equal:", all(torch.equal(ref[o], outs[o]) for o in outs))
