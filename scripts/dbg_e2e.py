"""Debug: bench-style exec of a config; rebind the input to fresh buffers."""
import sys
import torch
sys.path[:0] = ["."]
import bench
from paper_2401_10652_b200 import api

cfg = sys.argv[1]
cg, doc = bench.c_graph(cfg)
prof0, _ = api.estimate_memory(cg)
plan = api.ac_plan(cg, int(0.2 * prof0.peak_bytes))
samples, dev = bench.device_inputs(doc, torch)
ws = torch.empty(max(plan.workspace_bytes(), 16), dtype=torch.uint8, device="cuda")
outs = {o: torch.empty(doc.tensors[o][1], dtype=torch.bfloat16, device="cuda") for o in doc.outputs}
ins = {t: dev[t] for t in doc.order}
ex = api.Exec(plan, ws)
def go(tag, inputs):
    try:
        ex.run(inputs, outs)
        torch.cuda.synchronize()
        print(tag, "ok", {o: float(v.float().abs().max()) for o, v in outs.items()}, flush=True)
    except Exception as e:
        print(tag, "FAIL", e, flush=True)
        sys.exit(1)
go("base", ins)
go("base2", ins)
xin = doc.inputs[0]
dx = dev[xin].clone()
i2 = dict(ins); i2[xin] = dx
go("clone", i2)
hx = dev[xin].cpu().pin_memory()
dx2 = torch.empty_like(dev[xin]); dx2.copy_(hx, non_blocking=True)
i3 = dict(ins); i3[xin] = dx2
go("pinned", i3)
print(ws.data_ptr() % 4096, dx.data_ptr() % 4096, dx2.data_ptr() % 4096, ws.numel())
