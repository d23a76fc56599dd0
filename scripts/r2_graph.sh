#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/r2_graph.txt
for c in tiny gpt unet af gpt_fa; do
  for g in "" "--no-graph"; do
    timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e $g > gpurun_out/r2_graph_b.json 2>gpurun_out/r2_graph_b.err
    python - <<PY >> gpurun_out/r2_graph.txt
import json
d=json.loads(open("gpurun_out/r2_graph_b.json").read())
print("$c", "$g" or "graph", d["ms_per_step"], round(d["unchunked"]["ms_per_step"],4), round(d["unchunked"]["speed_loss"],4), d["config"]["launch"][:12])
PY
  done
done
cat gpurun_out/r2_graph.txt
