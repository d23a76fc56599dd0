#!/bin/bash
# f1 regime: planner plan (raw features) vs normalised features, both pipelined
mkdir -p gpurun_out
: > gpurun_out/norm.txt
for rep in 1 2; do
for a in "" "--normalize"; do
  timeout 300 python bench.py --config gpt_fa $a --steps 20 --warmup 5 --no-cpu > gpurun_out/norm.json 2>gpurun_out/norm_err.txt
  python - <<PY >> gpurun_out/norm.txt
import json
d=json.loads(open("gpurun_out/norm.json").read())
u=d.get("unchunked") or {}
print("rep$rep '$a'", d["ms_per_step"], "loss", u.get("speed_loss"), "plan", d["config"]["plan"], "pipelined", d["config"].get("pipelined_chunks"),
      "peak", json.dumps(d["peak_activation_bytes"])[:400], "e2e", d["e2e"]["value"])
PY
cp gpurun_out/norm.json gpurun_out/norm_rep${rep}_${a:-raw}.json
done; done
cat gpurun_out/norm.txt
