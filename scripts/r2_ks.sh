#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or fa or degenerate" > gpurun_out/r2_ks_t.log 2>&1; echo "rc=$?" >> gpurun_out/r2_ks_t.log
: > gpurun_out/r2_ks.txt
for i in 1 2; do
  timeout 120 python bench.py --config gpt_fa --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_ks_b.json 2>/dev/null
  python - <<PY >> gpurun_out/r2_ks.txt
import json
d=json.loads(open("gpurun_out/r2_ks_b.json").read())
print("$i", "step", d["ms_per_step"], "attn_chunked", d["stages"]["attn"]["ms_per_step"], "attn_unchunked", d["unchunked"]["stages_ms"]["attn"], "unch_step", round(d["unchunked"]["ms_per_step"],4), d["roofline"]["frac"])
PY
done
tail -2 gpurun_out/r2_ks_t.log; cat gpurun_out/r2_ks.txt
