#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -x -k "fused or fa" > gpurun_out/r2_fa5_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2_fa5_parity.log
for rep in 1 2; do
  timeout 120 python bench.py --config gpt_fa --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_fa5_bench.json 2> gpurun_out/r2_fa5_bench.err
  python - <<PY >> gpurun_out/r2_fa5.txt
import json
d=json.loads(open("gpurun_out/r2_fa5_bench.json").read())
print("$rep", "step", d["ms_per_step"], "attn_chunked", d["stages"]["attn"]["ms_per_step"], "attn_unchunked", d["unchunked"]["stages_ms"]["attn"], "unch_step", round(d["unchunked"]["ms_per_step"],4), "err", (d.get("error_vs_oracle") or {}).get("normwise_rel"))
PY
done
tail -2 gpurun_out/r2_fa5_parity.log; cat gpurun_out/r2_fa5.txt
