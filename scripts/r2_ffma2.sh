#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -x > gpurun_out/r2_ffma2_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2_ffma2_parity.log
: > gpurun_out/r2_ffma2.txt
for c in gpt gpt gpt_fa unet; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2_ffma2_b.json 2>/dev/null
  python - <<PY >> gpurun_out/r2_ffma2.txt
import json
d=json.loads(open("gpurun_out/r2_ffma2_b.json").read())
st={k:v["ms_per_step"] for k,v in d["stages"].items() if isinstance(v,dict)}
print("$c", d["ms_per_step"], round(d["unchunked"]["ms_per_step"],4), round(d["unchunked"]["speed_loss"],4), {k:st[k] for k in list(st)[:3]}, {k:d["unchunked"]["stages_ms"][k] for k in list(d["unchunked"]["stages_ms"])[:3]})
PY
done
tail -2 gpurun_out/r2_ffma2_parity.log; cat gpurun_out/r2_ffma2.txt
