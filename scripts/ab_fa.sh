#!/bin/bash
# A/B of fused-attention variants (scratch_libs/lib_<v>.so): attention stage time unchunked
# and in the f1 plan, interleaved twice.
mkdir -p gpurun_out
: > gpurun_out/ab_fa.txt
for rep in 1 2; do
for v in base poly3 poly1 intpack both; do
  AC_LIB_PATH=scratch_libs/lib_$v.so timeout 300 python bench.py --config gpt_fa --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_fa_$v.json 2>/dev/null
  python - <<PY >> gpurun_out/ab_fa.txt
import json
d=json.loads(open("gpurun_out/ab_fa_$v.json").read())
print("$rep $v", "step", d["ms_per_step"], "attn_chunked", d["stages"]["attn"]["ms_per_step"], "attn_unchunked", d["unchunked"]["stages_ms"]["attn"], "unch_step", round(d["unchunked"]["ms_per_step"],4))
PY
done; done
timeout 300 env AC_LIB_PATH=scratch_libs/lib_both.so python -m pytest tests/test_gpu_parity.py -q -k "fused or fa" >> gpurun_out/ab_fa.txt 2>&1
cat gpurun_out/ab_fa.txt
