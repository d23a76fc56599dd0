#!/bin/bash
# chunk pipelining: GPU tests, then A/B against AC_PIPELINE=0 on the configs it touches
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q \
  -k "pipelining or fused_attention or af_ or whole_block or gpt_fa or gpt_block or evoformer or graph_capture or planned_peak or stacked" > gpurun_out/pipe_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pipe_pytest.log
: > gpurun_out/pipe_ab.txt
for C in gpt_fa gpt_fa_ffn gpt_block; do
case $C in
  gpt_fa) ARGS=(--config gpt_fa) ;;
  gpt_fa_ffn) ARGS=(--config gpt_fa --plan "region s=ln2 e=ffn2 n=2 dims=0") ;;
  gpt_block) ARGS=(--config gpt --plan "region s=proj_q e=ffn2 n=8 dims=0") ;;
esac
for rep in 1 2; do
for v in 1 0; do
  AC_PIPELINE=$v timeout 300 python bench.py "${ARGS[@]}" --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/pipe_${C}_${v}.json 2>gpurun_out/pipe_err.txt
  python - <<PY >> gpurun_out/pipe_ab.txt
import json
try:
    d=json.loads(open("gpurun_out/pipe_${C}_${v}.json").read())
    print("$C rep$rep pipe=$v", d["ms_per_step"], "unchunked", (d.get("unchunked") or {}).get("ms_per_step"), "plan", d["config"].get("plan"))
except Exception as e:
    print("$C $v failed", e, open("gpurun_out/pipe_err.txt").read()[-500:])
PY
done; done; done
cat gpurun_out/pipe_ab.txt
