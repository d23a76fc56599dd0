#!/bin/bash
# On the GPU box: GPU tests, smoke, the default bench line and the other configs' lines.
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/r2_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
timeout 600 python bench.py > gpurun_out/r2_bench_gpt.json 2> gpurun_out/r2_bench_gpt.err
for C in unet af af_attn vit tiny gpt_fa; do
  timeout 600 python bench.py --config $C --steps 10 --warmup 3 > gpurun_out/r2_bench_$C.json 2> gpurun_out/r2_bench_$C.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
      --log-file gpurun_out/r2_launches_gpt.csv python bench.py --profile --config gpt --steps 2 --warmup 1 > gpurun_out/r2_launches_gpt.log 2>&1
tail -3 gpurun_out/r2_pytest_gpu.log
