#!/bin/bash
# On the GPU box: launch list + ncu --set full of the top kernels of one bench step.
# Usage: scripts/profile.sh TAG [config]
set -x
TAG=$1; CFG=${2:-gpt}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --profile --config $CFG --steps 2 --warmup 1 > gpurun_out/launches_${TAG}.log 2>&1
for K in softmax gemm_tc layernorm; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 2 \
      -o gpurun_out/prof_${TAG}_${K} python bench.py --profile --config $CFG --steps 1 --warmup 1 > gpurun_out/prof_${TAG}_${K}.log 2>&1
done
ls -la gpurun_out
