#!/bin/bash
# ncu filtered by the executor's NVTX ranges: only chunk 3 of the GPT attention region
mkdir -p gpurun_out
ncu --nvtx --nvtx-include "ac_run/region 0 scores..pv n=8/chunk 3/" --metrics gpu__time_duration.sum \
    --clock-control none -c 8 --csv --log-file gpurun_out/nvtx_chunk3.csv \
    python bench.py --profile --no-graph --steps 1 --warmup 1 > gpurun_out/nvtx_bench.log 2>&1
echo "rc=$?" >> gpurun_out/nvtx_bench.log
ncu --nvtx --nvtx-include "regex:chunk 3/" --metrics gpu__time_duration.sum \
    --clock-control none -c 8 --csv --log-file gpurun_out/nvtx_chunk3_regex.csv \
    python bench.py --profile --no-graph --steps 1 --warmup 1 >> gpurun_out/nvtx_bench.log 2>&1
echo "rc=$?" >> gpurun_out/nvtx_bench.log
