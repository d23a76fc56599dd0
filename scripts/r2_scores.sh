#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gpt or fused or tiny or unet" > gpurun_out/r2_sc_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2_sc_parity.log
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2_sc_bench_$i.json 2> gpurun_out/r2_sc_bench_$i.err
done
tail -2 gpurun_out/r2_sc_parity.log
