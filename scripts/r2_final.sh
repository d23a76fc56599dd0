#!/bin/bash
# On the GPU box: the round-end checks the driver runs (GPU tests, smoke, default bench) plus
# the reference arm.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2f_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2f_reference.json 2> gpurun_out/r2f_reference.err
tail -n 3 gpurun_out/r2f_pytest_gpu.log; tail -n 3 gpurun_out/r2f_smoke.log
