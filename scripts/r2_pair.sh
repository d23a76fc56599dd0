#!/bin/bash
mkdir -p gpurun_out
timeout 100 python scripts/dbg_pair.py > gpurun_out/dbg_pair.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/r2_pair_test.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pair_test.log
timeout 600 python scripts/gemm_bench.py > gpurun_out/r2_pair_gemm_bench.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x > gpurun_out/r2_pair_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pair_parity.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2_pair_bench_gpt.json 2> gpurun_out/r2_pair_bench_gpt.err
tail -3 gpurun_out/r2_pair_test.log gpurun_out/r2_pair_parity.log
