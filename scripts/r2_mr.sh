#!/bin/bash
# On the GPU box: multi-rank emulation tests, full GPU suite, bench line with the new fields.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q > gpurun_out/r2_mr_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2_mr_pytest.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu2.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest_gpu2.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_gpt2.json 2> gpurun_out/r2_bench_gpt2.err
timeout 300 python bench.py --gpus 2 > gpurun_out/r2_bench_gpus2.json 2> gpurun_out/r2_bench_gpus2.err
tail -3 gpurun_out/r2_mr_pytest.log gpurun_out/r2_pytest_gpu2.log
