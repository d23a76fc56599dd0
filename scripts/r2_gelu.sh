#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -k "gelu or epilogue or gpt or tiny" > gpurun_out/r2_gelu_t.log 2>&1; echo "rc=$?" >> gpurun_out/r2_gelu_t.log
timeout 300 python scripts/gemm_bench.py ffn1 > /dev/null 2>&1
timeout 300 python scripts/gemm_bench.py > gpurun_out/r2_gelu_gb.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2_gelu_b.json 2>/dev/null
tail -2 gpurun_out/r2_gelu_t.log
