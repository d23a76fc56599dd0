#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x > gpurun_out/r2_epi2_t.log 2>&1; echo "rc=$?" >> gpurun_out/r2_epi2_t.log
timeout 300 python scripts/gemm_bench.py ffn1 > /dev/null 2>&1
timeout 300 python scripts/gemm_bench.py > gpurun_out/r2_epi2_gb.txt 2>&1
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2_epi2_b$i.json 2>/dev/null; done
timeout 300 python bench.py --config af --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_epi2_af.json 2>/dev/null
tail -2 gpurun_out/r2_epi2_t.log
