#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "fused or fa or tiny or gpt" > gpurun_out/r2_fa3_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2_fa3_parity.log
B="timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e"
$B --config gpt_fa > gpurun_out/r2_fa3_bench.json 2> gpurun_out/r2_fa3_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fused -c 1 \
    -o gpurun_out/r2_full_fa3_attn python bench.py --profile --config gpt_fa --plan "$(printf 'autochunk-plan 1\n')" --steps 1 --warmup 1 > gpurun_out/r2_full_fa3_attn.log 2>&1
timeout 300 python scripts/dbg_evo_inv.py > gpurun_out/r2_dbg_evo.log 2>&1
tail -3 gpurun_out/r2_fa3_parity.log
