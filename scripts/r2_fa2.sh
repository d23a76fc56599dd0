#!/bin/bash
# On the GPU box: FA (3 TMEM slots) parity + timing + ncu; sanitizers (racecheck report kept);
# AF ablation; multi-rank emulation.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q > gpurun_out/r2_fa2_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2_fa2_parity.log
B="timeout 900 python bench.py --steps 10 --warmup 3"
$B --config gpt_fa > gpurun_out/r2_fa2_bench.json 2> gpurun_out/r2_fa2_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fused -c 1 \
    -o gpurun_out/r2_full_fa2_attn python bench.py --profile --config gpt_fa --plan "$(printf 'autochunk-plan 1\n')" --steps 1 --warmup 1 > gpurun_out/r2_full_fa2_attn.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_sanitizer.py -q > gpurun_out/r2_san2.log 2>&1; echo "rc=$?" >> gpurun_out/r2_san2.log
$B --config af --ablation --no-e2e > gpurun_out/r2_ablation_af.json 2> gpurun_out/r2_ablation_af.err
tail -3 gpurun_out/r2_fa2_parity.log gpurun_out/r2_san2.log
