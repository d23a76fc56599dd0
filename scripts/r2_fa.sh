#!/bin/bash
# On the GPU box: the FA4-style fused attention (parity, timing, ncu), new linear layouts,
# sanitizers, AF ablation, max-length capacity runs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2_fa_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2_fa_parity.log
B="timeout 900 python bench.py --steps 10 --warmup 3"
$B --config gpt_fa > gpurun_out/r2_fa_bench.json 2> gpurun_out/r2_fa_bench.err
$B --config gpt_fa --plan "$(printf 'autochunk-plan 1\nregion s=ln2 e=ffn2 n=2 dims=0\n')" --no-cpu > gpurun_out/r2_fa_bench_ffn.json 2> gpurun_out/r2_fa_bench_ffn.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fused -c 1 \
    -o gpurun_out/r2_full_fa_attn python bench.py --profile --config gpt_fa --plan "$(printf 'autochunk-plan 1\n')" --steps 1 --warmup 1 > gpurun_out/r2_full_fa_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fused -c 1 \
    -o gpurun_out/r2_full_fa_chunk python bench.py --profile --config gpt_fa --steps 1 --warmup 1 > gpurun_out/r2_full_fa_chunk.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_sanitizer.py -x -q > gpurun_out/r2_san.log 2>&1; echo "rc=$?" >> gpurun_out/r2_san.log
$B --config af --ablation --no-e2e > gpurun_out/r2_ablation_af.json 2> gpurun_out/r2_ablation_af.err
for C in gpt af unet vit; do
  timeout 1200 python bench.py --maxlen --config $C > gpurun_out/r2_maxlen_$C.json 2> gpurun_out/r2_maxlen_$C.err
done
tail -3 gpurun_out/r2_fa_parity.log gpurun_out/r2_san.log
