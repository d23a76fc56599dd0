#!/bin/bash
# On the GPU box: the report rows of SURVEY §8(d)/(f) - ablations (GPT forced region, AF),
# the forced whole-block GPT plan at full size, chunk sweeps, max-length runs (1D + 2D).
mkdir -p gpurun_out
B="timeout 900 python bench.py --steps 10 --warmup 3"
$B --ablation > gpurun_out/r2_ablation_gpt.json 2> gpurun_out/r2_ablation_gpt.err
$B --config af --ablation --no-e2e > gpurun_out/r2_ablation_af.json 2> gpurun_out/r2_ablation_af.err
$B --plan "$(printf 'autochunk-plan 1\nregion s=proj_q e=ffn2 n=8 dims=0\n')" > gpurun_out/r2_bench_gpt_block.json 2> gpurun_out/r2_bench_gpt_block.err
$B --sweep --no-e2e > gpurun_out/r2_sweep_gpt.json 2> gpurun_out/r2_sweep_gpt.err
$B --config unet --sweep --no-e2e > gpurun_out/r2_sweep_unet.json 2> gpurun_out/r2_sweep_unet.err
$B --config af --sweep --no-e2e > gpurun_out/r2_sweep_af.json 2> gpurun_out/r2_sweep_af.err
$B --config vit --sweep --no-e2e --steps 4 > gpurun_out/r2_sweep_vit.json 2> gpurun_out/r2_sweep_vit.err
for C in gpt af unet vit; do
  timeout 1200 python bench.py --maxlen --config $C > gpurun_out/r2_maxlen_$C.json 2> gpurun_out/r2_maxlen_$C.err
done
ls -la gpurun_out
