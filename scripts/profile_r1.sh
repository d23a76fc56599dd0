#!/bin/bash
# On the GPU box: launch lists + ncu --set full captures of the f2 attention kernels
# (GPT chunk 4: scores, combine, PV; UNet chunk 1 PV; AF row pair).  Reports land in gpurun_out/.
set -x
mkdir -p gpurun_out
for C in gpt unet af; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
      --log-file gpurun_out/launches_${C}.csv python bench.py --profile --config $C --steps 2 --warmup 1 \
      > gpurun_out/launches_${C}.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 11 -c 2 \
    -o gpurun_out/full_gpt_attn python bench.py --profile --config gpt --steps 1 --warmup 1 > gpurun_out/full_gpt_attn.log 2>&1
ncu --set full --clock-control none -k regex:stats_combine -s 4 -c 1 \
    -o gpurun_out/full_gpt_combine python bench.py --profile --config gpt --steps 1 --warmup 1 > gpurun_out/full_gpt_combine.log 2>&1
ncu --set full --clock-control none -k regex:gemm_tc -s 22 -c 3 \
    -o gpurun_out/full_gpt_ffn python bench.py --profile --config gpt --steps 1 --warmup 1 > gpurun_out/full_gpt_ffn.log 2>&1
ncu --set full --clock-control none -k regex:gemm_tc -s 5 -c 2 \
    -o gpurun_out/full_unet_attn python bench.py --profile --config unet --steps 1 --warmup 1 > gpurun_out/full_unet_attn.log 2>&1
ncu --set full --clock-control none -k regex:"gemm_tc|softmax" -s 8 -c 3 \
    -o gpurun_out/full_af_row python bench.py --profile --config af --steps 1 --warmup 1 > gpurun_out/full_af_row.log 2>&1
ls -la gpurun_out | tail -20
