#!/bin/bash
# Round-1 refresh on the GPU box: bench lines of every config, launch lists, DRAM
# traffic per kernel, ncu --set full of the dominant kernels.  Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
for C in gpt unet vit af gpt_fa; do
  timeout 600 python bench.py --config $C > gpurun_out/r1b_bench_$C.json 2> gpurun_out/r1b_bench_$C.err
done
timeout 600 python bench.py --config unet --sweep --no-cpu --no-e2e > gpurun_out/r1b_bench_unet_sweep.json 2>> gpurun_out/r1b_bench_unet.err
timeout 600 python bench.py --config gpt --ablation --no-cpu --no-e2e --no-unchunked > gpurun_out/r1b_ablation_gpt.json 2> gpurun_out/r1b_ablation.err
timeout 600 python bench.py --config gpt --layers 4 --no-cpu --no-e2e > gpurun_out/r1b_bench_gpt_l4.json 2> gpurun_out/r1b_l4.err
timeout 900 python bench.py --config gpt --maxlen > gpurun_out/r1b_maxlen_gpt.json 2> gpurun_out/r1b_maxlen.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r1b_reference.json 2> gpurun_out/r1b_reference.err
for C in gpt unet af gpt_fa; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/r1b_launches_${C}.csv python scripts/node_run.py $C > /dev/null 2>&1
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:"gemm_tc|stats_combine|attn_fused" --csv --log-file gpurun_out/r1b_traffic_${C}.csv \
      python scripts/node_run.py $C > /dev/null 2>&1
done
# full captures (index among gemm_tc launches of one step): GPT scores / PV of chunk 5 (13 / 14),
# GPT FFN1 (20), AF row scores of chunk 3 (11); fused attention chunk 8 of gpt_fa
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 13 -c 2 \
    -o gpurun_out/r1b_full_gpt_attn python scripts/node_run.py gpt > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 20 -c 1 \
    -o gpurun_out/r1b_full_gpt_ffn1 python scripts/node_run.py gpt > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 11 -c 2 \
    -o gpurun_out/r1b_full_af_attn python scripts/node_run.py af > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fused -s 8 -c 1 \
    -o gpurun_out/r1b_full_gpt_fa_attn python scripts/node_run.py gpt_fa > /dev/null 2>&1
ls -la gpurun_out | tail -40
