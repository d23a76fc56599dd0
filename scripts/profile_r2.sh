#!/bin/bash
# Round-2 refresh on the GPU box: bench lines of every config, launch lists, DRAM traffic
# per kernel, ncu --set full of the dominant kernels.  Outputs in gpurun_out/r2p_*.
mkdir -p gpurun_out
for C in gpt unet vit af af_attn gpt_fa tiny; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 5 > gpurun_out/r2p_bench_$C.json 2> gpurun_out/r2p_bench_$C.err
done
timeout 600 python bench.py --config gpt --layers 4 --no-cpu --no-e2e > gpurun_out/r2p_bench_gpt_l4.json 2> gpurun_out/r2p_l4.err
timeout 600 python bench.py --config gpt_fa --normalize --steps 20 --warmup 5 > gpurun_out/r2p_bench_gpt_fa_norm.json 2> gpurun_out/r2p_fa_norm.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2p_reference.json 2> gpurun_out/r2p_reference.err
for C in gpt unet af gpt_fa; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/r2p_launches_${C}.csv python scripts/node_run.py $C > /dev/null 2>&1
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:"gemm_tc|attn_fused" --csv --log-file gpurun_out/r2p_traffic_${C}.csv \
      python scripts/node_run.py $C > /dev/null 2>&1
done
# full captures (index among gemm_tc launches of one step): GPT scores / PV of chunk 5 (13 / 14),
# GPT FFN1 (20), AF row scores + PV of chunk 3; fused attention unchunked and a row chunk
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 13 -c 2 \
    -o gpurun_out/r2p_full_gpt_attn python scripts/node_run.py gpt > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 20 -c 1 \
    -o gpurun_out/r2p_full_gpt_ffn1 python scripts/node_run.py gpt > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fused -c 1 \
    -o gpurun_out/r2p_full_gpt_fa_attn python scripts/node_run.py gpt_fa unchunked > /dev/null 2>&1
ls -la gpurun_out | grep r2p_ | tail -60
