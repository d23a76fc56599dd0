#!/bin/bash
# Copy the outputs of scripts/profile_r1b.sh (gpurun_out/r1b_*) into profiles/ (round 1).
set -e
cd "$(dirname "$0")/.."
cat gpurun_out/r1b_bench_{gpt,unet,vit,af,gpt_fa}.json gpurun_out/r1b_bench_unet_sweep.json \
    gpurun_out/r1b_ablation_gpt.json gpurun_out/r1b_bench_gpt_l4.json gpurun_out/r1b_maxlen_gpt.json \
    gpurun_out/r1b_reference.json | grep "^{" > profiles/r1_bench_lines.jsonl
for c in gpt unet af gpt_fa; do
  cp gpurun_out/r1b_launches_$c.csv profiles/r1_${c}_launches.csv
  python scripts/launches.py gpurun_out/r1b_launches_$c.csv > profiles/r1_${c}_launches.txt
  cp gpurun_out/r1b_traffic_$c.csv profiles/r1_${c}_traffic.csv
  python scripts/traffic_json.py gpurun_out/r1b_traffic_$c.csv $c > /dev/null
done
for f in gpt_attn gpt_ffn1 af_attn gpt_fa_attn; do
  python scripts/ncu_summary.py gpurun_out/r1b_full_$f.ncu-rep > profiles/r1_full_${f}_ncu.txt 2>&1
  echo "== stall sampling (top SASS)" >> profiles/r1_full_${f}_ncu.txt
  python scripts/ncu_hot.py gpurun_out/r1b_full_$f.ncu-rep 12 >> profiles/r1_full_${f}_ncu.txt 2>&1
done
wc -l profiles/r1_bench_lines.jsonl
