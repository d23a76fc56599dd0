#!/bin/bash
# Copy the outputs of scripts/profile_r2.sh (gpurun_out/r2p_*) into profiles/ (round 2).
set -e
cd "$(dirname "$0")/.."
for c in gpt unet vit af af_attn gpt_fa gpt_fa_norm tiny gpt_l4; do
  grep -h "^{" gpurun_out/r2p_bench_$c.json | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); d['_file']='r2p_bench_$c'; print(json.dumps(d))"
done > profiles/r2_refresh_lines.jsonl
grep -h "^{" gpurun_out/r2p_reference.json >> profiles/r2_refresh_lines.jsonl
for c in gpt unet af gpt_fa; do
  cp gpurun_out/r2p_launches_$c.csv profiles/r2_${c}_launches.csv
  python scripts/launches.py gpurun_out/r2p_launches_$c.csv > profiles/r2_${c}_launches.txt
  cp gpurun_out/r2p_traffic_$c.csv profiles/r2_${c}_traffic.csv
  python scripts/traffic_json.py gpurun_out/r2p_traffic_$c.csv $c > /dev/null
done
for f in gpt_attn gpt_ffn1 gpt_fa_attn; do
  python scripts/ncu_summary.py gpurun_out/r2p_full_$f.ncu-rep > profiles/r2_full_${f}_ncu.txt 2>&1
  echo "== stall sampling (top SASS)" >> profiles/r2_full_${f}_ncu.txt
  python scripts/ncu_hot.py gpurun_out/r2p_full_$f.ncu-rep 12 >> profiles/r2_full_${f}_ncu.txt 2>&1
done
wc -l profiles/r2_refresh_lines.jsonl
