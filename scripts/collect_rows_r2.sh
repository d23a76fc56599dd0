#!/bin/bash
# Copy the report rows of scripts/r2_rows.sh (gpurun_out/r2_*.json) into
# profiles/r2_bench_lines.jsonl (one line per file, tagged with its file name); the
# fused-attention FFN-region line of the earlier round-2 run is kept.
set -e
cd "$(dirname "$0")/.."
keep=$(grep '"_file": "r2_fa_bench_ffn"' profiles/r2_bench_lines.jsonl || true)
: > /tmp/rows.jsonl
for f in r2_ablation_gpt r2_ablation_af r2_bench_gpt_block r2_sweep_gpt r2_sweep_unet r2_sweep_af r2_sweep_vit \
         r2_maxlen_gpt r2_maxlen_af r2_maxlen_unet r2_maxlen_vit; do
  [ -f gpurun_out/$f.json ] || continue
  grep -h "^{" gpurun_out/$f.json | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); d['_file']='$f'; print(json.dumps(d))" >> /tmp/rows.jsonl
done
[ -n "$keep" ] && echo "$keep" >> /tmp/rows.jsonl
mv /tmp/rows.jsonl profiles/r2_bench_lines.jsonl
wc -l profiles/r2_bench_lines.jsonl
