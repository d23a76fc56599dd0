#!/bin/bash
# A/B timing of env variants of one bench config, interleaved.  Usage: scripts/ab.sh CONFIG REPS "ENV_A" "ENV_B" ...
cfg=$1; reps=$2; shift 2
for r in $(seq $reps); do
  i=0
  for v in "$@"; do
    ms=$(env $v timeout 300 python bench.py --config $cfg --steps 20 --warmup 3 --no-unchunked --no-e2e --no-cpu 2>/dev/null | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')
    echo "$i [$v] $ms"
    i=$((i+1))
  done
done
