#!/bin/bash
# chunked / unchunked ms and speed loss for env variants, interleaved.  Usage: scripts/ab_loss.sh CONFIG REPS "ENV_A" ...
cfg=$1; reps=$2; shift 2
for r in $(seq $reps); do
  i=0
  for v in "$@"; do
    env $v timeout 300 python bench.py --config $cfg --steps 20 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c '
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); u=d.get("unchunked") or {}
print(d["ms_per_step"], u.get("ms_per_step"), u.get("speed_loss"), (d.get("stages") or {}).get("pv",{}).get("ms_per_step"))' | sed "s/^/$i [$v] /"
    i=$((i+1))
  done
done
