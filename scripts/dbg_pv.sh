#!/bin/bash
# PV experiments: split-K on/off (dynamic unit scheduling)
for c in unet gpt; do for sk in 0 1; do
  r=$(AC_PV_SPLITK=$sk timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages']['pv']['ms_per_step'], d['unchunked']['speed_loss'])")
  echo "$c split=$sk step/pv/loss=$r"
done; done
