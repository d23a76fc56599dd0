#!/bin/bash
# PV experiments on UNet (no split), grid capped at 16 CTAs: per-CTA streaming rate
for d in 0 1 3 7 4; do
  r=$(AC_PV_SPLITK=0 AC_DBG=$d AC_DBG_GRID=16 timeout 300 python bench.py --config unet --steps 3 --warmup 2 --no-e2e --no-unchunked 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['stages']['pv']['ms_per_step'])")
  echo "grid=16 dbg=$d pv_ms=$r"
done
