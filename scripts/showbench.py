"""Summarise bench JSON lines: value, speed loss, per-stage chunked vs unchunked ms."""
import json
import sys

for fn in sys.argv[1:]:
    for ln in open(fn):
        if not ln.startswith("{"):
            continue
        d = json.loads(ln)
        u = d.get("unchunked") or {}
        r = d.get("roofline") or {}
        print(f"== {fn}: {d['value']:.4g} tok/s  {d['ms_per_step']:.3f} ms  unchunked {u.get('ms_per_step')}  "
              f"loss {u.get('speed_loss')}  roof {r.get('kernel')} {r.get('frac')}  e2e {(d.get('e2e') or {}).get('value')}"
              f"  clocks {d.get('clocks')}")
        us = u.get("stages_ms", {})
        for k, v in d.get("stages", {}).items():
            if not isinstance(v, dict):
                print(f"   {k} {v}")
                continue
            rf = (v.get("roofline") or {}).get("frac")
            print(f"   {k:14s} {v['ms_per_step']:8.4f}  unchunked {us.get(k, float('nan')):8.4f}  x{v['launches_per_step']:.0f}"
                  f"  roof {rf}")
