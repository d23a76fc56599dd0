"""Summarise AC_TRACE per-unit PV timelines (trace_NNN.txt: unit cta t_load0 t_tfull t_done, ns):
per launch the span, SM busy fraction and the tail after the first CTA runs dry."""
import glob
import sys

for fn in sorted(glob.glob(sys.argv[1] + "/trace_*.txt")):
    rows = [list(map(int, l.split())) for l in open(fn) if l.strip()]
    rows = [r for r in rows if r[2] > 0 and r[4] > 0]
    if not rows:
        continue
    t0 = min(r[2] for r in rows)
    t1 = max(r[4] for r in rows)
    per_cta = {}
    for u, cta, a, b, c in rows:
        lo, hi, busy = per_cta.get(cta, (a, c, 0))
        per_cta[cta] = (min(lo, a), max(hi, c), busy + (c - a))
    last_end = sorted(v[1] for v in per_cta.values())
    busy = sum(v[2] for v in per_cta.values())
    span = t1 - t0
    dur = sorted(r[4] - r[2] for r in rows)
    print(f"{fn.split('/')[-1]}: units {len(rows)} ctas {len(per_cta)} span {span/1e3:8.1f} us  busy {busy / (148 * span):5.1%}"
          f"  first CTA done at {(last_end[0]-t0)/1e3:7.1f} us  unit us min/med/max {dur[0]/1e3:.1f}/{dur[len(dur)//2]/1e3:.1f}/{dur[-1]/1e3:.1f}")
