"""Summarise AC_TRACE per-unit PV timelines (trace_NNN.txt: unit cta t_load0 t_tfull t_done, ns):
per launch the span, the gap to the previous launch, SM busy fraction, the time until
the first CTA runs dry, the first-MMA latency and the unit durations."""
import glob
import sys

prev_end = None
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
    first_start = sorted(v[0] for v in per_cta.values())
    busy = sum(v[2] for v in per_cta.values())
    span = t1 - t0
    dur = sorted(r[4] - r[2] for r in rows)
    lat = sorted(r[3] - r[2] for r in rows if r[3] > 0)
    gap = (t0 - prev_end) / 1e3 if prev_end else float("nan")
    prev_end = t1
    print(f"{fn.split('/')[-1]}: units {len(rows):4d} ctas {len(per_cta)} span {span/1e3:7.1f} us gap {gap:6.1f} "
          f"busy {busy / (148 * span):5.1%} starts within {(first_start[-1]-t0)/1e3:5.1f} us "
          f"first dry {(last_end[0]-t0)/1e3:6.1f} us  unit us min/med/max {dur[0]/1e3:.1f}/{dur[len(dur)//2]/1e3:.1f}/"
          f"{dur[-1]/1e3:.1f}  first-MMA lat med {lat[len(lat)//2]/1e3 if lat else 0:.2f} us")

# per-CTA gaps between the end of one unit's slab stream and the next unit's first MMA
# (time the scale warps spend on unit ends: output / partial stores, merges)
tot_gap = tot_busy = 0
for fn in sorted(glob.glob(sys.argv[1] + "/trace_*.txt")):
    rows = [list(map(int, l.split())) for l in open(fn) if l.strip()]
    rows = [r for r in rows if r[3] > 0 and r[4] > 0]
    by = {}
    for u, cta, a, b, c in rows:
        by.setdefault(cta, []).append((b, c))
    for v in by.values():
        v.sort()
        tot_busy += sum(c - b for b, c in v)
        tot_gap += sum(max(0, v[i + 1][0] - v[i][1]) for i in range(len(v) - 1))
if tot_busy:
    print(f"unit-end gaps: {tot_gap / 1e3:.1f} us total over CTAs vs {tot_busy / 1e3:.1f} us streaming ({tot_gap / tot_busy:.1%})")
