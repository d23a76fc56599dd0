"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
total device time, launches, share.  Usage: launches.py CSV [--skip-steps N]"""
import csv
import io
import sys


def load(path):
    txt = open(path).read().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(txt[start:]))))
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        v = float(r[iv].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r[iu], 1.0)
        name = r[ik]
        short = name.split("(")[0].replace("void ", "").replace("ac::<unnamed>::", "")
        out.append((short, v * scale))
    return out


def main(path):
    ls = load(path)
    tot = {}
    for k, us in ls:
        a = tot.setdefault(k, [0.0, 0])
        a[0] += us
        a[1] += 1
    T = sum(v[0] for v in tot.values())
    print(f"{len(ls)} launches, {T:.1f} us total")
    for k, (us, n) in sorted(tot.items(), key=lambda x: -x[1][0]):
        print(f"  {k:60s} {us:10.1f} us  x{n:<4d} share {us / T:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
