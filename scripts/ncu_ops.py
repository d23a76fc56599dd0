"""Per-opcode instruction counts and stall samples of each kernel in an ncu report
(source page, SASS view): where a kernel's issue slots and stalls go."""
import csv
import io
import subprocess
import sys


def main(path, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    for b in out.split('"Kernel Name",')[1:]:
        lines = b.splitlines()
        rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
        hdr = rows[0]
        ie = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        agg = {}
        stalls = {}
        for r in rows[1:]:
            if len(r) <= si or not r[1].strip():
                continue
            toks = r[1].split()
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            op = ".".join(op.split(".")[:2])
            n = float(r[ie] or 0)
            s = float(r[si] or 0)
            a = agg.setdefault(op, [0.0, 0.0])
            a[0] += n
            a[1] += s
            for i in stall_cols:
                stalls[hdr[i]] = stalls.get(hdr[i], 0) + float(r[i] or 0)
        tn = sum(v[0] for v in agg.values()) or 1
        ts = sum(v[1] for v in agg.values()) or 1
        print(lines[0][:100], f"warp-instructions {tn:.3e}, stall samples {ts:.0f}")
        for op, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
            print(f"  {op:28s} inst {100 * n / tn:5.1f}%  stall {100 * s / ts:5.1f}%")
        tot = sum(stalls.values()) or 1
        print("  stall reasons:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in
                                           sorted(stalls.items(), key=lambda kv: -kv[1])[:10]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
