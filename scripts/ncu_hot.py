"""Top SASS lines by warp-stall samples per kernel of an ncu report (source page)."""
import csv
import io
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = out.split('"Kernel Name",')
    for b in blocks[1:]:
        lines = b.splitlines()
        name = lines[0]
        rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
        hdr = rows[0]
        si = hdr.index("Warp Stall Sampling (All Samples)")
        data = [(int(r[si] or 0), r[0][-5:], r[1].strip()) for r in rows[1:] if len(r) > si]
        tot = sum(d[0] for d in data) or 1
        print(name[:90], "total samples", tot)
        for s, a, src in sorted(data, reverse=True)[:top]:
            print(f"  {100 * s / tot:5.1f}%  {a}  {src[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)


def by_opcode(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    seen = set()
    for b in out.split('"Kernel Name",')[1:]:
        lines = b.splitlines()
        if lines[0] in seen:
            continue
        seen.add(lines[0])
        rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
        hdr = rows[0]
        si = hdr.index("Warp Stall Sampling (All Samples)")
        agg = {}
        for r in rows[1:]:
            if len(r) <= si:
                continue
            toks = r[1].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            op = op.split(".")[0]
            agg[op] = agg.get(op, 0) + int(r[si] or 0)
        tot = sum(agg.values()) or 1
        print(lines[0][:90])
        print("  " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:18]))
