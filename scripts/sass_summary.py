#!/usr/bin/env python
"""Per-kernel SASS instruction census of libautochunk.so (cuobjdump -sass): the
Blackwell-specific mnemonics that prove the hot path runs on tcgen05 / TMEM / TMA
(B200_PROFILING.md): UTCHMMA / UTCQMMA (tcgen05.mma), UTMALDG / UTMASTG (TMA tensor
loads / stores), UBLKCP (bulk copies), LDTM / STTM (TMEM loads / stores), UTCBAR
(tcgen05.commit), MUFU.EX2, plus the register count from cuobjdump -res-usage.

    python scripts/sass_summary.py [lib] > profiles/r2_sass_summary.txt
"""
import collections
import os
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "paper_2401_10652_b200",
                                                          "libautochunk.so")
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "LDTM", "STTM", "MUFU.EX2",
        "SYNCS", "HMMA"]

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
regs = {}
cur = None
for ln in res.splitlines():
    m = re.search(r"Function (\S+):", ln)
    if m:
        cur = m.group(1)
    m = re.search(r"REG:(\d+).*SHARED:(\d+)", ln)
    if m and cur:
        regs[cur] = (int(m.group(1)), int(m.group(2)))
counts = collections.OrderedDict()
cur = None
for ln in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", ln)
    if not m:
        continue
    op = m.group(2)
    for k in KEYS:
        if op == k or op.startswith(k + "."):
            counts[cur][k] += 1
demangle = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
print(f"# SASS census of {os.path.basename(LIB)} (cuobjdump -sass, sm_100a); regs / static smem from -res-usage")
print("kernel".ljust(70) + "".join(k.rjust(9) for k in KEYS) + "  regs")
tot = collections.Counter()
for (mangled, c), name in zip(counts.items(), demangle):
    if not sum(c.values()):
        continue
    tot.update(c)
    short = re.sub(r"\(.*", "", name.replace("ac::(anonymous namespace)::", ""))[:68]
    print(short.ljust(70) + "".join(str(c[k]).rjust(9) for k in KEYS) + f"  {regs.get(mangled, ('?',))[0]}")
print("TOTAL".ljust(70) + "".join(str(tot[k]).rjust(9) for k in KEYS))
