"""AutoChunk ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU reimplementation of what the AutoChunk
hot path computes (arXiv 2401.10652, /root/reference/PAPER.md = "P:<line>"):

* ops.py       — fp64 definitions of every IR node kind (block math, O1)
* graph.py     — the graph IR, its text document, shapes and FLOPs
* executor.py  — run / run_chunked / tracked_run (Eq. 2 chunk procedure P:99-102)
* memory.py    — Eq. 1 profile and Eq. 2 estimate under a plan
* search.py    — chunk flows, Rules 1-4, Algorithm 1
* select.py    — cost model Eq. 8-10 and DP + beam selection Eq. 11
* workloads.py — the five BASELINE.json configurations as graphs

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
anything under oracle/.  The product path (paper_2401_10652_b200/) never does;
it shares no code with this package (only the seeded generators in synth/).

Parity status per function is listed in DESIGN.md §"Oracle pins".
"""
