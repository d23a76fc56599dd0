"""bench.py contract pieces that run without a GPU: the reference arm (the fp64
oracle timed on the host) prints one JSON line with the agreed keys,
and the roofline bookkeeping counts algorithmic work as DESIGN.md §5 states."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("GPT-style decoder block")


def test_algorithmic_work_per_node():
    sys.path.insert(0, ROOT)
    import bench
    from paper_2401_10652_b200 import graphdoc
    cg, doc = bench.c_graph("gpt")
    N, d, h, f = 16384, 1024, 16, 4096
    assert bench.algorithmic(doc, "ffn1") == ("tensor", 2 * N * d * f)
    # causal scores: the lower triangle of S (bf16) plus q and k read once
    bound, b = bench.algorithmic(doc, "scores")
    assert bound == "hbm" and b == h * N * (N + 1) // 2 * 2 + 2 * (N * d * 2)
    cgf, docf = bench.c_graph("gpt_fa")
    assert bench.algorithmic(docf, "attn") == ("tensor", 4 * h * (d // h) * N * (N + 1) // 2)
