"""Compact summary of profiles/r2_bench_lines.jsonl (sweeps, ablations, forced plan, max length)."""
import json
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "profiles/r2_bench_lines.jsonl"
for line in open(path):
    d = json.loads(line)
    f = d["_file"]
    if "chunk_sweep" in d:
        pts = d["chunk_sweep"]
        print(f, " | ".join(f"len {p.get('chunk_len')}: {p.get('tokens_per_s', 0) / 1e6:.2f}M "
                             f"({p.get('speed_vs_unchunked', p.get('speed', 0)):.2f}, {100 * p.get('planned_peak_frac', 0):.1f}%)"
                             for p in pts))
    elif "ablation" in d:
        for p in d["ablation"]:
            print(f, p.get("budget_frac"), p.get("toggle"), p.get("speed_vs_all"), p.get("plan", [""])[0][:60])
    elif "unchunked_max" in d:
        print(f, "value", d["value"], "unchunked_max", d["unchunked_max"], "ratio", d["ratio"], "side", d.get("side_ratio"),
              "run", json.dumps(d.get("run"))[:200])
    else:
        u = d.get("unchunked") or {}
        print(f, f"{d['value'] / 1e6:.3f}M", d["ms_per_step"], "loss", u.get("speed_loss"),
              "red", (d.get("peak_activation_bytes") or {}).get("reduction"))
