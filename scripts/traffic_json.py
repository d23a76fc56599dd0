"""DRAM bytes per launch of the f2 / fused kernels from an ncu CSV
(--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum) of one
ac_run -> profiles/traffic_<config>.json keyed by the graph nodes bench.py's roofline
names.  Usage: traffic_json.py CSV CONFIG"""
import csv
import io
import json
import sys

KIND = {  # kernel template -> node ids it runs in the bench configs
    "gemm_tc_kernel<256, 1>": ["scores"], "gemm_tc_kernel<128, 1>": ["scores"],
    "gemm_tc_kernel<256, 3>": ["row_scores", "col_scores"], "gemm_tc_kernel<256, 4>": ["row_scores", "col_scores"],
    "gemm_tc_kernel<64, 2>": ["pv"], "gemm_tc_kernel<32, 2>": ["row_pv", "col_pv"],
    "stats_combine_kernel": ["softmax", "row_softmax", "col_softmax"],
    "attn_fused_kernel": ["attn"], "attn_fused_kernel<2>": ["attn"], "attn_fused_kernel<1>": ["attn"],
}


def main(path, cfg):
    txt = open(path).read().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(txt[start:]))))
    hdr = rows[0]
    ik, im, iv, iu = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    per = {}
    for r in rows[1:]:
        name = r[ik].replace("void ", "").replace("ac::<unnamed>::", "").replace("(int)", "")
        name = name.split("(")[0].strip().split("::")[-1]
        if r[im] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[iu], 1)
        key = (name, r[0])
        per[key] = per.get(key, 0.0) + float(r[iv].replace(",", "")) * mult
    agg = {}
    for (name, _), b in per.items():
        a = agg.setdefault(name, [0.0, 0])
        a[0] += b
        a[1] += 1
    out = {"_source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum over one {cfg} ac_run; bytes per launch "
                      "averaged over the kernel's launches"}
    for name, (b, n) in agg.items():
        for k, nodes in KIND.items():
            if name.replace(" ", "") == k.replace(" ", ""):
                for node in nodes:
                    out[node] = int(b / n)
    out["_kernels"] = {name: {"launches": n, "bytes_per_launch": int(b / n)} for name, (b, n) in agg.items()}
    json.dump(out, open(f"profiles/traffic_{cfg}.json", "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
