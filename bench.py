#!/usr/bin/env python
"""Benchmark of the AutoChunk hot path: one block forward under the plan that
ac_plan selects for BASELINE.json's GPT config at a 20 % activation budget
(configs[1]), executed chunk by chunk by libautochunk's sm_100a kernels.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config gpt|vit|unet|af|tiny]

Prints ONE JSON line (rank 0).  A step = one pass of the whole hot path (LN1,
Q/K/V projections, the chunk loop of QK^T -> softmax -> PV, out-projection,
LN2, FFN1+GELU, FFN2) over one synthetic sequence resident in HBM.  `value` is
tokens/s over all ranks (device time, max over ranks); `e2e` is the same metric
through ac_run with the input copied from pinned host memory and the output
copied back inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/s and peak activation bytes vs unchunked (speed loss %) at 1/2/4/8 B200"
WORKLOADS = {
    "gpt": "GPT-style decoder block, seq 16384, hidden 1024, 16 heads, FFN 4096, causal, bf16, "
           "budget = 20% of unchunked activation (BASELINE.json configs[1])",
    "vit": "ViT-Large encoder block, 65536 tokens, hidden 1024, 16 heads, FFN 4096, bf16, budget 20%",
    "unet": "UNet self-attention, 16384 tokens, hidden 640, 10 heads, bf16, budget 20%",
    "af": "AlphaFold Evoformer pair stack (triangle multiplication outgoing / incoming, triangle attention "
          "starting / ending node, pair transition), N_res 1024, c_z 128, 4 heads, c 32, bf16, budget 20% "
          "(BASELINE.json configs[3]; tokens = pair positions N_res^2)",
    "af_attn": "AlphaFold triangle attention pair (rows then columns), N_res 1024, c_z 128, 4 heads, c 32, bf16, "
               "budget 20% (tokens = pair positions N_res^2)",
    "tiny": "tiny attention+MLP block, seq 256, hidden 64, 2 heads, fp32, chunk 32 along seq",
    "gpt_fa": "GPT-style decoder block with fused attention (NEXT f1, P:350-351), seq 16384, hidden 1024, "
              "16 heads, FFN 4096, causal, bf16, budget 90% of its unchunked activation",
}
DEFAULT_BUDGET = {"gpt_fa": 0.9}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=list(WORKLOADS), default="gpt")
    ap.add_argument("--budget-frac", type=float, default=None,
                    help="activation budget as a fraction of the unchunked peak (default 0.2; gpt_fa 0.9)")
    ap.add_argument("--plan", default=None, help="user plan text (ac_plan_parse) instead of ac_plan")
    ap.add_argument("--normalize", action="store_true",
                    help="ac_plan with normalised cost features and unit weights (AC_FLAG_NORMALIZE, R27)")
    ap.add_argument("--no-unchunked", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time direct ac_run launches instead of a captured CUDA graph of one ac_run")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no extras)")
    ap.add_argument("--sweep", action="store_true", help="also sweep the attention chunk length 64..4096")
    ap.add_argument("--layers", type=int, default=1,
                    help="stack this many blocks (NEXT f3 multi-block plans; one region per block)")
    ap.add_argument("--maxlen", action="store_true",
                    help="NEXT f3: max sequence length whose unchunked / ac_plan peak fits this GPU's free HBM "
                         "(api.max_length), then run the chunked plan at --maxlen-run tokens")
    ap.add_argument("--maxlen-run", type=int, default=0,
                    help="length of the capacity run (0: the chunked maximum itself)")
    ap.add_argument("--ablation", action="store_true",
                    help="also run the paper's Table 1 toggles (P:319-332): ac_plan with each cost term / "
                         "graph optimisation switched off, at 20/10/5 %% budgets; every distinct plan timed")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled every 5 ms through NVML
    while the timed regions run (nvidia-smi per sample is too slow for 2.5 ms steps)."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))

    def __init__(self, index: int, period: float = 0.005):
        self.index = index
        self.period = period
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._nv = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((float(sm), int(rs)))
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = sorted(x[0] for x in self.samples)
        reasons = sorted({nm for _, r in self.samples for nm, bit in self.REASONS if r & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_mhz, "sm_min_mhz": sm[0], "reasons": reasons,
                "samples": len(self.samples), "source": "NVML, 5 ms period, over the timed and profiled passes"}


# ------------------------------------------------------------------ workload
# BASELINE.json configs as ac_graph_block descriptors (kind, N, d, h, f, causal, dtype)
BLOCKS = {
    "tiny": ("transformer", 256, 64, 2, 256, False, "f32"),
    "gpt": ("transformer", 16384, 1024, 16, 4096, True, "bf16"),
    "vit": ("transformer", 65536, 1024, 16, 4096, False, "bf16"),
    "af": ("evoformer_pair", 1024, 128, 4, 32, False, "bf16"),
    "af_attn": ("tri_attn_pair", 1024, 128, 4, 32, False, "bf16"),
    "unet": ("attn_only", 16384, 640, 10, 0, False, "bf16"),
    "gpt_fa": ("transformer_fa", 16384, 1024, 16, 4096, True, "bf16"),
}


def c_graph(name, layers=1, N=None):
    """The workload graph, built by libautochunk (ac_graph_block), and its document."""
    from paper_2401_10652_b200 import api, graphdoc
    kind, N0, d, h, f, causal, dt = BLOCKS[name]
    cg = api.graph_block(kind, N or N0, d, h, f, causal, dt, name=name, layers=layers)
    return cg, graphdoc.parse(cg.serialize())


def oracle_graph(name, layers=1):
    from oracle import workloads
    c = workloads.CONFIGS[name]
    return workloads.block(c["kind"], c["N"], c["d"], c["h"], c["f"], c["causal"], c["dtype"], name, layers=layers)


def tokens_per_step(name, doc):
    shp = doc.tensors[doc.inputs[0]][1]
    return shp[0] * shp[1] if name in ("af", "af_attn") else shp[0]


def device_inputs(doc, torch):
    import numpy as np
    import synth
    samples = synth.make_inputs(doc.input_specs(), 0)
    dev = {}
    for t, s in samples.items():
        if s.dtype == "bf16":
            dev[t] = torch.from_numpy(s.storage.astype(np.int16)).view(torch.bfloat16).cuda()
        else:
            dev[t] = torch.from_numpy(np.ascontiguousarray(s.storage)).cuda()
    return samples, dev


def device_inputs_gpu(doc, torch, seed=0):
    """Inputs of the synth recipe's distributions, drawn on the device
    with torch's generator: for capacity runs at lengths whose host-side fp64 copies
    would not fit in host memory (no oracle comparison is made on them)."""
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    TD = {"bf16": torch.bfloat16, "f32": torch.float32}
    dev = {}
    for t, kind, dt, shp, role, fan in doc.input_specs():
        v = torch.randn(shp, generator=gen, device="cuda", dtype=TD[dt])   # (no fp32 temporaries)
        if role == "matrix":
            v *= 1.0 / max(fan, 1) ** 0.5
        elif role in ("bias", "ln_beta"):
            v *= 0.02
        elif role == "ln_gamma":
            v.mul_(0.02).add_(1.0)
        dev[t] = v
    torch.cuda.empty_cache()
    return dev


# ------------------------------------------------------------------ roofline bookkeeping
def _prod(xs):
    p = 1
    for x in xs:
        p *= x
    return p


def algorithmic(doc, node_id):
    """Algorithmic work of one node summed over one step.
    HBM-bound kinds: the bytes the operation must move — inputs read once,
    outputs written once, and for a causal score matrix only its lower triangle
    (j <= i).  GEMM-shaped linears: 2*M*N*K FLOPs."""
    nid, kind, ins, out, attrs = doc.node(node_id)
    B = doc.nbytes
    causal_scores = {o for (_, k, _, o, a) in doc.nodes if k == "attn_scores" and a.get("causal") == "1"}
    causal_p = {o for (_, k, i, o, _) in doc.nodes if k == "softmax" and i[0] in causal_scores}
    if kind == "linear":
        a_shape = doc.tensors[ins[0]][1]
        kin = int(attrs["kin"])
        R, K = _prod(a_shape[: len(a_shape) - kin]), _prod(a_shape[len(a_shape) - kin:])
        O = doc.tensors[ins[1]][1][0]
        return "tensor", 2 * R * K * O
    if kind == "attn_scores":
        h, N, M = doc.tensors[out][1]
        esz = B(out) // (h * N * M)
        s = h * N * (N + 1) // 2 * esz if out in causal_scores else B(out)
        return "hbm", s + B(ins[0]) + B(ins[1])
    if kind == "softmax":
        if out in causal_p:
            h, N, M = doc.tensors[out][1]
            esz = B(out) // (h * N * M)
            return "hbm", 2 * h * N * (N + 1) // 2 * esz
        return "hbm", B(ins[0]) + B(out)
    if kind == "attn_pv":
        p = B(ins[0])
        if ins[0] in causal_p:
            h, N, M = doc.tensors[ins[0]][1]
            p = h * N * (N + 1) // 2 * (p // (h * N * M))
        return "hbm", p + B(ins[1]) + B(out)
    if kind == "attn_fused":
        N, h, dh = doc.tensors[ins[0]][1]
        Nk = doc.tensors[ins[1]][1][0]
        pairs = N * (N + 1) // 2 if attrs.get("causal") == "1" else N * Nk
        return "tensor", 4 * h * dh * pairs
    if kind == "tri_mul":        # batched GEMM over channels: 2 C I J K
        C_, I, K = doc.tensors[ins[0]][1]
        return "tensor", 2 * C_ * I * K * doc.tensors[ins[1]][1][1]
    if kind in ("tri_scores", "tri_pv", "layernorm", "ln_cfirst"):
        return "hbm", sum(B(t) for t in ins) + B(out)
    return "hbm", B(out)


def cpu_baseline(name, og, samples, budget_s=20.0):
    """The oracle as it stands on this host: sampled output rows of the block
    (K/V of all rows + R query rows), rows/s, with the full-block time extrapolated
    from a 1-row and an R-row run (precompute + N x per-row).  Returns (line, rows,
    oracle values at those rows) so the GPU output can be compared with them."""
    import numpy as np
    from oracle import blocks, executor
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    vals = {t: s.value for t, s in samples.items()}
    if name in ("gpt", "vit", "unet", "tiny"):
        N = og.tensors["x"].shape[0]
        rows = np.arange(0, N, max(1, N // 32))[:32]
        t0 = time.perf_counter()
        blocks.transformer_rows(og, vals, rows[:1])
        t1 = time.perf_counter() - t0
        t0 = time.perf_counter()
        ref = blocks.transformer_rows(og, vals, rows)
        dt = time.perf_counter() - t0
        per_row = max(dt - t1, 1e-9) / (len(rows) - 1)
        pre = max(t1 - per_row, 0.0)
        return ({"value": len(rows) / dt, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                 "sample": f"{len(rows)} output rows of the {name} block incl. LN1/K/V of all {N} rows "
                           f"(fp64 numpy, {dt:.1f} s)",
                 "extrapolated_block_s": round(pre + N * per_row, 1),
                 "extrapolation": f"precompute {pre:.2f} s (LN1, K, V of all rows) + N x {per_row * 1e3:.1f} ms "
                                  f"per row, from a 1-row and a {len(rows)}-row run"},
                rows, ref)
    if name in ("af", "af_attn"):
        from oracle import workloads
        mk = workloads.evoformer_pair if name == "af" else workloads.tri_attn_pair
        small = mk(128, 128, 4, 32, "bf16", name="af_sample")
        import synth
        v = {t: s.value for t, s in synth.make_inputs(small.input_specs(), 0).items()}
        t0 = time.perf_counter()
        executor.run(small, v)
        dt = time.perf_counter() - t0
        return ({"value": 128 * 128 / dt, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                 "sample": f"the full {small.name} block at N_res=128 (fp64 numpy, {dt:.1f} s); the work per pair "
                           f"grows with N_res, so this overstates the oracle's rate at 1024",
                 "extrapolated_block_s": round(dt * (1024 / 128) ** 3, 1),
                 "extrapolation": "x (1024/128)^3: the triangle updates and attentions are cubic in N_res"},
                None, None)
    return None, None, None


def error_vs_oracle(doc, outs, rows, ref):
    """Elementwise and normwise error of the GPU block output at the oracle's sampled
    rows (fp64, the same seeded inputs): max |g - r|, normwise ||g - r||_inf / ||r||_inf
    (R18, the tolerance metric), and the elementwise relative error |g - r| / |r| over
    elements with |r| >= 1e-2 ||r||_inf (max and 99.9th percentile)."""
    import numpy as np
    if rows is None:
        return None
    key = "y" if "y" in ref else "x1"
    g = outs[doc.outputs[0]][rows].double().cpu().numpy()
    r = ref[key]
    d = np.abs(g - r)
    big = np.abs(r) >= 1e-2 * np.abs(r).max()
    el = d[big] / np.abs(r[big])
    return {"rows": len(rows), "tensor": doc.outputs[0], "max_abs": float(d.max()),
            "normwise_rel": float(d.max() / np.abs(r).max()),
            "elementwise_rel_max": float(el.max()), "elementwise_rel_p999": float(np.quantile(el, 0.999)),
            "tolerance": 2e-2 if doc.tensors[doc.outputs[0]][0] == "bf16" else 1e-4}


def planner_timing(name, cg, budget):
    """ac_plan (C++) vs the oracle's planner (Alg. 1 + Eq. 8-11 in numpy-free Python)
    on the config graph at the bench budget (the search-cost claim)."""
    from oracle import graph as og_graph, plan as oplan, select
    from paper_2401_10652_b200 import api
    og = oracle_graph(name)
    t0 = time.perf_counter()
    cp = api.ac_plan(cg, budget)
    t_c = time.perf_counter() - t0
    t0 = time.perf_counter()
    op = select.select(og, budget)
    t_o = time.perf_counter() - t0
    return {"ac_plan_ms": round(t_c * 1e3, 2), "oracle_plan_ms": round(t_o * 1e3, 1),
            "plans_identical": oplan.serialize(op, og) == cp.serialize(), "nodes": len(og.nodes)}


# ------------------------------------------------------------------ reference arm
def reference_arm(args):
    """The oracle timed as the base contract's reference arm."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    import synth
    from oracle import blocks
    og = oracle_graph(args.config)
    samples = synth.make_inputs(og.input_specs(), 0)
    vals = {t: s.value for t, s in samples.items()}
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    N = og.tensors[og.inputs[0]].shape[0]
    R = 16
    times = []
    for k in range(args.warmup + args.steps):
        rows = (np.arange(R) * (N // R) + k) % N
        t0 = time.perf_counter()
        if args.config in ("af", "af_attn"):
            from oracle import executor, workloads
            mk = workloads.evoformer_pair if args.config == "af" else workloads.tri_attn_pair
            small = mk(64, 128, 4, 32, "bf16", name="af_sample")
            executor.run(small, {t: s.value for t, s in synth.make_inputs(small.input_specs(), 0).items()})
        else:
            blocks.transformer_rows(og, vals, rows)
        if k >= args.warmup:
            times.append(time.perf_counter() - t0)
    units = 64 * 64 if args.config in ("af", "af_attn") else R
    tot = sum(times)
    value = units * len(times) / tot
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOADS[args.config], "sample": f"{units} output rows per step"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                             "sample": f"{units} sampled output rows per step (incl. full K/V)"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------ max length (NEXT f3)
def maxlen_arm(args):
    """Max inference length on this GPU (SPEC cmd_maxlen S:478-486): the
    activation budget is the free HBM minus the weights and a 2 GiB margin; the
    lengths come from the planner's own peak model (api.max_length); the chunked plan
    is then run at --maxlen-run tokens (past the unchunked maximum) to show it fits."""
    import torch
    from paper_2401_10652_b200 import api
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    kind, N0, d, h, f, causal, dt = BLOCKS[args.config]
    _, doc0 = c_graph(args.config, args.layers)
    wbytes = sum(doc0.nbytes(w[0]) for w in doc0.weights)
    free, total = torch.cuda.mem_get_info()
    budget = free - wbytes - (2 << 30)
    pair = kind in ("tri_attn_pair", "evoformer_pair")
    step = 64 if pair else 128
    cap = (1 << 15) if pair else (1 << 23)
    t0 = time.perf_counter()
    ml = api.max_length(kind, d, h, f, causal, dt, budget, layers=args.layers, step=step, cap=cap)
    t_search = time.perf_counter() - t0
    run = None
    Nr = min(args.maxlen_run or ml["chunked"], ml["chunked"]) if ml["chunked"] else 0
    fit_note = None
    while Nr:
        # the caller holds the inputs and outputs for the whole run (the plan's liveness
        # frees x after its last use and allocates y when produced), so the capacity run
        # may need up to x + y more than the planned peak: step down until it fits
        cg, doc = c_graph(args.config, args.layers, N=Nr)
        plan = api.ac_plan(cg, budget)
        need = plan.workspace_bytes() + sum(doc.nbytes(t) for t in doc.inputs + doc.outputs) + wbytes
        if need < free - (1 << 30):
            break
        fit_note = (f"executed below the planner's maximum: workspace + caller-held inputs / outputs "
                    f"at {ml['chunked']} exceed the free HBM")
        Nr -= step * max(1, (Nr // 50) // step)
    if Nr:
        prof0, _ = api.estimate_memory(cg)
        profp, _ = api.estimate_memory(cg, plan)
        dev = device_inputs_gpu(doc, torch)   # (host-free: the capacity run checks finiteness only)
        TD = {"bf16": torch.bfloat16, "f32": torch.float32}
        outs = {o: torch.empty(doc.tensors[o][1], dtype=TD[doc.tensors[o][0]], device="cuda") for o in doc.outputs}
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        ws = torch.empty(max(plan.workspace_bytes(), 16), dtype=torch.uint8, device="cuda")
        ex = api.Exec(plan, ws)
        ins = {t: dev[t] for t in doc.order}
        if Nr <= 4 * N0:     # (a capacity run at the maximum is timed once: it runs for seconds)
            ex.run(ins, outs)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ex.run(ins, outs)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        y = outs[doc.outputs[0]]
        caller = sum(doc.nbytes(t) for t in doc.inputs + doc.outputs)
        run = {"tokens": Nr, "plan": [ln.split(" flow=")[0] for ln in plan.serialize().splitlines()
                                      if ln.startswith("region")],
               "ms": round(ms, 3), "tokens_per_s": round(Nr / (ms / 1e3), 1),
               "planned_peak_bytes": profp.peak_bytes, "unchunked_peak_bytes": prof0.peak_bytes,
               "workspace_bytes": ex.stats().workspace_high_water,
               "arena_live_peak": ex.stats().arena_live_peak,
               "torch_peak_delta_bytes": torch.cuda.max_memory_allocated() - base,
               "output_finite": all(bool(torch.isfinite(c).all().item()) for c in y.view(-1).split(1 << 26)),
               **({"note": fit_note} if fit_note else {})}
    line = {"metric": "max inference length under this GPU's HBM (P:357-361)", "value": ml["chunked"],
            "unit": "tokens" if not pair else "residues", "n_gpus": 1,
            "higher_is_better": True, "dtype": dt, "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config] + (f", {args.layers} stacked blocks" if args.layers > 1 else ""),
                       "activation_budget_bytes": budget, "hbm_free_bytes": free, "weights_bytes": wbytes,
                       "length_step": step, "search_cap": cap},
            "unchunked_max": ml["unchunked"], "ratio": ml["ratio"],
            # the paper's 2D models (ViT, UNet images; AlphaFold pair representation) extend a
            # side length: tokens grow with its square for ViT / UNet, residues are the side
            "side_ratio": (ml["ratio"] ** 0.5 if args.config in ("vit", "unet") else ml["ratio"])
            if ml["ratio"] else None,
            "dims": 1 if args.config in ("gpt", "gpt_fa", "tiny") else 2,
            "plan_at_max": ml["plan"],
            "search_s": round(t_search, 2), "run": run,
            "paper": {"claim": "11.7x (1D) / 3.2x avg (2D) max-length extension", "hardware": "A100 80GB (P:336)"}}
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------ our arm
def peak_block(profp, prof0, st, budget, caller, activation_alloc, unchunked):
    """Planned (Eq. 2 under R25, ac_estimate_memory) and measured peaks, side by side.
    measured = the device bytes torch holds for the run: inputs + outputs + the whole
    workspace, all allocated at once (the caller keeps x and y for the whole run, so
    this is >= planned, whose liveness frees x after its last use and allocates y when
    it is produced); measured_unchunked likewise for the unchunked run.  The arena's
    activation high-water (arena_live_peak) plus the caller tensors live at each step
    equals the per-step plan exactly (tests/test_host_lib.py, test_gpu_parity.py)."""
    meas = activation_alloc
    mu = (unchunked or {}).get("measured_peak_bytes")
    return {"planned": profp.peak_bytes, "unchunked": prof0.peak_bytes,
            "reduction": round(1 - profp.peak_bytes / prof0.peak_bytes, 4),
            "measured": meas, "measured_unchunked": mu,
            "measured_reduction": round(1 - meas / mu, 4) if mu else None,
            "budget": budget, "workspace_bytes": st.workspace_high_water,
            "control_bytes": st.control_bytes, "arena_live_peak": st.arena_live_peak,
            "note": "planned = Eq. 2 with the fused attention chains materialised as e-tiles + slab statistics "
                    "(DESIGN.md R25), == arena live slots + caller tensors live, per step; measured = inputs + "
                    "outputs + whole workspace as torch holds them for the run (weights excluded); "
                    "control_bytes = scheduler state in the workspace (work counters, overlap epochs)"}


def self_launch(args):
    """--gpus N > 1 without a torchrun environment: relaunch this command as N ranks
    (torch.distributed.run on this node, rendezvous on 127.0.0.1)."""
    import socket
    import torch
    if args.impl == "ours" and torch.cuda.device_count() < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but only {torch.cuda.device_count()} "
                                                     f"CUDA devices are visible"}))
        return 1
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def serial_exec(plan, ws, comm):
    """An executor of the same plan with the chunk-loop overlap and programmatic
    dependent launches off (AC_OVERLAP=0, AC_PDL=0, read when the executor is created):
    its per-launch CUDA events time each kernel alone, as the ncu launch list does.
    (With the overlap on, the next chunk's scores share the SMs with the PV's tail, so
    events around single launches would charge one kernel for the other.)"""
    from paper_2401_10652_b200 import api
    old = {k: os.environ.get(k) for k in ("AC_OVERLAP", "AC_PDL")}
    os.environ.update(AC_OVERLAP="0", AC_PDL="0")
    try:
        return api.Exec(plan, ws, comm)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.impl == "reference":
        return reference_arm(args)
    import torch
    import torch.distributed as dist

    from paper_2401_10652_b200 import api

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        print(f"bench: WORLD_SIZE={world} overrides --gpus {args.gpus}", file=sys.stderr)
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    if args.maxlen:
        return maxlen_arm(args)
    cg, doc = c_graph(args.config, args.layers)
    prof0, _ = api.estimate_memory(cg)
    if args.budget_frac is None:
        args.budget_frac = DEFAULT_BUDGET.get(args.config, 0.2)
    budget = int(args.budget_frac * prof0.peak_bytes)
    if args.plan:
        # full plan text, or region lines separated by ';' (header added)
        txt = args.plan if args.plan.startswith("autochunk-plan") else \
            "autochunk-plan 1\n" + "".join(r.strip() + "\n" for r in args.plan.split(";") if r.strip())
        plan = api.plan_parse(cg, txt)
    elif args.config == "tiny":
        plan = api.plan_parse(cg, "autochunk-plan 1\nregion s=scores e=pv n=8 dims=0\n")
    elif args.normalize:
        from paper_2401_10652_b200 import _lib as L
        plan = api.ac_plan(cg, budget, api.cost_params(flags=L.AC_FLAG_NORMALIZE, alpha=1.0, beta=1.0,
                                                       gamma=-1.0, lam=1.0))
    else:
        plan = api.ac_plan(cg, budget)
    profp, _ = api.estimate_memory(cg, plan)
    comm = None
    if world > 1:
        uid = [api.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = api.Comm(uid[0], rank, world, local)
    samples, dev = device_inputs(doc, torch)
    s = torch.cuda.current_stream()
    # device allocator evidence: everything torch holds for one run minus the weights
    # (parameter memory, excluded from activation by Eq. 1) - inputs, outputs, workspace
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    weights_bytes = sum(dev[w[0]].numel() * dev[w[0]].element_size() for w in doc.weights)
    ws = torch.empty(max(plan.workspace_bytes(rank, world), 16), dtype=torch.uint8, device="cuda")
    TD = {"bf16": torch.bfloat16, "f32": torch.float32}
    outs = {o: torch.empty(doc.tensors[o][1], dtype=TD[doc.tensors[o][0]], device="cuda") for o in doc.outputs}
    activation_alloc = torch.cuda.memory_allocated() - weights_bytes  # inputs + outputs + workspace
    ins = {t: dev[t] for t in doc.order}
    ex = api.Exec(plan, ws, comm)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    use_graph = not args.no_graph and world == 1

    def timed(exe, inputs, outputs, K, W, profile=False, pre=None, post=None):
        for _ in range(W):
            exe.run(inputs, outputs)
        exe.set_profiling(profile)
        torch.cuda.synchronize()
        graph = None
        if use_graph and not profile and pre is None and post is None:
            # one ac_run captured into a CUDA graph and replayed per step (ac_run is
            # stream-ordered with no host synchronisation; replay is bitwise the direct
            # run, test_ac_run_cuda_graph_capture): the host's per-launch cost leaves the
            # timed region, which matters for the launch-bound small configs
            gs = torch.cuda.Stream()
            gs.wait_stream(s)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=gs):
                exe.run(inputs, outputs, stream=gs)
            torch.cuda.synchronize()
        barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        kt = {}
        for k in range(K):
            flush.fill_(k & 0xFF)                      # L2 flushed between timed iterations
            evs[k][0].record(s)
            if pre:
                pre()
            if graph is not None:
                graph.replay()
            else:
                exe.run(inputs, outputs)
            if post:
                post()
            evs[k][1].record(s)
            if profile:
                for node, kind, ms, n in exe.kernel_times():
                    a = kt.setdefault(node, [kind, 0.0, 0])
                    a[1] += ms
                    a[2] += n
        torch.cuda.synchronize()
        barrier()
        exe.set_profiling(False)
        tot = sum(a.elapsed_time(b) for a, b in evs)
        if world > 1:
            t = torch.tensor([tot], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot = t.item()
        return tot, kt

    peaks, peak_src = load_peaks()
    units = tokens_per_step(args.config, doc)
    clk = ClockSampler(local)
    clk.__enter__()
    tot_ms, _ = timed(ex, ins, outs, args.steps, args.warmup)
    st = ex.stats()
    # per-stage device times from a separate profiled pass (per-launch events
    # serialise the chunk loop's overlapped launches, so they stay out of `value`)
    kp = max(2, min(args.steps, 5))
    ex_prof = serial_exec(plan, ws, comm)
    prof_ms, kt = timed(ex_prof, ins, outs, kp, 1, profile=True)
    del ex_prof
    value = units * args.steps / (tot_ms / 1e3)
    ms_step = tot_ms / args.steps

    # dominant kernel roofline (device time share inside the timed steps)
    roof = None
    shares = {}
    if kt:
        total_k = sum(v[1] for v in kt.values())
        dom = max(kt.items(), key=lambda kv: kv[1][1])
        node, (kind, ms, nl) = dom
        bound, work = algorithmic(doc, node)
        per_launch_ms = ms / nl
        launches_per_step = nl / kp
        work_per_launch = work / launches_per_step
        if bound == "hbm":
            ach = work_per_launch / (per_launch_ms / 1e3) / 1e9
            pk = peaks["hbm_gbs"]
            unit = "GB/s"
        else:
            ach = work_per_launch / (per_launch_ms / 1e3) / 1e12
            pk = peaks["bf16_tflops"]   # burst: each launch runs for microseconds inside a ms-long step
            unit = "TFLOP/s"
        traffic = None
        tf = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
        if os.path.exists(tf):
            traffic = json.load(open(tf)).get(node)
        roof = {"bound": bound, "achieved": round(ach, 1), "peak": pk, "unit": unit, "frac": round(ach / pk, 4),
                "traffic": traffic, "kernel": f"{node} ({kind})", "launches_per_step": launches_per_step,
                "share_of_step": round(ms / total_k, 4), "peak_source": peak_src,
                "peak_kind": "burst (MEASURED_PEAKS bf16_tflops / hbm_gbs): the timed region is tens of ms",
                "timing": "per-launch CUDA events on the launch stream in a profiled pass right after the timed "
                          "steps, chunk-loop overlap and PDL off so each kernel is timed alone (as in the ncu "
                          "launch list); value is timed without events, overlap on"}
        def stage_roof(node, ms_step):
            if ms_step <= 0 or doc.node(node)[1] == "softmax":
                return None  # (bf16 chains: the node is the f2 statistics combine, not a softmax pass)
            b, w = algorithmic(doc, node)
            if b == "hbm":
                return {"bound": "hbm", "achieved_gbs": round(w / (ms_step / 1e3) / 1e9, 1),
                        "frac": round(w / (ms_step / 1e3) / 1e9 / peaks["hbm_gbs"], 4)}
            tf = w / (ms_step / 1e3) / 1e12
            return {"bound": "tensor", "achieved_tflops": round(tf, 1),
                    "frac": round(tf / peaks["bf16_tflops"], 4)}

        shares = {k: {"kind": v[0], "ms_per_step": round(v[1] / kp, 4), "launches_per_step": v[2] / kp,
                      "roofline": stage_roof(k, v[1] / kp)}
                  for k, v in sorted(kt.items(), key=lambda kv: -kv[1][1])}
        shares["_profiled_ms_per_step"] = round(prof_ms / kp, 4)
        # the fused attention chains inside the overlapped step (derived, not a kernel time):
        # their algorithmic bytes over the step time left after every other stage's alone time
        chain = [k for k in kt if doc.node(k)[1] in ("attn_scores", "attn_pv", "tri_scores", "tri_pv")
                 and algorithmic(doc, k)[0] == "hbm"]
        other_ms = sum(v[1] for k, v in kt.items() if k not in chain) / kp
        if chain and roof is not None and ms_step - other_ms > 0:
            cb = sum(algorithmic(doc, k)[1] for k in chain)
            chain_gbs = cb / ((ms_step - other_ms) / 1e3) / 1e9
            roof["f2_chains_in_step"] = {
                "nodes": sorted(chain), "algorithmic_bytes_per_step": int(cb),
                "ms": round(ms_step - other_ms, 4), "achieved_gbs": round(chain_gbs, 1),
                "frac": round(chain_gbs / peaks["hbm_gbs"], 4),
                "derivation": "timed step minus the alone times of all other stages; the chains' "
                              "scores and PV overlap across chunks, so this is their joint in-step rate"}

    # same kernels, unchunked (speed loss) — when it fits
    caller_bytes = sum(doc.nbytes(t) for t in doc.inputs + doc.outputs)
    unchunked = None
    if not args.no_unchunked and not args.profile:
        try:
            up = api.plan_parse(cg, "autochunk-plan 1\n")
            need = up.workspace_bytes(rank, world)
            free, _ = torch.cuda.mem_get_info()
            if need + (1 << 30) < free:
                wsu = torch.empty(need, dtype=torch.uint8, device="cuda")
                exu = api.Exec(up, wsu, comm)
                ku = max(3, args.steps // 2)
                tu, _ = timed(exu, ins, outs, ku, 2)
                exs_ = serial_exec(up, wsu, comm)
                _, ktu = timed(exs_, ins, outs, ku, 1, profile=True)
                del exs_
                vu = units * ku / (tu / 1e3)
                stu = exu.stats()
                unchunked = {"value": vu, "ms_per_step": tu / ku,
                             **({"note": f"the empty plan on every rank (replicated work at {world} ranks)"}
                                if world > 1 else {}),
                             "speed_loss": 1.0 - value / vu, "workspace_bytes": need,
                             "arena_live_peak": stu.arena_live_peak,
                             "measured_peak_bytes": need + caller_bytes,
                             "stages_ms": {k: round(v[1] / ku, 4) for k, v in
                                           sorted(ktu.items(), key=lambda kv: -kv[1][1])}}
                del exu, wsu
            else:
                unchunked = {"value": None, "speed_loss": None, "note": f"unchunked OOM (needs {need} B)"}
        except Exception as e:  # pragma: no cover
            unchunked = {"error": str(e)}
        torch.cuda.empty_cache()
    clk.__exit__()
    clocks = clk.summary()

    # end to end: pinned host input -> device, ac_run, output -> pinned host, every
    # step.  Pipelined as a serving loop would run it: step k's H2D (copy stream)
    # and step k-1's D2H (second copy stream) overlap step k-1 / k's ac_run on the
    # compute stream; two device input / output slots, events order each slot's reuse.
    e2e = None
    if not args.no_e2e and not args.profile:
        xin = doc.inputs[0]
        yout = doc.outputs[0]
        hx = torch.empty_like(dev[xin], device="cpu").pin_memory()
        hx.copy_(dev[xin].cpu())
        hy = torch.empty_like(outs[yout], device="cpu").pin_memory()
        dxs = [torch.empty_like(dev[xin]) for _ in range(2)]
        outs2 = [outs, {o: torch.empty_like(t) for o, t in outs.items()}]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        K = args.steps

        def e2e_run(K, timed_region):
            ev = lambda: torch.cuda.Event(enable_timing=timed_region)  # noqa: E731
            in_ready = [ev() for _ in range(K)]
            run_done = [ev() for _ in range(K)]
            out_done = [ev() for _ in range(K)]
            t0, t1 = ev(), ev()
            torch.cuda.synchronize()
            barrier()
            t0.record(s_in)
            for k in range(K):
                slot = k & 1
                with torch.cuda.stream(s_in):
                    if k >= 2:
                        s_in.wait_event(run_done[k - 2])    # ac_run k-2 has read this input slot
                    dxs[slot].copy_(hx, non_blocking=True)
                    in_ready[k].record(s_in)
                s.wait_event(in_ready[k])
                if k >= 2:
                    s.wait_event(out_done[k - 2])           # D2H k-2 has read this output slot
                ins2 = dict(ins)
                ins2[xin] = dxs[slot]
                ex.run(ins2, outs2[slot])
                run_done[k].record(s)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(run_done[k])
                    hy.copy_(outs2[slot][yout], non_blocking=True)
                    out_done[k].record(s_out)
            s_in.wait_stream(s_out)
            t1.record(s_in)
            torch.cuda.synchronize()
            barrier()
            return t0.elapsed_time(t1) if timed_region else None

        e2e_run(2, False)
        te = e2e_run(K, True)
        if world > 1:
            t = torch.tensor([te], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = t.item()
        e2e = {"value": units * K / (te / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": hx.numel() * hx.element_size(),
               "d2h_bytes_per_step": hy.numel() * hy.element_size(),
               "pipelined": "H2D / D2H on two copy streams overlapping the neighbouring steps' ac_run"}

    # chunk-size sweep of the plan's regions (BASELINE.json configs[4]: UNet chunk
    # length 64..4096; the same for GPT / ViT; AlphaFold: n = 4..128 on both attentions)
    sweep = None
    if args.sweep and not args.profile:
        sweep = []
        base_regions = [dict(x.split("=", 1) for x in ln.split()[1:]) for ln in plan.serialize().splitlines()
                        if ln.startswith("region")]
        pair = args.config in ("af", "af_attn")
        ladder = (4, 8, 16, 32, 64, 128) if pair else \
            [-(-int(base_regions[0]["ext"]) // L) for L in (64, 128, 256, 512, 1024, 2048, 4096)] if base_regions else []
        for n in ladder:
            txt = "autochunk-plan 1\n" + "".join(f"region s={r['s']} e={r['e']} n={n} yc={r['yc']}\n"
                                                 for r in base_regions)
            sp = api.plan_parse(cg, txt)
            pr, _ = api.estimate_memory(cg, sp)
            wss = torch.empty(max(sp.workspace_bytes(rank, world), 16), dtype=torch.uint8, device="cuda")
            exs = api.Exec(sp, wss, comm)
            ks = max(2, args.steps // 2)
            ts, _ = timed(exs, ins, outs, ks, 1)
            sweep.append({"n": n, "chunk_len": -(-int(base_regions[0]["ext"]) // n),
                          "tokens_per_s": round(units * ks / (ts / 1e3), 1), "planned_peak": pr.peak_bytes,
                          "peak_frac": round(pr.peak_bytes / prof0.peak_bytes, 4),
                          "speed_vs_unchunked": round(units * ks / (ts / 1e3) / unchunked["value"], 4)
                          if unchunked and unchunked.get("value") else None})
            del exs, wss
        torch.cuda.empty_cache()

    # Table 1 ablation (NEXT f4): plans under each toggle, each distinct plan timed once
    ablation = None
    if args.ablation and not args.profile:
        import ctypes as C
        from paper_2401_10652_b200 import _lib as L
        toggles = [("all strategies", 0), ("no computation density", 2), ("no dimension strides", 4),
                   ("no number of nodes", 8), ("no flops", 16), ("no graph optimization", 1)]
        timed_plans = {}
        ablation = []
        for frac in (0.2, 0.1, 0.05):
            for name, flag in toggles:
                prm = L.CostParams()
                L.lib().ac_cost_params_default(C.byref(prm))
                prm.flags = flag
                ap_ = api.ac_plan(cg, int(frac * prof0.peak_bytes), prm)
                txt = "\n".join(ln.split(" flow=")[0] for ln in ap_.serialize().splitlines() if ln.startswith("region"))
                if txt not in timed_plans:
                    pr_, _ = api.estimate_memory(cg, ap_)
                    wsa = torch.empty(max(ap_.workspace_bytes(rank, world), 16), dtype=torch.uint8, device="cuda")
                    exa = api.Exec(ap_, wsa, comm)
                    ka = max(3, args.steps // 2)
                    ta, _ = timed(exa, ins, outs, ka, 2)
                    timed_plans[txt] = (units * ka / (ta / 1e3), pr_.peak_bytes / prof0.peak_bytes, ap_.feasible)
                    del exa, wsa
                tps, pfrac, feas = timed_plans[txt]
                ablation.append({"budget_frac": frac, "toggle": name, "plan": txt.splitlines(),
                                 "feasible": bool(feas), "planned_peak_frac": round(pfrac, 4),
                                 "tokens_per_s": round(tps, 1)})
        # "No graph optimization" where it bites: a forced region holding the K / V
        # projections (off the row flow), hoisted vs recomputed in every chunk (opt=0)
        if args.config in ("gpt", "vit", "unet", "gpt_fa"):
            n_f = 8
            s0, e0 = "proj_q", ("attn" if args.config == "gpt_fa" else "pv")
            for opt in ("", " opt=0"):
                txt = f"region s={s0} e={e0} n={n_f} dims=0{opt}"
                fp = api.plan_parse(cg, "autochunk-plan 1\n" + txt + "\n")
                pr_, _ = api.estimate_memory(cg, fp)
                wsa = torch.empty(max(fp.workspace_bytes(rank, world), 16), dtype=torch.uint8, device="cuda")
                exa = api.Exec(fp, wsa, comm)
                ka = max(3, args.steps // 2)
                ta, _ = timed(exa, ins, outs, ka, 2)
                del exa, wsa
                ablation.append({"budget_frac": None, "toggle": "forced region, graph optimization " +
                                 ("off" if opt else "on"), "plan": [txt], "feasible": None,
                                 "planned_peak_frac": round(pr_.peak_bytes / prof0.peak_bytes, 4),
                                 "tokens_per_s": round(units * ka / (ta / 1e3), 1)})
            on, off = ablation[-2]["tokens_per_s"], ablation[-1]["tokens_per_s"]
            ablation[-1]["speed_vs_all"] = round(off / on, 4)
            ablation[-2]["speed_vs_all"] = 1.0
        for frac in (0.2, 0.1, 0.05):
            ref = [a["tokens_per_s"] for a in ablation if a["budget_frac"] == frac and a["toggle"] == "all strategies"][0]
            for a in ablation:
                if a["budget_frac"] == frac:
                    a["speed_vs_all"] = round(a["tokens_per_s"] / ref, 4)
        torch.cuda.empty_cache()

    if rank != 0:
        return 0
    cpu, err, ptime = None, None, None
    if not args.no_cpu and not args.profile:
        try:
            base_cfg = "gpt" if args.config == "gpt_fa" else args.config   # same block maths, unfused ids
            if args.layers == 1:
                cpu, rows, ref = cpu_baseline(base_cfg, oracle_graph(base_cfg), samples)
                # the timed runs left the block output of the last step in `outs`
                err = error_vs_oracle(doc, outs, rows, ref)
            else:
                cpu = {"note": "oracle row sampler covers one block; stacks are parity-tested in tests/"}
        except Exception as e:  # pragma: no cover
            cpu = {"error": str(e)}
        if args.config not in ("tiny",) and args.layers == 1 and not args.plan:
            try:
                ptime = planner_timing(args.config, cg, budget)
            except Exception as e:  # pragma: no cover
                ptime = {"error": str(e)}
    plan_txt = plan.serialize().splitlines()
    regions = [ln.split(" flow=")[0] for ln in plan_txt if ln.startswith("region")]
    caller = sum(doc.nbytes(t) for t in doc.inputs + doc.outputs)
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": doc.tensors[doc.inputs[0]][0],
        "data": "synthetic (seeded PCG64, DESIGN.md §4)",
        "config": {"workload": WORKLOADS[args.config] + (f", {args.layers} stacked blocks" if args.layers > 1 else ""),
                   "plan": regions, "parallelism": f"chunk-split x{world}" + (
                       " (zigzag / round-robin chunk shares, row-partitioned post-region nodes, NCCL all-gather)"
                       if world > 1 else ""),
                   **({"cost": "normalised features, unit weights (AC_FLAG_NORMALIZE, R27)"} if args.normalize else {}),
                   "pipelined_chunks": st.pipelined_chunks,
                   "l2": "flushed between timed steps (256 MiB write)",
                   "launch": "one ac_run captured as a CUDA graph, replayed per step" if use_graph else
                             "direct ac_run launches"},
        "peak_activation_bytes": peak_block(profp, prof0, st, budget, caller, activation_alloc, unchunked),
        "unchunked": unchunked, "roofline": roof, "stages": shares, "cpu_baseline": cpu, "e2e": e2e,
        "error_vs_oracle": err, "planner_timing": ptime,
        **({"chunk_sweep": sweep} if sweep else {}),
        **({"ablation": ablation} if ablation else {}),
        "gpu_launches": st.launches * args.steps, "clocks": clocks,
        "paper": {"claim": ">80% activation reduction at <10% speed loss; <10% loss at 20% memory",
                  "hardware": "A100 80GB, PyTorch (P:336)"},
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
