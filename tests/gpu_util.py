"""Helpers shared by the -m gpu tests: seeded inputs (synth) uploaded bit for bit,
and one ac_run of a plan through the C-ABI binding."""
import numpy as np
import torch

import synth
from paper_2401_10652_b200 import api

TORCH_DT = {"bf16": torch.bfloat16, "f32": torch.float32}


def make_values(og, seed=0):
    """(oracle fp64 values, GPU tensors) from the same seeded draws."""
    samples = synth.make_inputs(og.input_specs(), seed)
    vals = {t: s.value for t, s in samples.items()}
    dev = {}
    for t, s in samples.items():
        if s.dtype == "bf16":
            dev[t] = torch.from_numpy(s.storage.astype(np.int16)).view(torch.bfloat16).cuda()
        else:
            dev[t] = torch.from_numpy(np.ascontiguousarray(s.storage)).cuda()
    return vals, dev


def c_graph(og):
    return api.graph_parse(__import__("oracle.graph", fromlist=["serialize"]).serialize(og))


GUARD = 1 << 16   # workspace canary: bytes of 0xA5 on both sides of the ac_run workspace
CANARY = 0xA5


def run(cg, plan, og, dev, stream=None, ws=None, canary=True):
    """Run `plan` once; returns ({output id: tensor}, exec).  With canary=True
    (the default when the caller passes no workspace) the workspace is carved
    out of a larger buffer whose guard bytes on both sides must be untouched
    after the run: every GPU test then checks that ac_run stays inside
    ac_plan_workspace_bytes (SURVEY §5 workspace canary)."""
    nbytes = plan.workspace_bytes()
    guarded = None
    if ws is None or ws.numel() < nbytes:
        if canary:
            guarded = torch.full((GUARD + max(nbytes, 16) + GUARD,), CANARY, dtype=torch.uint8, device="cuda")
            ws = guarded[GUARD:GUARD + max(nbytes, 16)]
        else:
            ws = torch.empty(max(nbytes, 16), dtype=torch.uint8, device="cuda")
    outs = {o: torch.empty(og.tensors[o].shape, dtype=TORCH_DT[og.tensors[o].dtype], device="cuda")
            for o in og.outputs}
    ex = api.Exec(plan, ws)
    ex.run({t: dev[t] for t in og.inputs + og.weights}, outs, stream)
    if guarded is not None:
        torch.cuda.synchronize()
        n = ws.numel()
        head, tail = guarded[:GUARD], guarded[GUARD + n:]
        assert bool((head == CANARY).all()) and bool((tail == CANARY).all()), \
            "ac_run wrote outside its workspace (canary overwritten)"
        ex.canary_buffer = guarded   # keep the parent alive with the exec
    return outs, ex


def empty_plan(cg):
    return api.plan_parse(cg, "autochunk-plan 1\n")


def rel_err(got, ref) -> float:
    """Normwise max relative error ||g - r||_inf / ||r||_inf (R18)."""
    g = got.double().cpu().numpy() if isinstance(got, torch.Tensor) else np.asarray(got, np.float64)
    r = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(g - r)) / max(np.max(np.abs(r)), 1e-300))
