"""Activation-memory estimator of the oracle (test infrastructure only).

* liveness / profile: Eq. 1, M = mem(X) + mem(Y) + mem(A), evaluated
  per execution step with exact live ranges.  Weights are
  parameter memory, not activation, and are excluded.
* estimate_with_plan: Eq. 2, M = mem(X) + mem(Y) + mem(A)/n, with the
  exact chunked liveness model of SURVEY §8(c) O3 (reading R6):
  inside a region every region input is held full from region start to region
  end, every region output is allocated full at region start, tensors that
  merely cross the region stay as they are, hoisted tensors are full, and each
  interior flow tensor is charged bytes/E * ceil(E/n) while it is live within
  one iteration.  The "memory cost due to continuous operation" is the
  optional contiguity charge, off for the GPU model.
"""
from __future__ import annotations

from dataclasses import dataclass

from .graph import Graph


@dataclass
class MemoryProfile:
    per_step: list
    peak_bytes: int
    peak_step: int
    peak_node: str
    x_bytes: int
    y_bytes: int
    a_bytes: int


def liveness(g: Graph):
    """tensor id -> (birth, death); inputs/weights born at step 0, outputs die
    at the final step, an unused tensor dies where it is born."""
    last = len(g.nodes) - 1
    rng = {}
    for i, n in enumerate(g.nodes):
        b = 0 if n.kind in ("input", "weight") else i
        rng[n.output] = [b, b]
    for i, n in enumerate(g.nodes):
        for t in n.inputs:
            rng[t][1] = max(rng[t][1], i)
    for o in g.outputs:
        rng[o][1] = last
    return {t: (b, d) for t, (b, d) in rng.items()}


def _finish(g: Graph, per_step, live_sets) -> MemoryProfile:
    if not per_step:
        return MemoryProfile([], 0, 0, "", 0, 0, 0)
    peak = max(per_step)
    ps = per_step.index(peak)                  # first step on ties
    xs = ys = 0
    for t, nb in live_sets[ps].items():
        if t in g.inputs:
            xs += nb
        elif t in g.outputs:
            ys += nb
    return MemoryProfile(per_step, peak, ps, g.nodes[ps].id, xs, ys, peak - xs - ys)


def profile(g: Graph) -> MemoryProfile:
    """Eq. 1 per step."""
    lv = liveness(g)
    wset = set(g.weights)
    per, sets = [], []
    for s in range(len(g.nodes)):
        live = {t: g.tensors[t].bytes for t, (b, d) in lv.items() if b <= s <= d and t not in wset}
        per.append(sum(live.values()))
        sets.append(live)
    return _finish(g, per, sets)


def contiguity_cost(shape, esize: int, dim: int, n: int) -> int:
    """Bytes of one materialised slice when slices along `dim` are not contiguous
    in row-major order; 0 otherwise."""
    if dim == 0 or all(s == 1 for s in shape[:dim]):
        return 0
    nb = esize
    for s in shape:
        nb *= s
    E = shape[dim]
    return nb // E * (-(-E // n))


def region_io(g: Graph, s: int, e: int, cons=None):
    """(inputs, outputs) of the interval [s, e]: inputs in order of first
    use, outputs in producer order (consumed after e, or graph outputs)."""
    if cons is None:
        cons = g.consumers()
    produced = {g.nodes[i].output for i in range(s, e + 1)}
    ins = []
    for i in range(s, e + 1):
        for t in g.nodes[i].inputs:
            if t not in produced and t not in ins:
                ins.append(t)
    outs = []
    for i in range(s, e + 1):
        t = g.nodes[i].output
        if t in g.outputs or any(c > e for c in cons[t]):
            outs.append(t)
    return ins, outs


def estimate_with_plan(g: Graph, regions, contiguity: bool = False) -> MemoryProfile:
    """Eq. 2 under a plan.  Regions with n <= 1 are dropped
    (reading R7).  Outside regions the result equals profile(g)."""
    lv = liveness(g)
    wset = set(g.weights)
    cons = g.consumers()
    per, sets = [], []
    owner = {}
    for r in regions:
        if r.n <= 1:
            continue
        for t in range(r.start, r.end + 1):
            owner[t] = r
    info = {}
    for r in regions:
        if r.n <= 1:
            continue
        ins, outs = region_io(g, r.start, r.end, cons)
        hoisted_out = {g.nodes[i].output for i in r.hoisted}
        outs = [t for t in outs if t not in hoisted_out]    # charged as hoisted tensors
        produced = {g.nodes[i].output: i for i in range(r.start, r.end + 1)}
        consumed_in = set()
        for i in range(r.start, r.end + 1):
            consumed_in.update(g.nodes[i].inputs)
        interior = {}
        for t, p in produced.items():
            if t in outs or t in hoisted_out:
                continue
            lastc = max([c for c in cons[t] if r.start <= c <= r.end], default=p)
            interior[t] = (p, lastc)
        contig = 0
        if contiguity:
            for t, d in list(r.xc) + list(r.yc):
                tm = g.tensors[t]
                contig += contiguity_cost(tm.shape, tm.esize, d, r.n)
        info[id(r)] = (ins, outs, produced, consumed_in, hoisted_out, interior, contig)
    for s in range(len(g.nodes)):
        r = owner.get(s)
        if r is None:
            live = {t: g.tensors[t].bytes for t, (b, d) in lv.items() if b <= s <= d and t not in wset}
        else:
            ins, outs, produced, consumed_in, hoisted_out, interior, contig = info[id(r)]
            live = {}
            for t in ins:
                if t not in wset:
                    live[t] = g.tensors[t].bytes
            for t in outs:
                live[t] = g.tensors[t].bytes
            for t in hoisted_out:
                live[t] = g.tensors[t].bytes
            for t, (b, d) in lv.items():
                if t in wset or t in produced or t in consumed_in:
                    continue
                if b <= s <= d:
                    live[t] = g.tensors[t].bytes
            for t, (p, lc) in interior.items():
                if p <= s <= lc:
                    tm = g.tensors[t]
                    if t in r.dims:
                        E = tm.shape[r.dims[t]]
                        live[t] = tm.bytes // E * (-(-E // r.n))
                    else:
                        live[t] = tm.bytes
            if contig:
                live["<contiguity>"] = contig
        per.append(sum(live.values()))
        sets.append(live)
    return _finish(g, per, sets)
