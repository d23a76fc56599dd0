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
* f2 materialisation (reading R25): in a bf16 graph the chain
  scores -> softmax(over keys) -> PV is executed with the softmax normalisation
  folded into the PV, so what exists in memory is not the IR's S and P but
    S: the exponentials e in 128-row x 64-key tiles (rows and keys padded up),
    P: per (row, 64-key slab) statistics (max, sum) in fp32 (8 bytes),
  with P written by the scores step and S read by the PV step.  Eq. 1 / Eq. 2
  charge those bytes (mem(A) is what is materialised).  The chain
  qualifies when S / P feed only the next node of the chain, the PV's head dim
  is <= 64 and a multiple of 8, the key count >= 64 and a multiple of 8, and all
  three nodes sit in the same region (not hoisted, S and P cut along the same
  dim, never the keys) or all outside regions.
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
    live_sets: list = None       # per step: {tensor id: bytes live at that step}


def f2_chains(g: Graph, regions=()):
    """The fused chains of R25 under `regions` (regions with n <= 1 ignored):
    list of (scores, softmax, pv) node indices."""
    live = [r for r in regions if r.n > 1]

    def region_of(i):
        for k, r in enumerate(live):
            if r.start <= i <= r.end:
                return k
        return None

    cons = g.consumers()
    out = []
    for i, n in enumerate(g.nodes):
        if n.kind not in ("attn_scores", "tri_scores"):
            continue
        s_t = n.output
        S = g.tensors[s_t]
        kd = len(S.shape) - 1
        if S.dtype != "bf16" or s_t in g.outputs or len(cons[s_t]) != 1:
            continue
        sm = cons[s_t][0]
        if g.nodes[sm].kind != "softmax" or g.nodes[sm].attrs.get("dim") != kd:
            continue
        p_t = g.nodes[sm].output
        if p_t in g.outputs or len(cons[p_t]) != 1:
            continue
        pv = cons[p_t][0]
        want = "tri_pv" if n.kind == "tri_scores" else "attn_pv"
        if g.nodes[pv].kind != want or g.nodes[pv].inputs[0] != p_t:
            continue
        dh = g.tensors[g.nodes[pv].output].shape[-1]
        nk = S.shape[kd]
        if dh > 64 or dh % 8 or nk < 64 or nk % 8:
            continue
        ks = {region_of(i), region_of(sm), region_of(pv)}
        if len(ks) != 1:
            continue
        k = ks.pop()
        if k is not None:
            r = live[k]
            if {i, sm, pv} & set(r.hoisted):
                continue
            ds, dp = r.dims.get(s_t), r.dims.get(p_t)
            if ds != dp or ds == kd:
                continue
        out.append((i, sm, pv))
    return out


def etile_bytes(shape) -> int:
    """S of a fused chain: [..B.., M, nk] as 128 x 64 tiles of bf16 (R25)."""
    B = 1
    for x in shape[:-2]:
        B *= x
    M, nk = shape[-2], shape[-1]
    return B * (-(-M // 128) * 128) * (-(-nk // 64) * 64) * 2


def stats_bytes(shape) -> int:
    """P of a fused chain: one fp32 (max, sum) per row and 64-key slab (R25)."""
    B = 1
    for x in shape[:-2]:
        B *= x
    M, nk = shape[-2], shape[-1]
    return B * M * (-(-nk // 64)) * 8


class _Mat:
    """Materialised bytes of a tensor, with its chunk dim cut to ceil(E/n)."""

    def __init__(self, g: Graph, chains):
        self.g = g
        self.role = {}
        for i, sm, pv in chains:
            self.role[g.nodes[i].output] = "e"
            self.role[g.nodes[sm].output] = "stats"

    def bytes(self, t, d=None, n=1) -> int:
        tm = self.g.tensors[t]
        shape = list(tm.shape)
        if d is not None:
            shape[d] = -(-shape[d] // n)
        kind = self.role.get(t)
        if kind == "e":
            return etile_bytes(shape)
        if kind == "stats":
            return stats_bytes(shape)
        if d is None:
            return tm.bytes
        return tm.bytes // tm.shape[d] * shape[d]


def liveness(g: Graph, chains=()):
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
    for i, sm, pv in chains:                  # R25: P written by the scores, S read by the PV
        rng[g.nodes[sm].output][0] = min(rng[g.nodes[sm].output][0], i)
        rng[g.nodes[i].output][1] = max(rng[g.nodes[i].output][1], pv)
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
    return MemoryProfile(per_step, peak, ps, g.nodes[ps].id, xs, ys, peak - xs - ys, live_sets)


def profile(g: Graph) -> MemoryProfile:
    """Eq. 1 per step, f2 chains materialised as R25 says."""
    chains = f2_chains(g)
    mat = _Mat(g, chains)
    lv = liveness(g, chains)
    wset = set(g.weights)
    per, sets = [], []
    for s in range(len(g.nodes)):
        live = {t: mat.bytes(t) for t, (b, d) in lv.items() if b <= s <= d and t not in wset}
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
    chains = f2_chains(g, regions)
    mat = _Mat(g, chains)
    f2_birth = {g.nodes[sm].output: i for i, sm, pv in chains}
    f2_death = {g.nodes[i].output: pv for i, sm, pv in chains}
    lv = liveness(g, chains)
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
            interior[t] = (min(p, f2_birth.get(t, p)), max(lastc, f2_death.get(t, lastc)))
        contig = 0
        if contiguity:
            for t, d in list(r.xc) + list(r.yc):
                tm = g.tensors[t]
                contig += contiguity_cost(tm.shape, tm.esize, d, r.n)
        info[id(r)] = (ins, outs, produced, consumed_in, hoisted_out, interior, contig)
    for s in range(len(g.nodes)):
        r = owner.get(s)
        if r is None:
            live = {t: mat.bytes(t) for t, (b, d) in lv.items() if b <= s <= d and t not in wset}
        else:
            ins, outs, produced, consumed_in, hoisted_out, interior, contig = info[id(r)]
            live = {}
            for t in ins:
                if t not in wset:
                    live[t] = mat.bytes(t)
            for t in outs:
                live[t] = mat.bytes(t)
            for t in hoisted_out:
                live[t] = mat.bytes(t)
            for t, (b, d) in lv.items():
                if t in wset or t in produced or t in consumed_in:
                    continue
                if b <= s <= d:
                    live[t] = mat.bytes(t)
            for t, (p, lc) in interior.items():
                if p <= s <= lc:
                    live[t] = mat.bytes(t, r.dims.get(t), r.n)
            if contig:
                live["<contiguity>"] = contig
        per.append(sum(live.values()))
        sets.append(live)
    return _finish(g, per, sets)
