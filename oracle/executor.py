"""Reference interpreter of the oracle (test infrastructure only).

* run          — Y = F(X): nodes in topological order, float64.
* run_chunked  — the chunk procedure of P:99-102: for each region the chunkable
                 inputs X^c are split into n segments (ceil split, short last
                 segment), y_i = F(x_i) is computed segment by segment
                 with X^nc passed whole, and y_i is written in place into the
                 pre-allocated Y^c, so Y = [y_1; ...; y_n].
* tracked_run  — the same execution with a buffer tracker that measures live
                 activation bytes per step from the buffers that actually exist
                 (the brute-force check of Eq. 1 / Eq. 2).  A fused
                 bf16 chain (R25, memory.f2_chains) allocates what the
                 GPU path materialises: the e-tile buffer (rows padded to 128,
                 keys to 64, bf16) at the scores step together with the slab
                 statistics buffer (fp32 pairs per row and 64-key slab), both
                 released after the PV; the chain's values are computed as usual.
Values are float64.  With mirror=True every bf16 tensor is rounded to bf16
(round-to-nearest-even) after it is produced, mirroring the GPU storage points
(reading R17); the default is pure fp64.
"""
from __future__ import annotations

import numpy as np

from . import ops
from .graph import Graph


def round_bf16(x: np.ndarray) -> np.ndarray:
    """float64 -> nearest bf16 value (ties to even), returned as float64."""
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    finite = np.isfinite(f)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    r = np.where(finite, r, u & 0xFFFF0000)
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def _eval(g: Graph, i: int, vals, ctx=None, mirror=False):
    n = g.nodes[i]
    out = ops.evaluate(n.kind, n.attrs, vals, ctx)
    if mirror and g.tensors[n.output].dtype == "bf16":
        out = round_bf16(out)
    return out


def run(g: Graph, values: dict, mirror: bool = False, keep_all: bool = False) -> dict:
    env = dict(values)
    for i, n in enumerate(g.nodes):
        if n.kind in ("input", "weight"):
            if n.output not in env:
                raise ValueError(f"missing value for {n.output}")
            continue
        env[n.output] = _eval(g, i, [env[t] for t in n.inputs], None, mirror)
    return env if keep_all else {o: env[o] for o in g.outputs}


def _slice(a: np.ndarray, d: int, off: int, ln: int) -> np.ndarray:
    idx = [slice(None)] * a.ndim
    idx[d] = slice(off, off + ln)
    return a[tuple(idx)]


class _Tracker:
    def __init__(self, g: Graph):
        self.g = g
        self.live = {}

    def alloc(self, key, nbytes):
        self.live[key] = nbytes

    def free(self, key):
        self.live.pop(key, None)

    def total(self):
        return sum(self.live.values())


def _last_use(g: Graph, chains=()):
    last = {}
    for i, n in enumerate(g.nodes):
        last.setdefault(n.output, 0 if n.kind in ("input", "weight") else i)
        for t in n.inputs:
            last[t] = i
    for o in g.outputs:
        last[o] = len(g.nodes)  # never freed
    for i, sm, pv in chains:    # the PV reads the e-tiles
        last[g.nodes[i].output] = max(last[g.nodes[i].output], pv)
    return last


def _f2_buffers(shape):
    """The two buffers a fused chain's scores step creates for an S of `shape`
    [..B.., M, nk]: e-tiles (bf16, 128-row x 64-key blocks) and the slab
    statistics (fp32 max and sum per row and 64-key slab).  Real arrays: the
    tracker counts their nbytes."""
    *lead, M, nk = shape
    e = np.empty(tuple(lead) + (-(-M // 128) * 128, -(-nk // 64) * 64), dtype=np.uint16)
    st = np.empty(tuple(lead) + (M, -(-nk // 64), 2), dtype=np.float32)
    return e, st


def tracked_run(g: Graph, values: dict, regions=(), mirror=False, contiguity=False, chunk_ranges=None):
    """Execute (chunked if regions are given) while measuring the live activation
    bytes at every step from real buffers.  Returns (outputs, per_step).
    chunk_ranges: optional {region index: (c0, c1)} — only those chunks run (one
    rank's share); Y^c slabs of other chunks stay zero."""
    ranges = {}
    for k, r in enumerate(regions):
        if r.n > 1 and chunk_ranges is not None and k in chunk_ranges:
            ranges[id(r)] = chunk_ranges[k]
    regions = [r for r in regions if r.n > 1]
    from .memory import f2_chains
    chains = f2_chains(g, regions)
    f2 = {i: (sm, pv) for i, sm, pv in chains}          # scores node -> (softmax, pv)
    f2_soft = {sm for i, sm, pv in chains}
    esz = {t: g.tensors[t].esize for t in g.tensors}
    wset = set(g.weights)
    tr = _Tracker(g)
    last = _last_use(g, chains)
    env = dict(values)
    per_step = [0] * len(g.nodes)
    for n in g.nodes:                         # inputs are born at step 0
        if n.kind == "input":
            tr.alloc(n.output, env[n.output].size * esz[n.output])
    at = {r.start: r for r in regions}
    i = 0
    while i < len(g.nodes):
        n = g.nodes[i]
        if i in at:
            r = at[i]
            _tracked_region(g, r, env, tr, per_step, esz, wset, last, mirror, contiguity,
                            ranges.get(id(r), (0, r.n)), f2, f2_soft)
            # free everything whose last use was inside the region
            for t in list(tr.live):
                if isinstance(t, str) and last.get(t, -1) <= r.end:
                    tr.free(t)
            i = r.end + 1
            continue
        if n.kind in ("input", "weight"):
            per_step[i] = tr.total()
        else:
            out = _eval(g, i, [env[t] for t in n.inputs], None, mirror)
            env[n.output] = out
            if i in f2:                     # fused chain: e-tiles + statistics
                e, st = _f2_buffers(out.shape)
                tr.alloc(n.output, e.nbytes)
                tr.alloc(g.nodes[f2[i][0]].output, st.nbytes)
            elif i not in f2_soft:          # (the statistics stand for P)
                tr.alloc(n.output, out.size * esz[n.output])
            per_step[i] = tr.total()
        for t in list(tr.live):
            if isinstance(t, str) and last.get(t, -1) <= i:
                tr.free(t)
        i += 1
    return {o: env[o] for o in g.outputs}, per_step


def _tracked_region(g, r, env, tr, per_step, esz, wset, last, mirror, contiguity, crange=None, f2=None,
                    f2_soft=()):
    from .memory import contiguity_cost
    E, n = r.extent, r.n
    L = -(-E // n)
    hs = set(r.hoisted)
    produced = {g.nodes[k].output for k in range(r.start, r.end + 1)}
    ydims = dict(r.yc)
    for k in r.hoisted:                         # hoisted nodes run once, before the loop
        nd = g.nodes[k]
        env[nd.output] = _eval(g, k, [env[t] for t in nd.inputs], None, mirror)
        tr.alloc(nd.output, env[nd.output].size * esz[nd.output])
    for y, d in r.yc:                           # Y^c allocated full at region start
        env[y] = np.zeros(g.tensors[y].shape)
        tr.alloc(y, env[y].size * esz[y])
    ctg = 0
    if contiguity:
        for t, d in list(r.xc) + list(r.yc):
            tm = g.tensors[t]
            ctg += contiguity_cost(tm.shape, tm.esize, d, n)
    f2 = f2 or {}
    ilast = {}                                  # last in-region (per-chunk) use
    for k in range(r.start, r.end + 1):
        if k not in hs:
            for t in g.nodes[k].inputs:
                if t in produced:
                    ilast[t] = k
    for k, (sm, pv) in f2.items():              # fused chain: the PV reads the e-tiles
        if r.start <= k <= r.end:
            ilast[g.nodes[k].output] = max(ilast.get(g.nodes[k].output, pv), pv)
    c0, c1 = crange if crange is not None else (0, n)
    for c in range(c0, c1):
        off = c * L
        ln = min(L, E - off)
        if ln <= 0:
            break
        if ctg:
            tr.alloc(("ctg",), ctg)
        local = {}

        def alloc_local(k, out):
            t = g.nodes[k].output
            if k in f2:                         # fused chain: e-tiles + statistics (R25)
                e, st = _f2_buffers(out.shape)
                tr.alloc(("slice", t), e.nbytes)
                tr.alloc(("slice", g.nodes[f2[k][0]].output), st.nbytes)
            elif k not in f2_soft:              # (the statistics stand for P)
                tr.alloc(("slice", t), out.size * esz[t])

        for k in range(r.start, r.end + 1):
            if k in hs:                         # nothing runs here per chunk
                per_step[k] = max(per_step[k], tr.total())
                continue
            nd = g.nodes[k]
            if nd.output not in r.dims:
                # off the flow, not hoisted (graph optimisation off): the node is
                # recomputed whole in every chunk from whole inputs; its output is a
                # full-size interior tensor (Eq. 2 term (v), R6)
                out = _eval(g, k, [local[t] if t in local else env[t] for t in nd.inputs], None, mirror)
                local[nd.output] = out
                alloc_local(k, out)
                per_step[k] = max(per_step[k], tr.total())
                for t in set(nd.inputs) | {nd.output}:
                    if t in local and ilast.get(t, k) <= k:
                        del local[t]
                        tr.free(("slice", t))
                continue
            res = ops.propagate(nd.kind, nd.attrs, [g.tensors[t].shape for t in nd.inputs],
                                g.tensors[nd.output].shape, r.dims[nd.output])
            vals = []
            for t, rr in zip(nd.inputs, res):
                if t in local:
                    vals.append(local[t])
                elif isinstance(rr, int) and t not in produced:
                    vals.append(_slice(env[t], rr, off, ln))
                else:
                    vals.append(env[t])
            out = _eval(g, k, vals, {"dim": r.dims[nd.output], "offset": off}, mirror)
            if nd.output in ydims:
                _slice(env[nd.output], ydims[nd.output], off, ln)[...] = out
                if nd.output in ilast:
                    local[nd.output] = out
            else:
                local[nd.output] = out
                alloc_local(k, out)
            per_step[k] = max(per_step[k], tr.total())
            for t in set(nd.inputs) | {nd.output}:
                if t in local and ilast.get(t, k) <= k:
                    del local[t]
                    tr.free(("slice", t))
        for t in list(local):
            tr.free(("slice", t))
        if ctg:
            tr.free(("ctg",))


def run_chunked(g: Graph, values: dict, regions, mirror: bool = False, chunk_ranges=None) -> dict:
    outs, _ = tracked_run(g, values, regions, mirror, chunk_ranges=chunk_ranges)
    return outs
