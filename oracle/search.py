"""Chunk search of the oracle (test infrastructure only): Algorithm 1.

For every region from GetNodePairs(G, n_p) (contiguous node intervals that
contain the peak node, length <= window k) and every
assignment of chunk dims to the region outputs ("check every chunk dim"),
a bottom-up BFS walks from the outputs toward the region inputs, mapping the
chunk dim through each node (chunk flow, Eq. 4) and checking
  Rules 1&2 (Eq. 5): no BREAK on the flow and some inputs chunkable,
  Rule 3   (Eq. 6): every output traces back to a chunked input,
  Rule 4   (Eq. 7): every node / tensor gets exactly one chunk setting.
Before the BFS a two-stage filter cheaply checks that some flow path
exists between each output and the inputs.  Afterwards the graph
optimisation hoists nodes that are not on the flow and shrinks
the region to the flow nodes.  Candidates whose best-case memory (largest n)
cannot lower the bytes at the peak step n_p are dropped (DESIGN.md
reading R13: judged at n_p, not globally, so tied peaks such as AlphaFold's
row and column attention are chunked one pass at a time).
"""
from __future__ import annotations

import itertools

from . import ops
from .graph import Graph
from .memory import estimate_with_plan, region_io
from .plan import Region


def get_node_pairs(n_nodes: int, p: int, k: int, sources=()):
    """All [s, e] with s <= p <= e, e - s + 1 <= k, containing no input/weight
    node (index in `sources`); ordered by (length, start)."""
    if k < 1:
        raise ValueError("window k must be >= 1")
    src = set(sources)
    out = []
    for length in range(1, k + 1):
        for s in range(max(0, p - length + 1), p + 1):
            e = s + length - 1
            if e >= n_nodes or any(j in src for j in range(s, e + 1)):
                continue
            out.append((s, e))
    return out


def propagate_node(g: Graph, i: int, d: int):
    n = g.nodes[i]
    return ops.propagate(n.kind, n.attrs, [g.tensors[t].shape for t in n.inputs],
                         g.tensors[n.output].shape, d)


def two_stage_filter(g: Graph, s: int, e: int, outs, assign, prod) -> bool:
    """Stage 1 of P:201: does some dim-compatible path lead from every output to a
    chunkable region input?  Ignores Rule 4; no false negatives."""
    wset = set(g.weights)
    for y, d in zip(outs, assign):
        seen = set()
        stack = [(y, d)]
        ok = False
        while stack and not ok:
            t, dd = stack.pop()
            if (t, dd) in seen:
                continue
            seen.add((t, dd))
            pi = prod[t]
            if not (s <= pi <= e):
                if t not in wset:
                    ok = True
                continue
            for u, r in zip(g.nodes[pi].inputs, propagate_node(g, pi, dd)):
                if isinstance(r, int):
                    stack.append((u, r))
        if not ok:
            return False
    return True


def bfs_region(g: Graph, s: int, e: int, ins, outs, assign, prod):
    """Stage 2: bottom-up BFS (Alg. 1 lines 'BottomUpBFS' / 'satisfy Equ. [5;6;7]').
    Returns (dims, flow_nodes) or None if a rule is violated."""
    wset = set(g.weights)
    produced = {g.nodes[i].output for i in range(s, e + 1)}
    dims = {}
    ext = None
    for y, d in zip(outs, assign):
        E = g.tensors[y].shape[d]
        if ext is None:
            ext = E
        elif E != ext:
            return None
        dims[y] = d
    if ext is None or ext < 2:
        return None
    whole = set()
    pending = {prod[y] for y in outs}
    flow_nodes = set()
    while pending:
        i = max(pending)                 # producers in descending topological index
        pending.discard(i)
        flow_nodes.add(i)
        node = g.nodes[i]
        res = propagate_node(g, i, dims[node.output])
        for u, r in zip(node.inputs, res):
            if r == ops.BREAK:
                return None              # Rules 1&2
            if r == ops.NC:
                if u in produced:
                    if u in dims:
                        return None      # Rule 4: chunked and needed whole
                    whole.add(u)
                continue
            if u in wset:
                return None              # weights are never chunked (X^nc leaves)
            if u in dims:
                if dims[u] != r:
                    return None          # Rule 4
                continue
            if u in whole:
                return None
            if g.tensors[u].shape[r] != ext:
                return None
            dims[u] = r
            if u in produced:
                pending.add(prod[u])
    # nodes off the flow must not consume chunked interior tensors
    for i in range(s, e + 1):
        if i in flow_nodes:
            continue
        for u in g.nodes[i].inputs:
            if u in produced and u in dims:
                return None
    # Rule 3: every output traces to a chunked region input
    chunked_inputs = {t for t in ins if t in dims}
    if not chunked_inputs:
        return None
    for y in outs:
        seen = set()
        stack = [y]
        ok = False
        while stack and not ok:
            t = stack.pop()
            if t in seen:
                continue
            seen.add(t)
            if t in chunked_inputs:
                ok = True
                break
            if t not in produced:
                continue
            pi = prod[t]
            for u, r in zip(g.nodes[pi].inputs, propagate_node(g, pi, dims[t])):
                if isinstance(r, int):
                    stack.append(u)
        if not ok:
            return None
    return dims, flow_nodes


def optimize_region(g: Graph, s: int, e: int, dims, flow_nodes, hoist: bool = True):
    """Graph optimisation: hoist the nodes not on the flow (they do not
    depend on chunked tensors) and shrink the interval to the flow nodes."""
    if not hoist:
        return s, e, []
    s2, e2 = min(flow_nodes), max(flow_nodes)
    hoisted = [i for i in range(s2, e2 + 1) if i not in flow_nodes]
    return s2, e2, hoisted


def make_region(g: Graph, s, e, dims, hoisted, assign, cons=None) -> Region:
    ins, outs = region_io(g, s, e, cons)
    hout = {g.nodes[i].output for i in hoisted}
    xc = [(t, dims[t]) for t in ins if t in dims]
    xnc = [t for t in ins if t not in dims]
    yc = [(t, dims[t]) for t in outs if t not in hout]   # hoisted outputs are computed once
    # keep only the flow entries that belong to this (possibly shrunk) region
    keep = set(ins) | {g.nodes[i].output for i in range(s, e + 1)}
    fl = {t: d for t, d in dims.items() if t in keep and t not in hout}
    ext = g.tensors[outs[0]].shape[yc[0][1]]
    return Region(s, e, fl, list(hoisted), xc, xnc, yc, ext, 1, assign=tuple(assign))


def candidate_for(g: Graph, s: int, e: int, assign, hoist=True, prod=None, cons=None):
    """Full search for one (region, assignment); None if illegal."""
    prod = prod or g.producer_index()
    cons = cons or g.consumers()
    ins, outs = region_io(g, s, e, cons)
    if not outs or len(assign) != len(outs):
        return None
    r = bfs_region(g, s, e, ins, outs, assign, prod)
    if r is None:
        return None
    dims, fnodes = r
    s2, e2, hoisted = optimize_region(g, s, e, dims, fnodes, hoist)
    return make_region(g, s2, e2, dims, hoisted, assign, cons)


def ladder(E: int, cap: int = 4096):
    """Chunk-count ladder: powers of two < E up to cap, plus E itself if E <= cap
    ("powers of two up to 4096", clamped to the extent S:344)."""
    out = []
    v = 2
    while v <= cap and v < E:
        out.append(v)
        v *= 2
    if E <= cap and E >= 2:
        out.append(E)
    return out


class SearchStats:
    def __init__(self):
        self.filtered_in = 0
        self.filtered_total = 0


def search(g: Graph, n_p: int, plan_regions, cur_peak: int, window: int = 32,
           hoist: bool = True, contiguity: bool = False, stats: SearchStats = None,
           allowed_dims=None):
    """Algorithm 1: all legal chunk candidates around the peak node n_p that do not
    overlap committed regions.  Ordered by (region length, start, assignment)."""
    prod = g.producer_index()
    cons = g.consumers()
    sources = [i for i, n in enumerate(g.nodes) if n.kind in ("input", "weight")]
    taken = [(r.start, r.end) for r in plan_regions]
    out = []
    seen = set()
    for s, e in get_node_pairs(len(g.nodes), n_p, window, sources):
        if any(not (e < a or s > b) for a, b in taken):
            continue
        ins, outs = region_io(g, s, e, cons)
        if not outs:
            continue
        for assign in itertools.product(*[range(len(g.tensors[y].shape)) for y in outs]):
            if allowed_dims is not None and any(d not in allowed_dims for d in assign):
                continue
            if stats is not None:
                stats.filtered_total += 1
            if not two_stage_filter(g, s, e, outs, assign, prod):
                continue
            if stats is not None:
                stats.filtered_in += 1
            res = bfs_region(g, s, e, ins, outs, assign, prod)
            if res is None:
                continue
            dims, fnodes = res
            s2, e2, hoisted = optimize_region(g, s, e, dims, fnodes, hoist)
            if any(not (e2 < a or s2 > b) for a, b in taken):
                continue
            reg = make_region(g, s2, e2, dims, hoisted, assign, cons)
            sig = reg.signature()
            if sig in seen:
                continue
            seen.add(sig)
            lad = ladder(reg.extent)
            if not lad:
                continue
            best = estimate_with_plan(g, list(plan_regions) + [reg.with_n(lad[-1])], contiguity)
            if best.per_step[n_p] >= cur_peak:   # must lower the peak step
                continue
            out.append(reg)
    return out
