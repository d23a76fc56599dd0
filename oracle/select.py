"""Chunk selection of the oracle (test infrastructure only).

* macro cost  Eq. 8:  L_macro = alpha*N_node + beta*N_flop
* micro cost  Eq. 9:  L_micro = gamma*N_density + lambda*N_stride
* total       Eq. 10: L = L_macro + L_micro
* selection   Eq. 11: min sum_i L(s_i)  s.t. peak < budget, by dynamic programming
  with beam search over passes; each pass re-estimates memory, finds the new
  peak node and runs the chunk search (the pass loop of P:153).
Readings (R8-R12): gamma < 0, lambda > 0 (SPEC defaults);
optional normalised features (R27, off by default, SURVEY c.2 #10): N_node / S_g,
N_flop / F_g, N_density / (F_g / S_g), N_stride / numel(largest flow tensor), with
S_g the graph's compute nodes and F_g their FLOPs, so that O(1) weights compare
terms of the same scale (the paper tunes its weights);
N_node / N_flop count the nodes executed per chunk (hoisted nodes run once);
N_stride is the row-major stride of the chunk dim of the largest flow tensor
(first in BFS order on ties); DP key = sorted set of region intervals; beam 4;
16 passes; chunk size = smallest n on the ladder whose region fits.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .graph import Graph
from .memory import estimate_with_plan, profile
from .plan import Cost, Plan, Region
from .search import SearchStats, ladder, search


@dataclass
class CostParams:
    alpha: float = 1.0
    beta: float = 1e-9
    gamma: float = -1e-5
    lam: float = 0.01
    beam: int = 4
    window: int = 32
    max_passes: int = 16
    hoist: bool = True
    contiguity: bool = False
    use_node: bool = True
    use_flop: bool = True
    use_density: bool = True
    use_stride: bool = True
    allowed_dims: tuple = None
    normalize: bool = False


def macro_cost(n_node: int, n_flop: int, p: CostParams) -> float:
    a = p.alpha if p.use_node else 0.0
    b = p.beta if p.use_flop else 0.0
    return a * float(n_node) + b * float(n_flop)


def micro_cost(density: float, stride: int, p: CostParams) -> float:
    c = p.gamma if p.use_density else 0.0
    l = p.lam if p.use_stride else 0.0
    return c * density + l * float(stride)


def graph_scales(g: Graph):
    """(S_g, F_g) of the normalised features: compute nodes and their FLOPs (>= 1)."""
    nodes = [i for i, n in enumerate(g.nodes) if n.kind not in ("input", "weight")]
    return max(len(nodes), 1), max(sum(g.flops(i) for i in nodes), 1)


def region_cost(g: Graph, r: Region, p: CostParams) -> Cost:
    hs = set(r.hoisted)
    nodes = [i for i in range(r.start, r.end + 1) if i not in hs]
    n_node = len(nodes)
    n_flop = sum(g.flops(i) for i in nodes)
    density = float(n_flop) / float(n_node)
    big, bigb = None, -1
    for t, d in r.dims.items():
        b = g.tensors[t].bytes
        if b > bigb:
            big, bigb = t, b
    stride = g.tensors[big].strides[r.dims[big]]
    if p.normalize:
        sg, fg = graph_scales(g)
        numel = 1
        for e in g.tensors[big].shape:
            numel *= e
        a = p.alpha if p.use_node else 0.0
        b = p.beta if p.use_flop else 0.0
        c = p.gamma if p.use_density else 0.0
        lm = p.lam if p.use_stride else 0.0
        ma = a * (float(n_node) / float(sg)) + b * (float(n_flop) / float(fg))
        mi = c * (density / (float(fg) / float(sg))) + lm * (float(stride) / float(numel))
        return Cost(n_node, n_flop, density, stride, ma, mi, ma + mi)
    ma = macro_cost(n_node, n_flop, p)
    mi = micro_cost(density, stride, p)
    return Cost(n_node, n_flop, density, stride, ma, mi, ma + mi)


def choose_chunk_size(g: Graph, regions, cand: Region, budget: int, p: CostParams):
    """Smallest n on the ladder whose region steps fit under the budget
    (pro-rata target).  Returns (n, fits)."""
    lad = ladder(cand.extent)
    for n in lad:
        est = estimate_with_plan(g, list(regions) + [cand.with_n(n)], p.contiguity)
        if max(est.per_step[cand.start: cand.end + 1]) < budget:
            return n, True
    return lad[-1], False


@dataclass
class _State:
    regions: list = field(default_factory=list)
    cost: float = 0.0

    @property
    def key(self):
        return tuple(sorted((r.start, r.end) for r in self.regions))


def select(g: Graph, budget: int, p: CostParams = None, stats: SearchStats = None):
    """Multi-pass DP + beam (Eq. 11).  Returns a Plan; plan.feasible is False when
    no state met the budget (best-effort plan = lowest peak in the final beam)."""
    p = p or CostParams()
    base = profile(g)
    plan = Plan(budget=budget, baseline=base.peak_bytes, graph_name=g.name)
    if base.peak_bytes < budget:
        plan.peak = base.peak_bytes
        return plan
    beam = [_State()]
    for npass in range(p.max_passes + 1):
        feas = []
        for st in beam:
            est = estimate_with_plan(g, st.regions, p.contiguity)
            if est.peak_bytes < budget:
                feas.append((st.cost, st.key, st, est.peak_bytes))
        if feas:
            feas.sort(key=lambda x: (x[0], x[1]))
            c, _, st, pk = feas[0]
            return Plan(list(st.regions), budget, base.peak_bytes, pk, True, c, g.name)
        if npass == p.max_passes:
            break
        per_state = []
        any_fit = False
        for st in beam:
            est = estimate_with_plan(g, st.regions, p.contiguity)
            cands = search(g, est.peak_step, st.regions, est.peak_bytes, p.window, p.hoist,
                           p.contiguity, stats, p.allowed_dims)
            scored = []
            for c in cands:
                n, fits = choose_chunk_size(g, st.regions, c, budget, p)
                cc = c.with_n(n)
                cc.cost = region_cost(g, cc, p)
                scored.append((cc, fits))
                any_fit = any_fit or fits
            per_state.append((st, scored))
        ext = {}
        for st, scored in per_state:
            for cc, fits in scored:
                if any_fit and not fits:
                    continue
                new = _State(st.regions + [cc], st.cost + cc.cost.total)
                k = new.key
                if k not in ext or new.cost < ext[k].cost:
                    ext[k] = new
        if not ext:
            break
        beam = sorted(ext.values(), key=lambda s: (s.cost, s.key))[: p.beam]
    best = None
    for st in beam:
        est = estimate_with_plan(g, st.regions, p.contiguity)
        k = (est.peak_bytes, st.cost, st.key)
        if best is None or k < best[0]:
            best = (k, st, est.peak_bytes)
    _, st, pk = best
    return Plan(list(st.regions), budget, base.peak_bytes, pk, False, st.cost, g.name)


def exhaustive(g: Graph, budget: int, p: CostParams, max_passes: int = 3):
    """Brute force for AC-6: enumerate every candidate sequence level by
    level (same extension rule as select, no dedupe, no pruning) and return the
    minimum cost among feasible plans at the first level that has any."""
    base = profile(g)
    if base.peak_bytes < budget:
        return 0.0, []
    level = [([], 0.0)]
    for _ in range(max_passes):
        nxt = []
        per = []
        any_fit = False
        for regs, cost in level:
            est = estimate_with_plan(g, regs, p.contiguity)
            cands = search(g, est.peak_step, regs, est.peak_bytes, p.window, p.hoist, p.contiguity,
                           None, p.allowed_dims)
            sc = []
            for c in cands:
                n, fits = choose_chunk_size(g, regs, c, budget, p)
                cc = c.with_n(n)
                cc.cost = region_cost(g, cc, p)
                sc.append((cc, fits))
                any_fit = any_fit or fits
            per.append((regs, cost, sc))
        for regs, cost, sc in per:
            for cc, fits in sc:
                if any_fit and not fits:
                    continue
                nxt.append((regs + [cc], cost + cc.cost.total))
        if not nxt:
            return None
        feas = [(c, tuple(sorted((r.start, r.end) for r in rg)), rg) for rg, c in nxt
                if estimate_with_plan(g, rg, p.contiguity).peak_bytes < budget]
        if feas:
            feas.sort(key=lambda x: (x[0], x[1]))
            return feas[0][0], feas[0][2]
        level = nxt
    return None


def user_plan(g: Graph, specs, p: CostParams = None) -> Plan:
    """A user-fixed plan (ac_plan_parse): specs = [(start_node_id, end_node_id, n,
    dims[, hoist])].  Flows, X^c / X^nc / Y^c and hoisting are derived as the search does."""
    from .search import candidate_for
    p = p or CostParams()
    names = [n.id for n in g.nodes]
    regions = []
    for spec in specs:
        s_id, e_id, n, dims = spec[:4]
        hoist = spec[4] if len(spec) > 4 else True     # False: opt=0, no graph optimisation
        s, e = names.index(s_id), names.index(e_id)
        if any(g.nodes[i].kind in ("input", "weight") for i in range(s, e + 1)):
            raise ValueError("illegal region: contains an input/weight node")
        r = candidate_for(g, s, e, tuple(dims), hoist=hoist)
        if r is None:
            raise ValueError("illegal region: no legal chunk flow for these dims")
        if not 1 <= n <= r.extent:
            raise ValueError("chunk count n outside [1, extent]")
        r = r.with_n(n)
        for o in regions:
            if not (r.end < o.start or r.start > o.end):
                raise ValueError("overlapping regions")
        r.cost = region_cost(g, r, p)
        regions.append(r)
    cost = 0.0
    for r in regions:
        cost = cost + r.cost.total
    return Plan(regions, 0, profile(g).peak_bytes, estimate_with_plan(g, regions).peak_bytes, True, cost, g.name)
