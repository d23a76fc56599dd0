"""Chunk plan structures and the canonical plan document (oracle; test infrastructure only).

A plan is S = [s_1, ..., s_l] (Eq. 11).  Each committed step is one
chunk region (Eq. 3): a contiguous topological interval of nodes,
the per-tensor chunk dims of its flow (Eq. 4), X^c / X^nc / Y^c, the hoisted
nodes of the graph optimisation and n, the number of chunks
("chunk size"; reading R1).

Document (schema 1):
    autochunk-plan 1
    graph <name>
    budget <int>
    baseline <int>
    peak <int>
    status <feasible|infeasible>
    cost <%.17g>
    region s=<node> e=<node> n=<n> ext=<E> len=<ceil(E/n)> hoist=<ids|-> flow=<t:d,...>
           xc=<t:d,...|-> xnc=<t,...|-> yc=<t:d,...> n_node=<i> n_flop=<i>
           density=<g> stride=<i> macro=<g> micro=<g> total=<g>      (one line)
A user-fixed plan may give only `region s=<node> e=<node> n=<n> dims=<d,...>`.
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class Cost:
    n_node: int = 0
    n_flop: int = 0
    density: float = 0.0
    stride: int = 0
    macro: float = 0.0
    micro: float = 0.0
    total: float = 0.0


@dataclass
class Region:
    start: int
    end: int
    dims: dict                       # tensor id -> chunk dim, BFS discovery order
    hoisted: list = field(default_factory=list)   # node indices executed once
    xc: list = field(default_factory=list)        # [(tid, dim)]
    xnc: list = field(default_factory=list)       # [tid]
    yc: list = field(default_factory=list)        # [(tid, dim)]
    extent: int = 0
    n: int = 1
    cost: Cost = field(default_factory=Cost)
    assign: tuple = ()               # output-dim assignment it was searched with

    @property
    def chunk_len(self) -> int:
        return -(-self.extent // self.n)

    def with_n(self, n: int) -> "Region":
        r = Region(self.start, self.end, dict(self.dims), list(self.hoisted), list(self.xc),
                   list(self.xnc), list(self.yc), self.extent, n, self.cost, self.assign)
        return r

    def signature(self):
        return (self.start, self.end, tuple(self.hoisted), tuple(self.dims.items()))


@dataclass
class Plan:
    regions: list = field(default_factory=list)
    budget: int = 0
    baseline: int = 0
    peak: int = 0
    feasible: bool = True
    cost: float = 0.0
    graph_name: str = "g"


def _g(x: float) -> str:
    return "%.17g" % x


def serialize(plan: Plan, g) -> str:
    names = [n.id for n in g.nodes]
    lines = ["autochunk-plan 1", f"graph {g.name}", f"budget {plan.budget}",
             f"baseline {plan.baseline}", f"peak {plan.peak}",
             f"status {'feasible' if plan.feasible else 'infeasible'}", f"cost {_g(plan.cost)}"]
    for r in plan.regions:
        hoist = ",".join(names[i] for i in r.hoisted) or "-"
        flow = ",".join(f"{t}:{d}" for t, d in r.dims.items())
        xc = ",".join(f"{t}:{d}" for t, d in r.xc) or "-"
        xnc = ",".join(r.xnc) or "-"
        yc = ",".join(f"{t}:{d}" for t, d in r.yc)
        c = r.cost
        lines.append(
            f"region s={names[r.start]} e={names[r.end]} n={r.n} ext={r.extent} len={r.chunk_len} "
            f"hoist={hoist} flow={flow} xc={xc} xnc={xnc} yc={yc} n_node={c.n_node} "
            f"n_flop={c.n_flop} density={_g(c.density)} stride={c.stride} macro={_g(c.macro)} "
            f"micro={_g(c.micro)} total={_g(c.total)}")
    return "\n".join(lines) + "\n"


def parse_user_regions(text: str):
    """Parse the region records of a plan document: [(start_id, end_id, n, dims|None[, hoist])].
    Only s/e/n/dims/opt are read; the library re-derives flows (SURVEY §8(b) ac_plan_parse)."""
    lines = [ln.strip() for ln in text.splitlines() if ln.strip()]
    if not lines or lines[0] != "autochunk-plan 1":
        raise ValueError("plan parse error: missing header")
    out = []
    for ln in lines[1:]:
        f = ln.split()
        if f[0] != "region":
            continue
        kv = dict(x.split("=", 1) for x in f[1:])
        dims = None
        if "dims" in kv:
            dims = tuple(int(x) for x in kv["dims"].split(","))
        elif "yc" in kv:
            dims = tuple(int(x.rsplit(":", 1)[1]) for x in kv["yc"].split(","))
        # opt=0: graph optimisation (hoisting) off for this region (Table 1's
        # "No graph optimization" on a user-fixed region)
        out.append((kv["s"], kv["e"], int(kv["n"]), dims) + ((False,) if kv.get("opt") == "0" else ()))
    return out
