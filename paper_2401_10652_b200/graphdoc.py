"""Read-only view of a graph document (the text ac_graph_serialize returns).

Host-side plumbing for the bench and the examples: tensor ids, dtypes, shapes,
weight roles and the node list, so callers can allocate and bind buffers for
ac_run.  No arithmetic of the method lives here.
"""
from __future__ import annotations

from dataclasses import dataclass, field

ESIZE = {"f32": 4, "bf16": 2, "f64": 8}


@dataclass
class Doc:
    name: str = ""
    tensors: dict = field(default_factory=dict)   # id -> (dtype, shape)
    inputs: list = field(default_factory=list)
    weights: list = field(default_factory=list)   # (id, role, fan_in)
    nodes: list = field(default_factory=list)     # (id, kind, inputs, output, attrs{str: str})
    outputs: list = field(default_factory=list)
    order: list = field(default_factory=list)     # input/weight ids in declaration order

    def nbytes(self, tid: str) -> int:
        dt, shp = self.tensors[tid]
        n = ESIZE[dt]
        for s in shp:
            n *= s
        return n

    def input_specs(self):
        """(tid, kind, dtype, shape, role, fan_in) in declaration order (synth.make_inputs)."""
        w = {t: (r, f) for t, r, f in self.weights}
        out = []
        for t in self.order:
            dt, shp = self.tensors[t]
            if t in w:
                out.append((t, "weight", dt, shp, w[t][0], w[t][1]))
            else:
                out.append((t, "input", dt, shp, "act", 0))
        return out

    def node(self, nid: str):
        return next(n for n in self.nodes if n[0] == nid)


def parse(text: str) -> Doc:
    d = Doc()
    for ln in text.splitlines():
        f = ln.split()
        if not f:
            continue
        if f[0] == "name":
            d.name = f[1]
        elif f[0] == "tensor":
            d.tensors[f[1]] = (f[2], tuple(int(x) for x in f[3].split(",")))
        elif f[0] == "input":
            d.inputs.append(f[1])
            d.order.append(f[1])
        elif f[0] == "weight":
            d.weights.append((f[1], f[2], int(f[3])))
            d.order.append(f[1])
        elif f[0] == "node":
            attrs = dict(kv.split("=", 1) for kv in f[5:])
            d.nodes.append((f[1], f[2], f[3].split(",") if f[3] else [], f[4], attrs))
        elif f[0] == "output":
            d.outputs.append(f[1])
    return d
