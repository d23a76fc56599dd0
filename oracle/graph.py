"""Graph IR + text document for the oracle (test infrastructure only).

The graph is the paper's "computational graph G" (Alg. 1 input) at
kernel granularity: nodes are kept in one topological list;
`input` / `weight` nodes come first and execution step s = node s
(reading R4).

Document (schema version 1, one record per line, canonical order):
    autochunk-graph 1
    name <name>
    tensor <id> <dtype> <d0,d1,...>
    input <tensor-id>
    weight <tensor-id> <role> <fan_in>
    node <id> <kind> <in1,in2,...> <out> [key=value ...]   (keys sorted)
    output <tensor-id>
Floats are printed with %.17g; int lists comma-separated; slice ranges s:e,...
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import ops

DTYPE_SIZE = {"f32": 4, "f64": 8, "bf16": 2}


class GraphError(ValueError):
    pass


@dataclass
class TensorMeta:
    id: str
    dtype: str
    shape: tuple

    @property
    def esize(self) -> int:
        return DTYPE_SIZE[self.dtype]

    @property
    def bytes(self) -> int:
        return ops.prod(self.shape) * self.esize

    @property
    def strides(self) -> tuple:
        st = [1] * len(self.shape)
        for i in range(len(self.shape) - 2, -1, -1):
            st[i] = st[i + 1] * self.shape[i + 1]
        return tuple(st)


@dataclass
class Node:
    id: str
    kind: str
    inputs: list
    output: str
    attrs: dict = field(default_factory=dict)


@dataclass
class Graph:
    name: str = "g"
    tensors: dict = field(default_factory=dict)     # id -> TensorMeta (declaration order)
    nodes: list = field(default_factory=list)
    inputs: list = field(default_factory=list)
    weights: list = field(default_factory=list)
    weight_info: dict = field(default_factory=dict)  # id -> (role, fan_in)
    outputs: list = field(default_factory=list)
    input_info: dict = field(default_factory=dict)   # id -> role ("act")

    # ------------------------------------------------------------ helpers
    def producer_index(self) -> dict:
        return {n.output: i for i, n in enumerate(self.nodes)}

    def consumers(self) -> dict:
        c = {t: [] for t in self.tensors}
        for i, n in enumerate(self.nodes):
            for t in n.inputs:
                if i not in c[t]:
                    c[t].append(i)
        return c

    def flops(self, i: int) -> int:
        n = self.nodes[i]
        return ops.flops(n.kind, n.attrs, [self.tensors[t].shape for t in n.inputs],
                         self.tensors[n.output].shape)

    def input_specs(self):
        """(tid, kind, dtype, shape, role, fan_in) in declaration order, for synth."""
        out = []
        for n in self.nodes:
            if n.kind == "input":
                t = self.tensors[n.output]
                out.append((t.id, "input", t.dtype, t.shape, "act", 0))
            elif n.kind == "weight":
                t = self.tensors[n.output]
                role, fan = self.weight_info[t.id]
                out.append((t.id, "weight", t.dtype, t.shape, role, fan))
        return out


# ------------------------------------------------------------------ builder
class Builder:
    """Small helper used by workloads.py and tests to assemble graphs."""

    def __init__(self, name="g", dtype="f32"):
        self.g = Graph(name=name)
        self.dtype = dtype
        self._n = 0

    def input(self, tid, shape, dtype=None):
        self.g.tensors[tid] = TensorMeta(tid, dtype or self.dtype, tuple(shape))
        self.g.inputs.append(tid)
        self.g.nodes.append(Node(tid, "input", [], tid, {}))
        return tid

    def weight(self, tid, shape, role="matrix", fan_in=None, dtype=None):
        self.g.tensors[tid] = TensorMeta(tid, dtype or self.dtype, tuple(shape))
        self.g.weights.append(tid)
        self.g.weight_info[tid] = (role, int(fan_in if fan_in is not None else shape[-1]))
        self.g.nodes.append(Node(tid, "weight", [], tid, {}))
        return tid

    def op(self, kind, inputs, _out, dtype=None, nid=None, **attrs):
        ins = [self.g.tensors[t].shape for t in inputs]
        shp = ops.shape(kind, attrs, ins)
        self.g.tensors[_out] = TensorMeta(_out, dtype or self.dtype, shp)
        self._n += 1
        self.g.nodes.append(Node(nid or f"n_{_out}", kind, list(inputs), _out, dict(attrs)))
        return _out

    def output(self, tid):
        self.g.outputs.append(tid)

    def build(self) -> Graph:
        validate(self.g)
        return self.g


# ------------------------------------------------------------------ document
def _fmt_attr(v, tag):
    if tag == "int":
        return str(int(v))
    if tag == "float":
        return "%.17g" % float(v)
    if tag == "ints":
        return ",".join(str(int(x)) for x in v)
    if tag == "ranges":
        return ",".join(f"{int(s)}:{int(e)}" for s, e in v)
    return str(v)


def _parse_attr(s, tag):
    if tag == "int":
        return int(s)
    if tag == "float":
        return float(s)
    if tag == "ints":
        return [int(x) for x in s.split(",")] if s else []
    if tag == "ranges":
        return [tuple(int(y) for y in x.split(":")) for x in s.split(",")]
    return s


def serialize(g: Graph) -> str:
    lines = ["autochunk-graph 1", f"name {g.name}"]
    for t in g.tensors.values():
        lines.append(f"tensor {t.id} {t.dtype} {','.join(str(s) for s in t.shape)}")
    for n in g.nodes:
        if n.kind == "input":
            lines.append(f"input {n.output}")
        elif n.kind == "weight":
            role, fan = g.weight_info[n.output]
            lines.append(f"weight {n.output} {role} {fan}")
        else:
            schema = ops.ATTR_SCHEMA.get(n.kind, {})
            at = " ".join(f"{k}={_fmt_attr(n.attrs[k], schema[k])}" for k in sorted(n.attrs))
            rec = f"node {n.id} {n.kind} {','.join(n.inputs)} {n.output}"
            lines.append(rec + (" " + at if at else ""))
    for o in g.outputs:
        lines.append(f"output {o}")
    return "\n".join(lines) + "\n"


def load_graph(text: str, infer: bool = True) -> Graph:
    """Parse a document (SPEC load_graph S:55-63), then infer shapes and validate."""
    g = Graph()
    declared = {}
    lines = [ln.strip() for ln in text.splitlines() if ln.strip() and not ln.strip().startswith("#")]
    if not lines or lines[0] != "autochunk-graph 1":
        raise GraphError("parse error: missing header 'autochunk-graph 1'")
    node_ids = set()
    for ln in lines[1:]:
        f = ln.split()
        rec = f[0]
        try:
            if rec == "name":
                g.name = f[1]
            elif rec == "tensor":
                tid, dt = f[1], f[2]
                if tid in declared:
                    raise GraphError(f"duplicate id {tid}")
                if dt not in DTYPE_SIZE:
                    raise GraphError(f"unknown dtype {dt}")
                shp = tuple(int(x) for x in f[3].split(",")) if len(f) > 3 and f[3] != "?" else None
                declared[tid] = (dt, shp)
            elif rec in ("input", "weight"):
                tid = f[1]
                if tid not in declared:
                    raise GraphError(f"unknown tensor id {tid}")
                dt, shp = declared[tid]
                if shp is None:
                    raise GraphError(f"{rec} {tid} needs a shape")
                if tid in g.tensors:
                    raise GraphError(f"duplicate id {tid}")
                g.tensors[tid] = TensorMeta(tid, dt, shp)
                if tid in node_ids:
                    raise GraphError(f"duplicate id {tid}")
                node_ids.add(tid)
                g.nodes.append(Node(tid, rec, [], tid, {}))
                if rec == "input":
                    g.inputs.append(tid)
                else:
                    g.weights.append(tid)
                    g.weight_info[tid] = (f[2], int(f[3]))
            elif rec == "node":
                nid, kind, ins, out = f[1], f[2], f[3], f[4]
                if kind not in ops.ALL_KINDS or kind in ops.SOURCE:
                    raise GraphError(f"unknown op kind {kind}")
                if nid in node_ids:
                    raise GraphError(f"duplicate id {nid}")
                node_ids.add(nid)
                schema = ops.ATTR_SCHEMA.get(kind, {})
                attrs = {}
                for kv in f[5:]:
                    k, v = kv.split("=", 1)
                    if k not in schema:
                        raise GraphError(f"unknown attribute {k} for {kind}")
                    attrs[k] = _parse_attr(v, schema[k])
                inputs = ins.split(",") if ins else []
                for t in inputs:
                    if t not in declared:
                        raise GraphError(f"unknown tensor id {t}")
                if out not in declared:
                    raise GraphError(f"unknown tensor id {out}")
                g.nodes.append(Node(nid, kind, inputs, out, attrs))
            elif rec == "output":
                if f[1] not in declared:
                    raise GraphError(f"unknown tensor id {f[1]}")
                g.outputs.append(f[1])
            else:
                raise GraphError(f"parse error: unknown record {rec}")
        except (IndexError, ValueError) as e:
            if isinstance(e, GraphError):
                raise
            raise GraphError(f"parse error in line {ln!r}: {e}") from None
    # register node outputs in declaration order of the tensor records
    produced = {n.output for n in g.nodes}
    ordered = {}
    for tid, (dt, shp) in declared.items():
        if tid in g.tensors:
            ordered[tid] = g.tensors[tid]
        elif tid in produced:
            ordered[tid] = TensorMeta(tid, dt, shp)
        else:
            raise GraphError(f"tensor {tid} is never produced")
    g.tensors = ordered
    _check_order(g)
    if infer:
        infer_shapes(g)
        validate(g)
    return g


def _check_order(g: Graph):
    prod_at = {}
    for i, n in enumerate(g.nodes):
        if n.output in prod_at:
            raise GraphError(f"tensor {n.output} produced twice")
        prod_at[n.output] = i
    for i, n in enumerate(g.nodes):
        for t in n.inputs:
            if t not in prod_at:
                raise GraphError(f"unknown tensor id {t}")
            if prod_at[t] >= i:
                if prod_at[t] == i:
                    raise GraphError("cycle detected")
                # consumer before producer: a cycle if the producer depends on us
                raise GraphError(f"order violation or cycle detected at {n.id}")


def infer_shapes(g: Graph) -> Graph:
    """SPEC infer_shapes: every output shape from its inputs; declared
    shapes must match."""
    for n in g.nodes:
        if n.kind in ops.SOURCE:
            continue
        try:
            shp = ops.shape(n.kind, n.attrs, [g.tensors[t].shape for t in n.inputs])
        except ValueError as e:
            raise GraphError(f"shape error at {n.id}: {e}") from None
        t = g.tensors[n.output]
        if t.shape is not None and tuple(t.shape) != tuple(shp):
            raise GraphError(f"shape mismatch at {n.id}: declared {t.shape} inferred {shp}")
        t.shape = tuple(shp)
    return g


def validate(g: Graph):
    errs = []
    seen = set()
    for i, n in enumerate(g.nodes):
        if n.kind not in ops.SOURCE:
            lo, hi = ops.ARITY[n.kind]
            if n.kind == "linear":
                lo = hi = ops.linear_arity(n.attrs)
            if not lo <= len(n.inputs) <= hi:
                errs.append(f"{n.id}: arity {len(n.inputs)}")
            for t in n.inputs:
                if t not in seen:
                    errs.append(f"{n.id}: order violation on {t}")
            if n.kind == "transpose":
                if sorted(n.attrs["perm"]) != list(range(len(g.tensors[n.inputs[0]].shape))):
                    errs.append(f"{n.id}: not a bijection")
        seen.add(n.output)
    if set(g.inputs) & set(g.weights):
        errs.append("inputs and weights overlap")
    for o in g.outputs:
        if o not in seen:
            errs.append(f"output {o} not produced")
    for t in g.tensors.values():
        if t.shape is None or any(int(s) < 1 for s in t.shape) or len(t.shape) == 0:
            errs.append(f"tensor {t.id}: bad shape {t.shape}")
    if errs:
        raise GraphError("; ".join(errs))


def graphs_equal(a: Graph, b: Graph) -> bool:
    return serialize(a) == serialize(b)
