"""Python binding of include/ac.h with the same names (marshalling only).

    g = graph_block("transformer", N, d, h, f, causal, "bf16")   # ac_graph_block
    g = graph_parse(text)                                          # ac_graph_parse
    prof, per_step = estimate_memory(g, plan=None)                 # ac_estimate_memory
    plan = ac_plan(g, budget)                                      # ac_plan
    plan = plan_parse(g, text)                                     # ac_plan_parse
    ex = Exec(plan, workspace_tensor)                              # ac_exec_create
    ex.run(inputs, outputs, stream)                                # ac_run
"""
from __future__ import annotations

import ctypes as C

from . import _lib as L
from ._lib import check, lib

DTYPES = {"f32": L.AC_F32, "bf16": L.AC_BF16, "f64": L.AC_F64}
KINDS = {"transformer": L.AC_BLOCK_TRANSFORMER, "attn_only": L.AC_BLOCK_ATTN_ONLY,
         "tri_attn_pair": L.AC_BLOCK_TRI_ATTN_PAIR}


class Graph:
    def __init__(self, handle):
        self._h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().ac_graph_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def serialize(self) -> str:
        n = C.c_size_t()
        check(lib().ac_graph_serialize(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(lib().ac_graph_serialize(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    @property
    def num_nodes(self) -> int:
        return lib().ac_graph_num_nodes(self._h)


def graph_parse(text: str) -> Graph:
    b = text.encode()
    h = C.c_void_p()
    check(lib().ac_graph_parse(b, len(b), C.byref(h)))
    return Graph(h.value)


def graph_block(kind: str, N: int, d: int, h: int, f: int = 0, causal: bool = False, dtype: str = "bf16",
                ln_eps: float = 1e-5, name: str | None = None) -> Graph:
    desc = L.BlockDesc(KINDS[kind], N, d, h, f, int(causal), DTYPES[dtype], ln_eps,
                       name.encode() if name else None)
    out = C.c_void_p()
    check(lib().ac_graph_block(C.byref(desc), C.byref(out)))
    return Graph(out.value)


class Plan:
    def __init__(self, handle, graph: Graph, status: int = L.AC_OK):
        self._h = C.c_void_p(handle)
        self.graph = graph          # keeps the graph alive
        self.status = status

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().ac_plan_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def feasible(self) -> bool:
        return self.status == L.AC_OK

    def serialize(self) -> str:
        n = C.c_size_t()
        check(lib().ac_plan_serialize(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(lib().ac_plan_serialize(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    @property
    def num_regions(self) -> int:
        return lib().ac_plan_num_regions(self._h)

    def workspace_bytes(self, rank: int = 0, world: int = 1) -> int:
        v = lib().ac_plan_workspace_bytes(self._h, rank, world)
        if v < 0:
            raise L.ACError(L.AC_ERR_PLAN, lib().ac_last_error().decode())
        return v


def cost_params(**kw) -> L.CostParams:
    p = L.CostParams()
    lib().ac_cost_params_default(C.byref(p))
    for k, v in kw.items():
        setattr(p, "lambda_" if k in ("lam", "lambda") else k, v)
    return p


def ac_plan(g: Graph, budget: int, params: L.CostParams | None = None) -> Plan:
    """ac_plan: returns the plan; plan.status is AC_ERR_BUDGET for a best-effort plan."""
    out = C.c_void_p()
    st = lib().ac_plan(g.handle, int(budget), C.byref(params) if params is not None else None, C.byref(out))
    if st not in (L.AC_OK, L.AC_ERR_BUDGET):
        check(st)
    return Plan(out.value, g, st)


def plan_parse(g: Graph, text: str) -> Plan:
    b = text.encode()
    out = C.c_void_p()
    check(lib().ac_plan_parse(g.handle, b, len(b), C.byref(out)))
    return Plan(out.value, g)


def estimate_memory(g: Graph, plan: Plan | None = None):
    prof = L.MemProfile()
    n = g.num_nodes
    arr = (C.c_int64 * max(n, 1))()
    check(lib().ac_estimate_memory(g.handle, plan.handle if plan is not None else None, C.byref(prof), arr))
    return prof, list(arr)[:n]
