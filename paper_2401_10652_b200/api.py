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
         "tri_attn_pair": L.AC_BLOCK_TRI_ATTN_PAIR, "transformer_fa": L.AC_BLOCK_TRANSFORMER_FA,
         "attn_only_fa": L.AC_BLOCK_ATTN_ONLY_FA, "evoformer_pair": L.AC_BLOCK_EVOFORMER_PAIR}


class Graph:
    def __init__(self, handle):
        self._h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            try:
                lib().ac_graph_free(self._h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
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
                ln_eps: float = 1e-5, name: str | None = None, layers: int = 1) -> Graph:
    desc = L.BlockDesc(KINDS[kind], N, d, h, f, int(causal), DTYPES[dtype], ln_eps,
                       name.encode() if name else None, int(layers))
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
            try:
                lib().ac_plan_free(self._h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
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

    def rank_chunks(self, region: int, rank: int, world: int):
        """ac_plan_rank_chunks: (chunks, n_eff, chunk_len, extent) - the chunks of
        `region` that `rank` of `world` runs."""
        cnt, ne, ln, ext = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().ac_plan_rank_chunks(self._h, region, rank, world, None, 0, C.byref(cnt), None, None, None))
        arr = (C.c_int64 * max(cnt.value, 1))()
        check(lib().ac_plan_rank_chunks(self._h, region, rank, world, arr, cnt.value, C.byref(cnt), C.byref(ne),
                                        C.byref(ln), C.byref(ext)))
        return list(arr)[: cnt.value], ne.value, ln.value, ext.value

    def chunk_pipeline(self):
        """ac_plan_chunk_pipeline: (wait, pipelined) - per node the node of the
        previous chunk it waits for (-1 none), per region whether its chunks alternate
        between two streams."""
        nn, nr = self.graph.num_nodes, self.num_regions
        w, p = (C.c_int32 * max(nn, 1))(), (C.c_int32 * max(nr, 1))()
        check(lib().ac_plan_chunk_pipeline(self._h, w, p))
        return list(w)[:nn], list(p)[:nr]

    def rank_schedule(self, rank: int, world: int):
        """ac_plan_rank_schedule: (node_region, node_dim, ops) - per node the region
        share it runs on (-1 whole) and its output dim, and the exchanges as dicts."""
        nn = self.graph.num_nodes
        nr, nd = (C.c_int32 * max(nn, 1))(), (C.c_int32 * max(nn, 1))()
        cnt = C.c_int32()
        check(lib().ac_plan_rank_schedule(self._h, rank, world, nr, nd, None, 0, C.byref(cnt)))
        ops = (L.ExchangeOp * max(cnt.value, 1))()
        check(lib().ac_plan_rank_schedule(self._h, rank, world, nr, nd, ops, cnt.value, C.byref(cnt)))
        out = [{f: (getattr(o, f).decode() if f == "tensor" else getattr(o, f)) for f, _ in L.ExchangeOp._fields_}
               for o in ops[: cnt.value]]
        return list(nr)[:nn], list(nd)[:nn], out

    def workspace_bytes(self, rank: int = 0, world: int = 1) -> int:
        v = lib().ac_plan_workspace_bytes(self._h, rank, world)
        if v < 0:
            raise L.ACError(L.AC_ERR_PLAN, lib().ac_last_error().decode())
        return v


def arena_profile(plan: Plan):
    """ac_plan_arena_profile: (live bytes of the arena's activation slots per step,
    their peak, control bytes) of the arena ac_exec_create lays out for `plan`."""
    n = plan.graph.num_nodes
    arr = (C.c_int64 * max(n, 1))()
    pk, cb = C.c_int64(), C.c_int64()
    check(lib().ac_plan_arena_profile(plan.handle, arr, C.byref(pk), C.byref(cb)))
    return list(arr)[:n], pk.value, cb.value


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


class Comm:
    """NCCL communicator (ac_comm_*); `unique_id` is broadcast by the caller."""

    def __init__(self, unique_id: bytes | None, rank: int, world: int, device: int, handle=None):
        if handle is not None:
            self._h = C.c_void_p(handle)
        else:
            out = C.c_void_p()
            check(lib().ac_comm_init(unique_id, rank, world, device, C.byref(out)))
            self._h = out
        self.rank, self.world = rank, world

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().ac_comm_get_unique_id(buf))
        return buf.raw

    @staticmethod
    def local(world: int) -> list:
        """ac_comm_init_local: `world` in-process ranks on the current device (tests)."""
        arr = (C.c_void_p * world)()
        check(lib().ac_comm_init_local(world, arr))
        return [Comm(None, r, world, 0, handle=arr[r]) for r in range(world)]

    def check(self):
        check(lib().ac_comm_check(self._h))

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            try:
                lib().ac_comm_free(self._h)
            except TypeError:  # interpreter shutdown
                pass
            self._h = None


_TORCH_DT = None


def _dtype_code(t) -> int:
    import torch
    return {torch.float32: L.AC_F32, torch.bfloat16: L.AC_BF16, torch.float64: L.AC_F64}[t.dtype]


def _tensor(tid: str, t, keep: list) -> L.Tensor:
    b = tid.encode()
    keep.append(b)
    at = L.Tensor()
    at.tensor_id = b
    at.dtype = _dtype_code(t)
    at.ndim = t.dim()
    for i in range(t.dim()):
        at.shape[i] = t.shape[i]
        at.stride[i] = t.stride(i)
    at.data = t.data_ptr()
    return at


class Exec:
    """ac_exec_create / ac_run / ac_exec_stats.  `workspace` is a caller-owned
    device tensor of at least plan.workspace_bytes() bytes."""

    def __init__(self, plan: Plan, workspace, comm: Comm | None = None):
        out = C.c_void_p()
        nbytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
        ptr = None if workspace is None else workspace.data_ptr()
        check(lib().ac_exec_create(plan.handle, ptr, nbytes, comm.handle if comm else None, C.byref(out)))
        self._h = out
        self.plan, self.workspace, self.comm = plan, workspace, comm

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            try:
                lib().ac_exec_free(self._h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self._h = None

    def run(self, inputs: dict, outputs: dict, stream=None):
        import torch
        keep = []
        ins = [_tensor(k, v, keep) for k, v in inputs.items()]
        outs = [_tensor(k, v, keep) for k, v in outputs.items()]
        ia = (L.Tensor * max(len(ins), 1))(*ins)
        oa = (L.Tensor * max(len(outs), 1))(*outs)
        if stream is None:
            stream = torch.cuda.current_stream()
        check(lib().ac_run(self._h, ia, len(ins), oa, len(outs), C.c_void_p(stream.cuda_stream)))

    def stats(self) -> L.RunStats:
        s = L.RunStats()
        check(lib().ac_exec_stats(self._h, C.byref(s)))
        return s

    def set_profiling(self, on: bool = True):
        check(lib().ac_exec_set_profiling(self._h, int(on)))

    def kernel_times(self) -> list:
        """[(node id, kind, total ms, launches)] of the last run (profiling on)."""
        n = C.c_int32()
        check(lib().ac_exec_kernel_times(self._h, None, 0, C.byref(n)))
        arr = (L.KernelTime * max(n.value, 1))()
        check(lib().ac_exec_kernel_times(self._h, arr, n.value, C.byref(n)))
        return [(a.node.decode(), a.kind.decode(), a.ms, a.launches) for a in arr[: n.value]]


def max_length(kind: str, d: int, h: int, f: int, causal: bool, dtype: str, budget: int, layers: int = 1,
               step: int = 128, cap: int = 1 << 22, params: L.CostParams | None = None) -> dict:
    """ac_max_length (the search runs in the library): the largest length, a multiple
    of `step` <= cap, whose unchunked Eq. 1 peak and whose ac_plan peak fit `budget`
    activation bytes (SPEC cmd_maxlen S:478-486).  Returns {"unchunked",
    "chunked", "ratio", "plan"} (plan: ac_plan's regions at the chunked maximum)."""
    desc = L.BlockDesc(KINDS[kind], 1, d, h, f, int(causal), DTYPES[dtype], 1e-5, None, int(layers))
    nu, nc = C.c_int64(), C.c_int64()
    check(lib().ac_max_length(C.byref(desc), budget, step, cap, C.byref(params) if params else None,
                              C.byref(nu), C.byref(nc)))
    plan = None
    if nc.value:
        p = ac_plan(graph_block(kind, nc.value, d, h, f, causal, dtype, name="maxlen", layers=layers), budget, params)
        plan = [ln.split(" flow=")[0] for ln in p.serialize().splitlines() if ln.startswith("region")]
    return {"unchunked": nu.value, "chunked": nc.value, "ratio": (nc.value / nu.value) if nu.value else None,
            "plan": plan}
