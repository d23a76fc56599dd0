"""Replay of one rank's multi-GPU schedule (ac_plan_rank_chunks / ac_plan_rank_schedule,
include/ac.h) with the oracle's node maths in fp64 on the host, and the
schedule's exchanges as torch.distributed collectives (gloo on CPU).

The library decides everything here - which chunks the rank runs, which nodes outside
the regions run on its rows only, which exchanges happen where; this module only
executes that decision with oracle.ops, so a test that compares every rank's outputs
with the unchunked single-process run checks the schedule ac_run follows on the GPU.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from oracle import ops


def _slice(a, d, off, ln):
    idx = [slice(None)] * a.ndim
    idx[d] = slice(off, off + ln)
    return a[tuple(idx)]


def _ranges(chunks, L, E):
    out = []
    for c in chunks:
        a, b = c * L, min(E, (c + 1) * L)
        if b <= a:
            continue
        if out and out[-1][1] == a:
            out[-1] = (out[-1][0], b)
        else:
            out.append((a, b))
    return out


def _is_dim(r):
    return isinstance(r, int) and r >= 0


def _run_region(g, R, env, chunks, L):
    """The rank's chunks of region R: X^c sliced, X^nc whole, Y^c written in place."""
    E = R.extent
    hs = set(R.hoisted)
    produced = {g.nodes[k].output for k in range(R.start, R.end + 1)}
    ydims = dict(R.yc)
    for k in R.hoisted:
        nd = g.nodes[k]
        env[nd.output] = ops.evaluate(nd.kind, nd.attrs, [env[t] for t in nd.inputs], None)
    for y, _ in R.yc:
        env[y] = np.zeros(g.tensors[y].shape)
    for c in chunks:
        off = c * L
        ln = min(L, E - off)
        if ln <= 0:
            continue
        local = {}
        for k in range(R.start, R.end + 1):
            if k in hs:
                continue
            nd = g.nodes[k]
            if nd.output not in R.dims:
                local[nd.output] = ops.evaluate(nd.kind, nd.attrs,
                                                [local[t] if t in local else env[t] for t in nd.inputs], None)
                continue
            res = ops.propagate(nd.kind, nd.attrs, [g.tensors[t].shape for t in nd.inputs],
                                g.tensors[nd.output].shape, R.dims[nd.output])
            vals = []
            for t, rr in zip(nd.inputs, res):
                if t in local:
                    vals.append(local[t])
                elif _is_dim(rr) and t not in produced:
                    vals.append(_slice(env[t], rr, off, ln))
                else:
                    vals.append(env[t])
            out = ops.evaluate(nd.kind, nd.attrs, vals, {"dim": R.dims[nd.output], "offset": off})
            if nd.output in ydims:
                _slice(env[nd.output], ydims[nd.output], off, ln)[...] = out
            local[nd.output] = out


def _exchange(g, env, o, rank, world, log):
    """One ac_exchange_op with gloo collectives (byte offsets over the graph dtype)."""
    t = o["tensor"]
    a = env[t]
    esz = g.tensors[t].esize
    log.append((o["kind"], t, o["before_node"], o["eager"], o["group"]))
    if o["kind"] == 2:                      # broadcast of a byte run from its owner
        flat = a.reshape(-1)
        lo, n = o["offset"] // esz, o["run_bytes"] // esz
        buf = torch.from_numpy(np.ascontiguousarray(flat[lo:lo + n]))
        dist.broadcast(buf, src=o["root"])
        flat[lo:lo + n] = buf.numpy()
        return
    d = o["dim"]
    shp = a.shape
    inner = int(np.prod(shp[d + 1:])) if d + 1 < len(shp) else 1
    L = o["run_bytes"] // (esz * inner)
    v = a.reshape(o["outer"], shp[d], inner)
    pos = (lambda q: world - 1 - q) if o["kind"] == 1 else (lambda q: q)
    mine = torch.from_numpy(np.ascontiguousarray(v[:, (o["c_first"] + pos(rank)) * L:(o["c_first"] + pos(rank) + 1) * L]))
    got = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(got, mine)
    for q in range(world):
        c = o["c_first"] + pos(q)
        v[:, c * L:(c + 1) * L] = got[q].numpy()


def run_rank(g, values, regions, cplan, rank, world):
    """Execute rank `rank`'s schedule.  `regions` are the oracle's Region objects of the
    same plan (flows, X^c, Y^c, hoisting); the chunk shares come from the library.
    Returns (outputs, exchange log)."""
    node_region, node_dim, xops = cplan.rank_schedule(rank, world)
    shares = [cplan.rank_chunks(k, rank, world) for k in range(len(regions))]
    env = dict(values)
    S = len(g.nodes)
    at = {R.start: k for k, R in enumerate(regions) if R.n > 1}
    log = []

    def before(i):
        for o in xops:
            if o["before_node"] == i:
                _exchange(g, env, o, rank, world, log)

    i = 0
    while i < S:
        nd = g.nodes[i]
        if nd.kind in ("input", "weight"):
            i += 1
            continue
        before(i)
        if i in at:
            k = at[i]
            chunks, _, L, _ = shares[k]
            _run_region(g, regions[k], env, chunks, L)
            i = regions[k].end + 1
            continue
        if node_region[i] >= 0:
            chunks, _, L, E = shares[node_region[i]]
            d = node_dim[i]
            res = ops.propagate(nd.kind, nd.attrs, [g.tensors[t].shape for t in nd.inputs],
                                g.tensors[nd.output].shape, d)
            out = np.zeros(g.tensors[nd.output].shape)
            for a, b in _ranges(chunks, L, E):
                vals = [_slice(env[t], rr, a, b - a) if _is_dim(rr) else env[t] for t, rr in zip(nd.inputs, res)]
                _slice(out, d, a, b - a)[...] = ops.evaluate(nd.kind, nd.attrs, vals, {"dim": d, "offset": a})
            env[nd.output] = out
        else:
            env[nd.output] = ops.evaluate(nd.kind, nd.attrs, [env[t] for t in nd.inputs], None)
        i += 1
    before(S)
    return {o: env[o] for o in g.outputs}, log
