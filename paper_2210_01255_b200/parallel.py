"""Multi-GPU decomposition of one full-potential evaluation.

One process per GPU. Each rank spreads a contiguous 1/W slice of the sources
into a full grid; the per-rank grids are summed with one all-reduce (NCCL
over NVLink on the box, gloo in the CPU tests); every rank runs the k-space
solve (cheap next to spread / real space at the BASELINE sizes) and
evaluates its 1/W part of the targets (real space + gather + terms). The
target parts are disjoint, so the assembled result is the sum of the
per-rank outputs. Spread is linear in the sources, so the sum of the slice
grids equals the single-GPU grid.

`session` is anything with the Session stage interface: spread(i0, i1,
grid), solve(grid, precompute_0p), evaluate(u, part, nparts, parts).
"""
from __future__ import annotations

import os
from typing import Callable, Optional

# D = 3 grids are slab-distributed too when SEWALD_SLAB_D3=1; by default they
# are all-reduced and solved on every rank (the whole D = 3 k-space step is
# 0.16 ms at c2).
SLAB_D3 = os.environ.get("SEWALD_SLAB_D3", "0") == "1"


def use_slabs(d: int, world: int) -> bool:
    """Whether the k-space step of a world-rank run is slab-distributed."""
    return world > 1 and (d == 0 or (d == 3 and SLAB_D3))


def slice_bounds(n: int, rank: int, world: int):
    """Contiguous, balanced [i0, i1) of n items for `rank` of `world`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank / world size")
    return n * rank // world, n * (rank + 1) // world


def sharded_step(session, n_sources: int, grid, u, rank: int, world: int,
                 all_reduce: Optional[Callable] = None, precompute_0p: bool = True, parts: int = 7,
                 gather_result: bool = True, slab_dist=None):
    """One distributed full-potential step. Each rank's evaluate() output
    holds its part's contributions (zero elsewhere); with gather_result the
    outputs are summed so every rank ends with the full velocity field.
    With `slab_dist` (torch.distributed) the D = 0 / D = 3 solve is slab-distributed
    (d0_sharded_solve) instead of replicated after a grid all-reduce."""
    i0, i1 = slice_bounds(n_sources, rank, world)
    session.spread(i0, i1, grid)
    if world > 1 and slab_dist is not None:
        d0_sharded_solve(session, grid, rank, world, slab_dist, precompute_0p)
        session.evaluate(u, rank, world, parts)
        if gather_result:
            all_reduce(u)
        return
    if world > 1:
        if all_reduce is None:
            raise ValueError("world > 1 needs an all_reduce")
        all_reduce(grid)
    session.solve(grid, precompute_0p)
    session.evaluate(u, rank, world, parts)
    if world > 1 and gather_result:
        all_reduce(u)


# ---------------------------------------------------------------------------
# Slab-distributed D = 0 solve (BASELINE config 5): x-slabs of the
# M_ext box for the z transforms, kz-slabs of the half spectrum for the 2-D
# (x, y) transforms and the scale, two all-to-all exchanges (NCCL) between.
# The stage functions are shared by the distributed driver (d0_sharded_solve)
# and the single-process emulation used by the tests.
# ---------------------------------------------------------------------------

class D0Slabs:
    """Split points and all-to-all split sizes (in complex elements) of the
    slab-distributed D = 0 solve for `world` ranks."""

    def __init__(self, geometry: dict, world: int):
        self.m, self.n, self.h2, self.C = geometry["m"], geometry["n"], geometry["h2"], geometry["C"]
        self.world = world
        self.xb = [slice_bounds(self.m[0], r, world)[0] for r in range(world)] + [self.m[0]]
        self.kb = [slice_bounds(self.h2, r, world)[0] for r in range(world)] + [self.h2]

    def nx(self, r):
        return self.xb[r + 1] - self.xb[r]

    def nk(self, r):
        return self.kb[r + 1] - self.kb[r]

    def fwd_send_splits(self, r):   # chunk q: [C][nx_r][m1][nk_q]
        return [self.C * self.nx(r) * self.m[1] * self.nk(q) for q in range(self.world)]

    def fwd_recv_splits(self, r):   # chunk p: [C][nx_p][m1][nk_r]
        return [self.C * self.nx(p) * self.m[1] * self.nk(r) for p in range(self.world)]

    def inv_send_splits(self, r):   # chunk q: [3][nk_r][nx_q][m1]
        return [3 * self.nk(r) * self.nx(q) * self.m[1] for q in range(self.world)]

    def inv_recv_splits(self, r):   # chunk p: [3][nk_p][nx_r][m1]
        return [3 * self.nk(p) * self.nx(r) * self.m[1] for p in range(self.world)]


def d0_stage_forward(session, slabs: D0Slabs, rank: int, grid_slab, precompute_0p: bool = True):
    import torch
    send = torch.empty(sum(slabs.fwd_send_splits(rank)), dtype=torch.complex128, device=grid_slab.device)
    session.d0_forward(grid_slab, slabs.xb[rank], slabs.xb[rank + 1], slabs.kb, send, precompute_0p)
    return send


def d0_stage_middle(session, slabs: D0Slabs, rank: int, recv, precompute_0p: bool = True):
    import torch
    send = torch.empty(sum(slabs.inv_send_splits(rank)), dtype=torch.complex128, device=recv.device)
    session.d0_middle(recv, slabs.xb, slabs.kb[rank], slabs.kb[rank + 1], send, precompute_0p)
    return send


def d0_stage_inverse(session, slabs: D0Slabs, rank: int, recv, precompute_0p: bool = True):
    import torch
    flow = torch.empty((3, slabs.nx(rank), slabs.m[1], slabs.m[2]), dtype=torch.float64, device=recv.device)
    session.d0_inverse(recv, slabs.xb[rank], slabs.xb[rank + 1], slabs.kb, flow, precompute_0p)
    return flow


def emulate_all_to_all(sends, send_splits, recv_splits):
    """All-to-all of per-rank flat buffers in one process (tests): rank r
    receives chunk r of every rank p's send buffer, in rank order."""
    import torch
    world = len(sends)
    chunks = [list(torch.split(sends[p], send_splits[p])) for p in range(world)]
    recvs = []
    for r in range(world):
        parts = [chunks[p][r] for p in range(world)]
        assert [t.numel() for t in parts] == recv_splits[r]
        recvs.append(torch.cat(parts))
    return recvs


def _all_to_all(dist, recv, send, recv_splits, send_splits, group=None):
    # complex buffers travel as real pairs (NCCL has no complex type)
    dist.all_to_all_single(__import__("torch").view_as_real(recv), __import__("torch").view_as_real(send),
                           recv_splits, send_splits, group=group)


def d0_sharded_solve(session, grid, rank: int, world: int, dist, precompute_0p: bool = True, group=None):
    """Distributed D = 0 solve. `grid` holds this rank's spread (full box,
    partial over its source slice); on return every rank's session holds the
    full flow field for evaluate(). Collectives: one reduce-scatter of the
    grid to x-slabs, two all-to-alls, one all-gather of the flow slabs."""
    import torch
    geo = session.d0_geometry(precompute_0p)
    sl = D0Slabs(geo, world)
    C, m = sl.C, sl.m
    g = grid.view(C, m[0], m[1], m[2])
    # reduce-scatter to x-slabs (chunks padded to a common size)
    mx = max(sl.nx(q) for q in range(world))
    ins = []
    for q in range(world):
        t = torch.zeros((C, mx, m[1], m[2]), dtype=grid.dtype, device=grid.device)
        t[:, :sl.nx(q)] = g[:, sl.xb[q]:sl.xb[q + 1]]
        ins.append(t)
    red = torch.empty((C, mx, m[1], m[2]), dtype=grid.dtype, device=grid.device)
    if dist.get_backend(group) == "gloo":  # no reduce-scatter in gloo (CPU tests): all-reduce + slice
        full = grid.clone()
        dist.all_reduce(full, group=group)
        red = full.view(C, m[0], m[1], m[2])[:, sl.xb[rank]:sl.xb[rank + 1]]
    else:
        dist.reduce_scatter(red, ins, group=group)
    slab = red[:, :sl.nx(rank)].contiguous()
    send = d0_stage_forward(session, sl, rank, slab, precompute_0p)
    recv = torch.empty(sum(sl.fwd_recv_splits(rank)), dtype=torch.complex128, device=grid.device)
    _all_to_all(dist, recv, send, sl.fwd_recv_splits(rank), sl.fwd_send_splits(rank), group)
    send2 = d0_stage_middle(session, sl, rank, recv, precompute_0p)
    recv2 = torch.empty(sum(sl.inv_recv_splits(rank)), dtype=torch.complex128, device=grid.device)
    _all_to_all(dist, recv2, send2, sl.inv_recv_splits(rank), sl.inv_send_splits(rank), group)
    flow_slab = d0_stage_inverse(session, sl, rank, recv2, precompute_0p)
    # all-gather the flow slabs (padded) and assemble the full field
    pad = torch.zeros((3, mx, m[1], m[2]), dtype=torch.float64, device=grid.device)
    pad[:, :sl.nx(rank)] = flow_slab
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    flow = torch.cat([outs[q][:, :sl.nx(q)] for q in range(world)], dim=1).contiguous()
    session.set_flow(flow)
    return flow


# ---------------------------------------------------------------------------
# Multi-GPU public entry point (host arrays in, host array out)
# ---------------------------------------------------------------------------

_SESSIONS = {}


def full_potential_sharded(system, targets, params, rank: int, world: int, dist=None, engine=None, out=None,
                           precompute_0p: bool = True, group=None):
    """full_potential (realspace.h:46-47) on `world` GPUs, one process each.

    Every rank calls it with the same host arrays (as it would call the
    reference's full_potential); rank r uploads the inputs (the real-space sum
    needs every source), spreads its 1/W slice of the sources, the grids are
    summed (all-reduce; for D = 0 the slab-distributed solve), rank r evaluates
    its 1/W of the cell-ordered targets, and the per-rank outputs are summed
    onto rank 0 (reduce), which copies the velocity to `out` (host, e.g.
    pinned). Returns u on rank 0 and None elsewhere. With world == 1 no
    collective is issued."""
    import numpy as np
    import torch

    from .api import Cell, Session, _system_arrays, _vec3, default_engine, InvalidArgument

    if world > 1 and dist is None:
        raise InvalidArgument("world > 1 needs torch.distributed")
    eng = engine or default_engine()
    dev = torch.device("cuda", eng.device)
    x, f, nu = _system_arrays(system, params)
    same = bool(targets.same_as_sources)
    xt = None if same else _vec3(targets.x, "targets")
    key = (id(eng), bytes(params.to_c()), tuple(float(v) for v in system.cell.L))
    sess = _SESSIONS.get(key)
    if sess is None:
        _SESSIONS.clear()
        sess = Session(params, Cell(tuple(system.cell.L)), eng)
        _SESSIONS[key] = sess
    T = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev, non_blocking=True)
    dx, df, dnu, dxt = T(x), T(f), T(nu), T(xt)
    sess.set_sources(dx, df, dnu)
    sess.set_targets(dxt, same)
    nt = x.shape[0] if same else xt.shape[0]
    grid = torch.empty(sess.grid_size(), dtype=torch.float64, device=dev)
    u = torch.empty((nt, 3), dtype=torch.float64, device=dev)
    reduce_sum = None
    if world > 1:
        reduce_sum = lambda t: dist.all_reduce(t, group=group)
    slab = dist if use_slabs(int(params.d), world) else None
    sharded_step(sess, x.shape[0], grid, u, rank, world, all_reduce=reduce_sum, precompute_0p=precompute_0p,
                 gather_result=False, slab_dist=slab)
    if world > 1:
        dist.reduce(u, dst=0, group=group)
    if rank != 0:
        torch.cuda.current_stream().synchronize()
        return None
    if out is None:
        out = np.empty((nt, 3))
    torch.from_numpy(out).copy_(u)  # D2H (synchronous)
    return out
