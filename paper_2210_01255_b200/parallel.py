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

from typing import Callable, Optional


def slice_bounds(n: int, rank: int, world: int):
    """Contiguous, balanced [i0, i1) of n items for `rank` of `world`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank / world size")
    return n * rank // world, n * (rank + 1) // world


def sharded_step(session, n_sources: int, grid, u, rank: int, world: int,
                 all_reduce: Optional[Callable] = None, precompute_0p: bool = True, parts: int = 7,
                 gather_result: bool = True):
    """One distributed full-potential step. Each rank's evaluate() output
    holds its part's contributions (zero elsewhere); with gather_result the
    outputs are summed so every rank ends with the full velocity field."""
    i0, i1 = slice_bounds(n_sources, rank, world)
    session.spread(i0, i1, grid)
    if world > 1:
        if all_reduce is None:
            raise ValueError("world > 1 needs an all_reduce")
        all_reduce(grid)
    session.solve(grid, precompute_0p)
    session.evaluate(u, rank, world, parts)
    if world > 1 and gather_result:
        all_reduce(u)
