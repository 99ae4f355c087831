"""BASELINE.json configurations as seeded synthetic workloads.

There is no public dataset for this path (the paper uses synthetic uniform
systems), so inputs are generated: numpy PCG64 seeded
with 1000 + config index, all positions first, then strengths (stresslet:
q ~ N(0,1)^3 then nu = g/|g|, g ~ N(0,1)^3; config 4 draws its separate
targets after the sources). The reference does not choose xi
(estimates.h:106-107), so xi is pinned per config and fed
identically to the GPU engine and the CPU reference.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from .api import Kernel, WindowKind


@dataclass(frozen=True)
class Config:
    index: int
    name: str
    kind: Kernel
    d: int
    L: Tuple[float, float, float]
    N: int
    Nt: Optional[int]   # None: targets are the sources
    tol: float
    xi: float
    window: WindowKind
    clustered: bool = False  # positions only in [0, 1/3)^3 and [2/3, 1)^3


CONFIGS = {
    1: Config(1, "c1_stokeslet_d3_N2e3", Kernel.stokeslet, 3, (1.0, 1.0, 1.0), 2000, None, 1e-8, 13.207, WindowKind.pkb),
    2: Config(2, "c2_stokeslet_d3_N1e6", Kernel.stokeslet, 3, (1.0, 1.0, 1.0), 1_000_000, None, 1e-8, 37.0, WindowKind.pkb),
    3: Config(3, "c3_stresslet_d2_N1e6", Kernel.stresslet, 2, (1.0, 1.0, 1.0), 1_000_000, None, 1e-8, 33.5, WindowKind.pkb),
    4: Config(4, "c4_rotlet_d1_N5e5", Kernel.rotlet, 1, (1.0, 1.0, 1.0), 500_000, 500_000, 1e-10, 34.0, WindowKind.tg),
    5: Config(5, "c5_stokeslet_d0_N4e6", Kernel.stokeslet, 0, (2.0, 1.0, 1.0), 4_000_000, None, 1e-6, 68.5, WindowKind.pkb),
    # not a BASELINE config: the paper's clustered random system (two dense
    # cubes) at c2's size and parameters - a load-balance
    # check (13.5x the local density: 13.5x the real-space pairs, tiles with
    # 13.5x the points, most tiles and cell rows empty)
    6: Config(6, "c6_stokeslet_d3_N1e6_clustered", Kernel.stokeslet, 3, (1.0, 1.0, 1.0), 1_000_000, None, 1e-8, 37.0,
              WindowKind.pkb, clustered=True),
}


def generate(cfg: Config, N: Optional[int] = None, Nt: Optional[int] = None, seed: Optional[int] = None):
    """Return (x, f, nu, xt) for a config; N/Nt override the sizes (parity
    tests use reduced N with the same distributions)."""
    n = cfg.N if N is None else N
    nt = cfg.Nt if Nt is None else Nt
    rng = np.random.default_rng(1000 + cfg.index if seed is None else seed)
    L = np.asarray(cfg.L)
    x = rng.random((n, 3)) * L
    if cfg.clustered:  # half the points in each of the two cubes of side L/3
        x = x / 3.0
        x[n // 2:] += 2.0 * L / 3.0
    f = rng.standard_normal((n, 3))
    nu = None
    if cfg.kind == Kernel.stresslet:
        g = rng.standard_normal((n, 3))
        nu = g / np.linalg.norm(g, axis=1, keepdims=True)
    xt = None
    if cfg.Nt is not None:
        xt = rng.random((nt, 3)) * L
    return x, f, nu, xt
