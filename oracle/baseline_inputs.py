"""ORACLE TEST INFRASTRUCTURE — the BASELINE configs' seeded inputs, drawn
without importing the product package, so the reference arm of bench.py and
the full-size fixtures load only oracle/ code.

The draw is the one SURVEY §8(d) prescribes and the product's
paper_2210_01255_b200/workloads.py repeats: numpy PCG64 seeded with
1000 + config index, all positions first (U[0,1) scaled by the box), then
the strengths (f ~ N(0,1)^3; stresslet: q ~ N(0,1)^3 then nu = g/|g|,
g ~ N(0,1)^3), then config 4's separate targets. tests/test_fullsize_inputs.py
checks that both draws give the same bytes (input_hash).

Kernel ids / window ids are include/sewald_gpu.h's (stokeslet 0, stresslet 1,
rotlet 2; KB 0, PKB 1, TG 2).
"""
from __future__ import annotations

import hashlib
import re
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np


@dataclass(frozen=True)
class Config:
    index: int
    name: str
    kind: int
    d: int
    L: Tuple[float, float, float]
    N: int
    Nt: Optional[int]
    tol: float
    xi: float
    window: int


CONFIGS = {
    1: Config(1, "c1_stokeslet_d3_N2e3", 0, 3, (1.0, 1.0, 1.0), 2000, None, 1e-8, 13.207, 1),
    2: Config(2, "c2_stokeslet_d3_N1e6", 0, 3, (1.0, 1.0, 1.0), 1_000_000, None, 1e-8, 37.0, 1),
    3: Config(3, "c3_stresslet_d2_N1e6", 1, 2, (1.0, 1.0, 1.0), 1_000_000, None, 1e-8, 33.5, 1),
    4: Config(4, "c4_rotlet_d1_N5e5", 2, 1, (1.0, 1.0, 1.0), 500_000, 500_000, 1e-10, 34.0, 2),
    5: Config(5, "c5_stokeslet_d0_N4e6", 0, 0, (2.0, 1.0, 1.0), 4_000_000, None, 1e-6, 68.5, 1),
}


def generate(index: int, N: Optional[int] = None, Nt: Optional[int] = None):
    cfg = CONFIGS[index]
    n = cfg.N if N is None else N
    nt = cfg.Nt if Nt is None else Nt
    rng = np.random.default_rng(1000 + cfg.index)
    L = np.asarray(cfg.L)
    x = rng.random((n, 3)) * L
    f = rng.standard_normal((n, 3))
    nu = None
    if cfg.kind == 1:
        g = rng.standard_normal((n, 3))
        nu = g / np.linalg.norm(g, axis=1, keepdims=True)
    xt = None
    if cfg.Nt is not None:
        xt = rng.random((nt, 3)) * L
    return x, f, nu, xt


def source_quantity(kind: int, f, nu) -> float:
    """domain.cpp:53-62: sum |f|^2, or sum |q|^2 |nu|^2 for the stresslet."""
    if kind == 1:
        return float(np.sum(np.sum(f * f, 1) * np.sum(nu * nu, 1)))
    return float(np.sum(f * f))


def input_hash(x, f, nu=None, xt=None) -> str:
    h = hashlib.sha256()
    for a in (x, f, nu, xt):
        if a is not None:
            h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def parse_tag(tag: str):
    """'c2' -> (2, None, None); 'c5n1e6' -> (5, 1000000, None); for configs with
    separate targets a reduced N lowers the target count to the same value."""
    m = re.fullmatch(r"c(\d)(?:n([0-9.e+]+))?", tag)
    if not m:
        raise ValueError(f"bad fixture tag {tag!r}")
    index = int(m.group(1))
    if m.group(2) is None:
        return index, None, None
    n = int(float(m.group(2)))
    return index, n, (n if CONFIGS[index].Nt is not None else None)
