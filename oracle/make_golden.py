"""ORACLE TEST INFRASTRUCTURE — generates tests/golden/*.npz from the
reference itself (oracle/_ref/libsewald_ref.so = the unmodified reference
sources compiled with the committed shims). Run in the builder container:

    make -C oracle && python oracle/make_golden.py

Each fixture stores its inputs, the parameter struct the reference selected
(raw bytes), and the reference outputs, so GPU parity tests on a box without
/root/reference compare against the reference's own numbers.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import sewald_ref as R  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def source_quantity(kind, f, nu):
    if kind == 1:
        return float(np.sum(np.sum(f * f, 1) * np.sum(nu * nu, 1)))
    return float(np.sum(f * f))


def case(name, kind, d, L, N, xi, tol, window=1, Nt=None, seed=0, extra_xi=(), fourier_direct=False):
    rng = np.random.default_rng(seed)
    x = rng.random((N, 3)) * np.asarray(L)
    f = rng.standard_normal((N, 3))
    nu = None
    if kind == 1:
        g = rng.standard_normal((N, 3))
        nu = g / np.linalg.norm(g, axis=1, keepdims=True)
    xt = rng.random((Nt, 3)) * np.asarray(L) if Nt else None
    same = xt is None
    Q = source_quantity(kind, f, nu)
    out = dict(x=x, f=f, kind=kind, d=d, L=np.asarray(L, float), xi=xi, tol=tol, window=window, Q=Q)
    if nu is not None:
        out["nu"] = nu
    if xt is not None:
        out["xt"] = xt
    for tag, xv in [("", xi)] + [(f"_xi{v:g}", v) for v in extra_xi]:
        p, rep = R.select_parameters(kind, d, L, Q, xv, tol, False, 4, window, True)
        out["params" + tag] = np.frombuffer(bytes(p), dtype=np.uint8)
        out["u" + tag] = R.full_potential(p, x, f, nu, xt, same)
        out["uF" + tag] = R.fourier_potential(p, x, f, nu, xt, same)
        out["uR" + tag] = R.realspace_potential(kind, d, L, x, f, nu, xt, same, xv, p.rc, same)
        if fourier_direct:
            out["uF_direct" + tag] = R.fourier_potential(p, x, f, nu, xt, same, precompute_0p=False)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print(f"{name}: N={N} u_rms={np.sqrt(np.mean(np.sum(out['u'] ** 2, 1))):.6g}")


def spread_case(name, kind, d, M, Mext, h, P, window, N, seed):
    """Stage fixture: spread and gather on a hand-built grid (test_fourier.cpp:20-33 style)."""
    rng = np.random.default_rng(seed)
    p = R.RefParams()
    p.kind, p.d, p.h, p.f_m = kind, d, h, 4
    for a in range(3):
        p.M[a], p.M_ext[a] = M[a], Mext[a]
        p.L[a] = h * M[a]
        p.L_ext[a] = h * Mext[a]
        p.pad[a] = p.L_ext[a] - p.L[a]
    p.win_kind, p.P, p.win_h = window, P, h
    p.beta, p.nu, p.alpha = 2.5 * P, min(P // 2 + 2, 10), 0.91 * 0.5 * np.pi * P
    L = np.array([p.L[0], p.L[1], p.L[2]])
    lo = np.array([0.0 if a < d else 0.2 for a in range(3)])
    hi = np.array([1.0 if a < d else 0.8 for a in range(3)])
    x = (lo + (hi - lo) * rng.random((N, 3))) * L
    f = rng.standard_normal((N, 3))
    nu = rng.standard_normal((N, 3)) if kind == 1 else None
    grid = R.spread(p, x, f, nu)
    field = rng.standard_normal((3,) + tuple(Mext))
    xt = (lo + (hi - lo) * rng.random((N, 3))) * L
    ug = R.gather(p, field, xt)
    out = dict(params=np.frombuffer(bytes(p), dtype=np.uint8), x=x, f=f, grid=grid, field=field, xt=xt, ug=ug)
    if nu is not None:
        out["nu"] = nu
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print(f"{name}: grid {grid.shape}")


def main():
    os.makedirs(OUT, exist_ok=True)
    # smoke(): N=400 stokeslet d=3, same RNG stream as __graft_entry__.smoke
    rng = np.random.default_rng(1001)
    x = rng.random((400, 3))
    f = rng.standard_normal((400, 3))
    p, _ = R.select_parameters(0, 3, (1, 1, 1), float(np.sum(f * f)), 10.0, 1e-8)
    np.savez_compressed(os.path.join(OUT, "smoke_stokeslet_d3.npz"), x=x, f=f, u=R.full_potential(p, x, f),
                        params=np.frombuffer(bytes(p), dtype=np.uint8))
    # config 1 (BASELINE configs[0]): N=2000, pinned xi=13.207, also xi=10
    case("c1_stokeslet_d3", 0, 3, (1, 1, 1), 2000, 13.207, 1e-8, seed=1001, extra_xi=(10.0,))
    case("stresslet_d3", 1, 3, (1, 1, 1), 500, 10.0, 1e-8, seed=2001)
    case("rotlet_d3", 2, 3, (1, 1, 1), 500, 10.0, 1e-8, seed=2002)
    case("stresslet_d2", 1, 2, (1, 1, 1), 300, 8.0, 1e-8, seed=2003)
    case("stokeslet_d2", 0, 2, (1, 1, 1), 300, 8.0, 1e-8, seed=2006)
    case("rotlet_d1_tg", 2, 1, (1, 1, 1), 300, 8.0, 1e-10, window=2, Nt=200, seed=2004)
    case("stokeslet_d1", 0, 1, (1, 1, 1), 300, 8.0, 1e-8, seed=2007)
    case("stokeslet_d0", 0, 0, (2, 1, 1), 300, 6.0, 1e-6, seed=2005, fourier_direct=True)
    spread_case("spread_kb_d3", 0, 3, (16, 16, 16), (16, 16, 16), 1 / 16, 8, 0, 60, 3001)
    spread_case("spread_pkb_d2_stresslet", 1, 2, (16, 16, 8), (16, 16, 24), 1 / 16, 8, 1, 60, 3002)
    spread_case("spread_tg_d0", 0, 0, (8, 8, 8), (20, 20, 20), 1 / 16, 10, 2, 60, 3003)


if __name__ == "__main__":
    main()
