"""GPU analytic oracles: slow, independently derived sums that validate the
fast Spectral Ewald path (SURVEY.md §8 f row 3; SPEC.md module `reference`,
SPEC.md:704-798; the reference ships it as a stub, proj/src/reference.cpp:1).

All numeric work runs in `csrc/analytic.cu` (sm_100a) behind the C-ABI
(include/sewald_gpu.h "analytic oracles"); nothing here falls back to the CPU.

    direct_sum_0p                 D = 0 bare-kernel sum
    direct_ewald_fourier_3p       D = 3 k-space sum + stresslet zero mode
    q2p, q2p_zero, q1p, q1p_zero  Appendix A / B tensors
    fourier_reference_potential   D = 2 / 1 q-sums, D = 3 -> direct Ewald
    incomplete_bessel_K4          K_nu(a, b), nu = -1..2 (PAPER.md Knu-def)
    rms_error, rel_rms_error      PAPER.md abs-/rel-rms-error
    stresslet_identity_check      PAPER.md:1218 (stresslet integral identity) through full_potential

Periodic sums are truncated at k_i = 2 pi j / L_i, -kmax_i <= j <= kmax_i - 1
(PAPER.md:1117-1130); `kmax_for(xi, L)` picks kmax so that the omitted modes
are below e^{-39} of the largest (the Fourier kernels decay like
e^{-k^2 / (4 xi^2)}).
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Optional, Sequence, Union

import numpy as np

from . import _abi
from .api import (Engine, EwaldParams, InvalidArgument, Kernel, SourceSystem, TargetSet, default_engine,
                  full_potential, strength_components, _system_arrays, _vec3)


def _dp(a):
    return a.ctypes.data_as(_abi.DP) if a is not None and a.size else None


def _eng(engine: Optional[Engine]) -> Engine:
    return engine or default_engine()


def kmax_for(xi: float, L: Sequence[float], decay: float = 39.0) -> list:
    """Smallest kmax per axis with e^{-k^2/(4 xi^2)} < e^{-decay} beyond it."""
    kc = 2.0 * float(xi) * math.sqrt(decay)
    return [int(math.ceil(kc * float(l) / (2.0 * math.pi))) + 1 for l in L]


def _kmax_arg(kmax, xi, L, d):
    if kmax is None:
        km = kmax_for(xi, L[:d])
    elif np.isscalar(kmax):
        km = [int(kmax)] * d
    else:
        km = [int(v) for v in kmax]
    if len(km) < d:
        raise InvalidArgument("kmax needs one entry per periodic direction")
    return (C.c_int * d)(*km[:d])


def _targets_of(system: SourceSystem, targets: Optional[TargetSet], x: np.ndarray) -> np.ndarray:
    if targets is None or targets.same_as_sources:
        return x
    return _vec3(targets.x, "targets")


def direct_sum_0p(system: SourceSystem, targets: TargetSet, starred: bool,
                  engine: Optional[Engine] = None) -> np.ndarray:
    """plain O(N * Nt) bare-kernel sum (D = 0), skipping the
    self pair when `starred` (targets = sources). Raises DomainError when a
    target coincides with a source otherwise."""
    if int(system.d) != 0:
        raise InvalidArgument("direct_sum_0p needs d = 0")
    x, f, nu = _system_arrays(system)
    xt = _targets_of(system, targets, x)
    if starred and xt.shape[0] != x.shape[0]:
        raise InvalidArgument("starred evaluation needs one target per source")
    u = np.zeros((xt.shape[0], 3))
    e = _eng(engine)
    with e._lock:
        e.check(e._lib.sewald_gpu_direct_sum_0p(e.ctx, int(system.kind), _dp(x), _dp(f), _dp(nu), x.shape[0],
                                                _dp(xt), xt.shape[0], int(bool(starred)), _dp(u)))
    return u


def direct_ewald_fourier_3p(system: SourceSystem, targets: TargetSet, xi: float,
                            kmax: Union[None, int, Sequence[int]] = None,
                            engine: Optional[Engine] = None) -> np.ndarray:
    """SPEC.md:728-735 / PAPER.md:673: (1/|B|) sum_{k != 0} G^F(k) . f_n
    e^{ik.(x - x_n)} over the truncated cube, plus the stresslet zero mode
    (PAPER.md:775). kmax = index half-width per axis (k_inf = 2 pi kmax / L)."""
    if int(system.d) != 3:
        raise InvalidArgument("direct_ewald_fourier_3p needs d = 3")
    return fourier_reference_potential(system, targets, xi, kmax, engine)


def fourier_reference_potential(system: SourceSystem, targets: TargetSet, xi: float,
                                kmax: Union[None, int, Sequence[int]] = None,
                                engine: Optional[Engine] = None) -> np.ndarray:
    """the Fourier-space part by direct summation, D = 2
    (Appendix A q-sums), D = 1 (Appendix B q-sums, gauge constants 1) or
    D = 3 (direct Ewald)."""
    d = int(system.d)
    if d not in (1, 2, 3):
        raise InvalidArgument("fourier_reference_potential needs d in 1..3 (d = 0: direct_sum_0p)")
    if not (float(xi) > 0.0):
        raise InvalidArgument("xi must be positive")
    x, f, nu = _system_arrays(system)
    xt = _targets_of(system, targets, x)
    L = (C.c_double * 3)(*[float(v) for v in system.cell.L])
    km = _kmax_arg(kmax, xi, list(system.cell.L), d)
    u = np.zeros((xt.shape[0], 3))
    e = _eng(engine)
    with e._lock:
        e.check(e._lib.sewald_gpu_fourier_reference_potential(
            e.ctx, int(system.kind), d, L, float(xi), km, _dp(x), _dp(f), _dp(nu), x.shape[0], _dp(xt),
            xt.shape[0], _dp(u)))
    return u


def _qtensor(kind: Kernel, d: int, zero: bool, args: np.ndarray, xi: float, engine) -> np.ndarray:
    args = np.ascontiguousarray(np.atleast_2d(np.asarray(args, dtype=np.float64)))
    if args.shape[-1] != 3:
        raise InvalidArgument("tensor arguments come in triples")
    n = args.shape[0]
    Cc = strength_components(Kernel(kind))
    out = np.zeros((n, 3, Cc), dtype=np.complex128)
    e = _eng(engine)
    with e._lock:
        e.check(e._lib.sewald_gpu_qtensor(e.ctx, int(kind), d, int(zero), n, _dp(args), float(xi),
                                          out.view(np.float64).ctypes.data_as(_abi.DP)))
    if Cc == 9:
        return out.reshape(n, 3, 3, 3)
    return out


def q2p(kind: Kernel, k1, k2, r3, xi: float, engine: Optional[Engine] = None) -> np.ndarray:
    """Q^{2P}(k1, k2, r3; xi), (k1, k2) != 0: (n, 3, 3) or (n, 3, 3, 3) complex."""
    a = np.stack(np.broadcast_arrays(np.asarray(k1, float), np.asarray(k2, float), np.asarray(r3, float)), -1)
    return _qtensor(kind, 2, False, a.reshape(-1, 3), xi, engine)


def q2p_zero(kind: Kernel, r3, xi: float, engine: Optional[Engine] = None) -> np.ndarray:
    """Q^{2P,(0)}(r3; xi)."""
    r3 = np.asarray(r3, float).reshape(-1)
    a = np.stack([np.zeros_like(r3), np.zeros_like(r3), r3], -1)
    return _qtensor(kind, 2, True, a, xi, engine)


def q1p(kind: Kernel, k1, r2, r3, xi: float, engine: Optional[Engine] = None) -> np.ndarray:
    """Q^{1P}(k1, r2, r3; xi), k1 != 0."""
    a = np.stack(np.broadcast_arrays(np.asarray(k1, float), np.asarray(r2, float), np.asarray(r3, float)), -1)
    return _qtensor(kind, 1, False, a.reshape(-1, 3), xi, engine)


def q1p_zero(kind: Kernel, r2, r3, xi: float, engine: Optional[Engine] = None) -> np.ndarray:
    """Q^{1P,(0)}(r2, r3; xi) with ell_H = ell_B = 1."""
    r2, r3 = np.broadcast_arrays(np.asarray(r2, float).reshape(-1), np.asarray(r3, float).reshape(-1))
    a = np.stack([np.zeros_like(r2), r2, r3], -1)
    return _qtensor(kind, 1, True, a, xi, engine)


def incomplete_bessel_K4(a, b, engine: Optional[Engine] = None) -> np.ndarray:
    """K_nu(a, b) for nu = -1, 0, 1, 2 (columns), a > 0, b >= 0, on the GPU."""
    a, b = np.broadcast_arrays(np.asarray(a, float).reshape(-1), np.asarray(b, float).reshape(-1))
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    out = np.zeros((a.size, 4))
    e = _eng(engine)
    with e._lock:
        e.check(e._lib.sewald_gpu_incomplete_bessel_k4(e.ctx, a.size, _dp(a), _dp(b), _dp(out)))
    return out


def rms_error(u, u_ref) -> float:
    """Absolute rms error sqrt(mean_i |u_i - u_ref,i|^2) (PAPER.md abs-rms-error)."""
    return _rms(u, u_ref)[0]


def rel_rms_error(u, u_ref) -> float:
    """rms_error divided by the rms of u_ref (PAPER.md rel-rms-error)."""
    return _rms(u, u_ref, rel=True)[1]


def _rms(u, u_ref, rel=False):
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64).reshape(-1, 3))
    r = np.ascontiguousarray(np.asarray(u_ref, dtype=np.float64).reshape(-1, 3))
    if u.shape != r.shape:
        raise InvalidArgument("rms error needs equal lengths")
    if u.shape[0] == 0:
        raise InvalidArgument("rms error of an empty set")
    a, b = C.c_double(), C.c_double()
    code = _abi.load().sewald_rms_error(_dp(u), _dp(r), u.shape[0], C.byref(a), C.byref(b) if rel else None)
    if code != _abi.OK:
        _abi.raise_for(code, "relative rms error of a zero reference")
    return float(a.value), float(b.value)


def sphere_quadrature(center, radius: float, order: int):
    """Nodes, outward normals and weights of a longitude-latitude rule on a
    sphere: Gauss-Legendre in cos(theta) (`order` nodes) times the trapezoid
    rule in phi (2 * order nodes), exact for spherical harmonics of degree
    < 2 * order."""
    t, wt = np.polynomial.legendre.leggauss(int(order))
    ph = 2.0 * np.pi * (np.arange(2 * order) + 0.5) / (2 * order)
    st = np.sqrt(1.0 - t * t)
    n = np.stack([np.outer(st, np.cos(ph)), np.outer(st, np.sin(ph)), np.outer(t, np.ones_like(ph))], -1)
    n = n.reshape(-1, 3)
    w = np.outer(wt, np.full(ph.size, 2.0 * np.pi / ph.size)).reshape(-1) * radius * radius
    x = np.asarray(center, float)[None, :] + radius * n
    return x, n, w


def stresslet_identity_check(d: int, center, radius: float, order: int, targets, params: EwaldParams,
                             q0=(1.0, 0.0, 0.0), cell=(1.0, 1.0, 1.0), expected: Optional[Sequence[float]] = None,
                             engine: Optional[Engine] = None) -> np.ndarray:
    """SPEC.md:765-772 / PAPER.md:1218: discretize a sphere, place stresslet
    sources q = q0 * w_i with unit outward normals, evaluate the full potential
    (the fast GPU path) at `targets` and return |u - expected| / (8 pi |q0|)
    per target. `expected` is the constant vector the identity predicts for
    those targets, in units of q0 (e.g. 0 or 8 pi)."""
    x, n, w = sphere_quadrature(center, radius, order)
    q0 = np.asarray(q0, float)
    f = w[:, None] * q0[None, :]
    system = SourceSystem(Kernel.stresslet, _cell(cell), int(d), x, f, n)
    xt = np.atleast_2d(np.asarray(targets, float))
    u = full_potential(system, TargetSet(xt), params, engine=engine)
    exp = np.zeros(3) if expected is None else float(expected) * q0
    return np.linalg.norm(u - exp[None, :], axis=1) / (8.0 * np.pi * np.linalg.norm(q0))


def _cell(L):
    from .api import Cell
    return L if isinstance(L, Cell) else Cell(tuple(float(v) for v in L))
