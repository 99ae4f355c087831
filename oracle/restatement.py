"""ORACLE TEST INFRASTRUCTURE — not product code.

Independent numpy restatement of the reference's triply periodic (D = 3)
hot path, used by tests/ to cross-check the compiled reference
(oracle/_ref) and the committed golden fixtures. It is slow and small-N only.
Free-direction periodicities (D = 0, 1, 2) are checked against the compiled
reference, which is the stronger oracle; they are not restated here.

Each function cites the reference code it restates.
"""
from __future__ import annotations

import numpy as np

PI = 3.14159265358979323846


# ---- parameter selection (estimates.cpp:24-268, grid.cpp:11-77, window.cpp:76-86)

def _model_k(kind, xi, L, Q):
    b = 1.0 / (4.0 * xi * xi)
    if kind == 0:
        return 4.0 / (PI * L) * np.sqrt(Q / 3.0), 0.0, b
    if kind == 1:
        return 4.0 / (3.0 * PI * L) * np.sqrt(3.5 * Q), 1.0, b
    return np.sqrt(8.0 * xi * xi * Q / (3.0 * PI * L ** 3)), -0.5, b


def _model_r(kind, xi, L, Q):
    b = xi * xi
    L3 = L ** 3
    if kind == 0:
        return np.sqrt(4.0 * Q / L3), 0.5, b
    if kind == 1:
        return np.sqrt(112.0 * Q * b * b / (9.0 * L3)), 1.5, b
    return np.sqrt(8.0 * Q / (3.0 * L3)), -0.5, b


def _invert(m, tau, floor_value):
    """decay_solve (estimates.cpp:57-87)."""
    c, a, b = m
    at = lambda x: c * x ** a * np.exp(-b * x * x)
    res = lambda x: np.log(c) + a * np.log(x) - b * x * x - np.log(tau)
    if a > 0:
        lo = np.sqrt(a / (2 * b))
        if at(lo) <= tau:
            return lo
    elif a == 0:
        return floor_value if c <= tau else np.sqrt(np.log(c / tau) / b)
    else:
        lo = 1e-14
        if res(lo) <= 0:
            return lo
    hi = max(2 * lo, 1 / np.sqrt(b))
    while res(hi) > 0:
        hi *= 2
    x = 0.5 * (lo + hi)
    for _ in range(200):
        g = res(x)
        if abs(g) < 1e-14:
            break
        if g > 0:
            lo = x
        else:
            hi = x
        step = x - g / (a / x - 2 * b * x)
        x = step if lo < step < hi else 0.5 * (lo + hi)
    return x


def select_parameters_d3(kind, L, Q, xi, tol, f_m=4):
    """select_parameters for D = 3, PKB window (estimates.cpp:211-268)."""
    Lc = np.cbrt(L[0] * L[1] * L[2])
    t = xi * Lc
    if kind == 0:
        U = 1.8 * np.sqrt(Q) * (1 + 1.323e-2 * t + 2.469e-4 * t * t) * np.exp(-5.205 / (t * t)) / Lc
    elif kind == 1:
        U = 7.2 * np.sqrt(Q) * np.sqrt(t) / (Lc * Lc)
    else:
        U = 2.4 * np.sqrt(Q) * np.sqrt(t) * np.exp(-11.60 / (t * t)) / (Lc * Lc)
    rc = _invert(_model_r(kind, xi, Lc, Q), tol, 0.0)
    if kind == 2:
        c = _model_k(kind, xi, Lc, Q)[0]
        from scipy.special import lambertw
        kinf = xi * np.sqrt(lambertw(c ** 4 / (xi * xi * tol ** 4)).real)
    else:
        kinf = _invert(_model_k(kind, xi, Lc, Q), tol, 2 * PI / Lc)
    h = PI / kinf / 1.05
    P_est = 2 if tol >= 10 * U else max(2 * int(np.ceil(0.5 * np.log(10 * U / tol) / 2.5 - 1e-9)), 2)
    P = 2 * ((P_est + 4 + 1) // 2)
    q = np.ceil(L[0] / h / f_m - 1e-9)
    M0 = f_m * int(max(q, 1))
    hh = L[0] / M0
    M = [M0] + [int(round(L[i] / hh)) for i in (1, 2)]
    return dict(kind=kind, d=3, xi=xi, rc=rc, h=hh, M=M, P=P, beta=2.5 * P, nu=min(P // 2 + 2, 10), L=list(L))


# ---- window (window.cpp:88-162)

def kb_value(p, r):
    aw = 0.5 * p["h"] * p["P"]
    t = r / aw
    from scipy.special import i0
    out = i0(p["beta"] * np.sqrt(np.maximum(1 - t * t, 0.0))) / i0(p["beta"])
    return np.where(np.abs(r) > aw, 0.0, out)


def kb_hat(p, k):
    from scipy.special import i0
    aw = 0.5 * p["h"] * p["P"]
    s = p["beta"] ** 2 - (k * aw) ** 2
    rt = np.sqrt(np.abs(s))
    front = 2 * aw / i0(p["beta"])
    with np.errstate(invalid="ignore", divide="ignore"):
        v = np.where(s > 1e-6, np.sinh(rt) / rt, np.where(s < -1e-6, np.sin(rt) / rt, 1 + s / 6 + s * s / 120))
    return front * v


def pkb_table(p):
    """pkb_build (window.cpp:112-138): Chebyshev-extrema interpolation per cell."""
    nu, P, h = p["nu"], p["P"], p["h"]
    nodes = np.cos(np.arange(nu + 1) * PI / nu)
    V = np.vander(nodes, nu + 1, increasing=True)
    rows = []
    for l in range(-P // 2, P // 2):
        mid = l * h + 0.5 * h
        rows.append(np.linalg.solve(V, kb_value(p, mid + 0.5 * h * nodes)))
    return np.array(rows)


def pkb_value(p, tab, r):
    P, h, nu = p["P"], p["h"], p["nu"]
    l = np.clip(np.floor(r / h).astype(int), -P // 2, P // 2 - 1)
    u = 2 * (r - l * h) / h - 1
    c = tab[l + P // 2]
    acc = np.zeros_like(r)
    for i in range(nu, -1, -1):
        acc = c[..., i] + acc * u
    return np.where(np.abs(r) > 0.5 * h * P, 0.0, acc)


# ---- Fourier part, D = 3 (fourier.cpp:168-309, 330-340, 425-437, 550-563)

def _stencil(p, tab, x):
    """build_stencil (fourier.cpp:168-188): weights (n,3,P), indices (n,3,P)."""
    P, h, M = p["P"], p["h"], np.asarray(p["M"])
    rel = x / h
    j0 = np.ceil(rel - 0.5 * P).astype(int)
    j = j0[:, :, None] + np.arange(P)[None, None, :]
    w = pkb_value(p, tab, (j - rel[:, :, None]) * h)
    return w, np.mod(j, M[None, :, None])


def spread(p, x, f, nu=None):
    tab = pkb_table(p)
    w, idx = _stencil(p, tab, x)
    M = p["M"]
    fc = f if nu is None else (f[:, :, None] * nu[:, None, :]).reshape(-1, 9)
    C = fc.shape[1]
    out = np.zeros((C,) + tuple(M))
    for n in range(x.shape[0]):
        blk = np.einsum("a,b,c->abc", w[n, 0], w[n, 1], w[n, 2])
        ii = np.ix_(idx[n, 0], idx[n, 1], idx[n, 2])
        for c in range(C):
            np.add.at(out[c], ii, blk * fc[n, c])
    return out


def gather(p, field, xt):
    tab = pkb_table(p)
    w, idx = _stencil(p, tab, xt)
    u = np.zeros((xt.shape[0], 3))
    for n in range(xt.shape[0]):
        blk = np.einsum("a,b,c->abc", w[n, 0], w[n, 1], w[n, 2])
        ii = np.ix_(idx[n, 0], idx[n, 1], idx[n, 2])
        for c in range(3):
            u[n, c] = np.sum(blk * field[c][ii])
    return u * p["h"] ** 3


def _operator(kind, k):
    """diffop_hat * A(k) (kernels.cpp:118-149, modified_kernels.cpp:162-167)."""
    kk = np.sum(k * k, axis=0)
    with np.errstate(divide="ignore", invalid="ignore"):
        if kind == 2:
            base = 4 * PI / kk
        else:
            base = -8 * PI / (kk * kk)
    base = np.where(kk == 0, 0.0, base)
    if kind == 0:
        G = np.einsum("i...,j...->ij...", k, k) - np.eye(3)[:, :, None, None, None] * kk
        return G * base
    if kind == 2:
        eps = np.zeros((3, 3, 3))
        eps[0, 1, 2] = eps[1, 2, 0] = eps[2, 0, 1] = 1
        eps[0, 2, 1] = eps[2, 1, 0] = eps[1, 0, 2] = -1
        return -1j * np.einsum("jlm,m...->jl...", eps, k) * base
    d = np.eye(3)
    dl = (np.einsum("jl,m...->jlm...", d, k) + np.einsum("mj,l...->jlm...", d, k) + np.einsum("lm,j...->jlm...", d, k))
    return 1j * (-dl * kk + 2 * np.einsum("j...,l...,m...->jlm...", k, k, k)) * base


def fourier_potential(p, x, f, nu=None, xt=None):
    kind, xi, h, M = p["kind"], p["xi"], p["h"], p["M"]
    phi = spread(p, x, f, nu) * h ** 3
    F = np.fft.fftn(phi, axes=(1, 2, 3))
    ks = [2 * PI / (M[a] * h) * np.where(np.arange(M[a]) < (M[a] + 1) // 2, np.arange(M[a]), np.arange(M[a]) - M[a])
          for a in range(3)]
    K = np.array(np.meshgrid(*ks, indexing="ij"))
    kk = np.sum(K * K, 0)
    q = kk / (4 * xi * xi)
    scr = np.exp(-q) if kind == 2 else np.exp(-q) * (1 + q)
    what = [kb_hat(p, kv) for kv in ks]
    wp = what[0][:, None, None] * what[1][None, :, None] * what[2][None, None, :]
    G = _operator(kind, K)
    fac = scr / (wp * wp)
    if kind == 1:
        out = np.einsum("jlm...,lm...->j...", G, F.reshape((3, 3) + F.shape[1:])) * fac
    else:
        out = np.einsum("jl...,l...->j...", G, F) * fac
    flow = np.fft.ifftn(out, axes=(1, 2, 3)).real / h ** 3
    return gather(p, flow, x if xt is None else xt)


# ---- real space (realspace.cpp:30-93, kernels.cpp:71-116) and terms

def realspace_potential(kind, L, x, f, nu, xt, xi, rc, same):
    from scipy.special import erfc
    L = np.asarray(L, float)
    xs = np.mod(x, L)
    tgt = np.mod(x if same else xt, L)
    shells = [int(np.ceil(rc / L[a])) for a in range(3)]  # folded points: |shift| <= ceil(rc/L)
    u = np.zeros((tgt.shape[0], 3))
    for sx in range(-shells[0], shells[0] + 1):
        for sy in range(-shells[1], shells[1] + 1):
            for sz in range(-shells[2], shells[2] + 1):
                sh = np.array([sx, sy, sz]) * L
                r = (tgt[:, None, :] - xs[None, :, :]) - sh
                r2 = np.sum(r * r, -1)
                mask = r2 < rc * rc
                if same and sx == 0 and sy == 0 and sz == 0:
                    np.fill_diagonal(mask, False)
                if not mask.any():
                    continue
                ti, si = np.nonzero(mask)
                rr = r[ti, si]
                rn = np.sqrt(r2[ti, si])
                xr = xi * rn
                et = erfc(xr) / rn
                g = 2 * xi / np.sqrt(PI) * np.exp(-xr * xr)
                if kind == 0:
                    c = et + g
                    fs = f[si]
                    contrib = (c - 2 * g)[:, None] * fs + (c / rn ** 2 * np.sum(rr * fs, 1))[:, None] * rr
                elif kind == 2:
                    c = (et + g) / rn ** 2
                    contrib = c[:, None] * np.cross(f[si], rr)
                else:
                    c1 = -2 / rn ** 4 * (3 * et + (3 + 2 * xr * xr) * g)
                    c2 = 2 * xi * xi * g
                    q, v = f[si], nu[si]
                    rq, rv, qv = np.sum(rr * q, 1), np.sum(rr * v, 1), np.sum(q * v, 1)
                    contrib = (c1 * rq * rv + c2 * qv)[:, None] * rr + c2[:, None] * (q * rv[:, None] + v * rq[:, None])
                np.add.at(u, ti, contrib)
    return u


def full_potential_d3(p, x, f, nu=None):
    """full_potential for targets = sources, D = 3 (realspace.cpp:205-219)."""
    kind, xi, L = p["kind"], p["xi"], p["L"]
    u = realspace_potential(kind, L, x, f, nu, None, xi, p["rc"], True)
    u += fourier_potential(p, x, f, nu)
    if kind == 0:
        u += -4 * xi / np.sqrt(PI) * f
    if kind == 1:
        qn = np.sum(f * nu, 1)
        u += -8 * PI / np.prod(L) * (np.sum(qn) * x - np.sum(qn[:, None] * x, 0))
    return u
