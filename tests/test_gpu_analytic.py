"""GPU analytic oracles (paper_2210_01255_b200.analytic, csrc/analytic.cu):
SURVEY §8 f row 3, SPEC.md module `reference`.

The closed forms are checked against independent numerics (mpmath for the
incomplete Bessel K; numerical Fourier quadrature of the defining integrals
PAPER.md Qtilde-2p-def / 1p-k0-integral-def for the q-tensors), then the
whole oracles against the Spectral Ewald path (the product, itself pinned to
the reference at 1e-12 elsewhere) with the SPEC's acceptance bands."""
import math

import numpy as np
import pytest

import paper_2210_01255_b200 as S
from paper_2210_01255_b200 import analytic as A

pytestmark = pytest.mark.gpu

KINDS = [S.Kernel.stokeslet, S.Kernel.stresslet, S.Kernel.rotlet]


# ---------------------------------------------------------------- helpers

def gf_hat_np(kind, k, xi):
    """G^F(k) (kernels.cpp:127-149 restated in numpy), k: (n, 3) -> (n, 3, C) complex."""
    k = np.asarray(k, float)
    k2 = np.sum(k * k, -1)
    q = k2 / (4 * xi * xi)
    n = k.shape[0]
    if kind == S.Kernel.rotlet:
        sc = 4 * np.pi / k2 * np.exp(-q)
        eps = np.zeros((3, 3, 3))
        eps[0, 1, 2] = eps[1, 2, 0] = eps[2, 0, 1] = 1
        eps[0, 2, 1] = eps[2, 1, 0] = eps[1, 0, 2] = -1
        return -1j * np.einsum("jlm,nm->njl", eps, k) * sc[:, None, None]
    sc = -8 * np.pi / (k2 * k2) * np.exp(-q) * (1 + q)
    if kind == S.Kernel.stokeslet:
        return ((-k2[:, None, None] * np.eye(3)[None] + k[:, :, None] * k[:, None, :]) * sc[:, None, None]).astype(
            complex)
    I = np.eye(3)
    dl = (np.einsum("jl,nm->njlm", I, k) + np.einsum("mj,nl->njlm", I, k) + np.einsum("lm,nj->njlm", I, k))
    t = -dl * k2[:, None, None, None] + 2 * np.einsum("nj,nl,nm->njlm", k, k, k)
    return 1j * t * sc[:, None, None, None]


def rand_system(kind, d, N, seed, Q1=True, L=(1.0, 1.0, 1.0)):
    rng = np.random.default_rng(seed)
    x = rng.random((N, 3)) * np.asarray(L)
    f = rng.standard_normal((N, 3))
    nu = None
    if kind == S.Kernel.stresslet:
        g = rng.standard_normal((N, 3))
        nu = g / np.linalg.norm(g, axis=1, keepdims=True)
    sys_ = S.SourceSystem(kind, S.Cell(L), d, x, f, nu)
    if Q1:
        sys_.f = f / math.sqrt(S.source_quantity(sys_))
    return sys_


# ------------------------------------------------- incomplete Bessel K

def kb_mp(nu, a, b):
    """K_nu(a, b) by mpmath Gauss-Legendre in s = ln t over the interval where
    the integrand is within e^-60 of its peak (25 digits)."""
    import mpmath as mp
    mp.mp.dps = 25
    grid = np.arange(0.0, 60.0, 0.05)
    psi = a * np.exp(grid) + b * np.exp(-grid) + nu * grid
    keep = grid[psi - psi.min() < 60.0]
    lo, hi = max(0.0, keep[0] - 0.05), keep[-1] + 0.05
    pts = [lo + (hi - lo) * i / 24 for i in range(25)]
    return float(mp.quad(lambda s: mp.exp(-a * mp.exp(s) - b * mp.exp(-s) - nu * s), pts, method="gauss-legendre"))


def test_incomplete_bessel_k4_vs_mpmath():
    pts = [(0.0987, 0.0), (0.0987, 1e-6), (0.0987, 0.37), (0.5, 3.0), (2.0, 0.01), (0.01, 50.0),
           (3.9, 120.0), (25.0, 0.2), (0.3, 200.0), (1e-3, 1e-3), (7.0, 7.0)]
    a = np.array([p[0] for p in pts])
    b = np.array([p[1] for p in pts])
    K = A.incomplete_bessel_K4(a, b)
    worst = 0.0
    for i, (ai, bi) in enumerate(pts):
        for q, nu in enumerate((-1, 0, 1, 2)):
            ref = kb_mp(nu, ai, bi)
            worst = max(worst, abs(K[i, q] - ref) / abs(ref))
    print(f"K4 worst rel err vs mpmath: {worst:.2e}")
    assert worst < 1e-13


def test_incomplete_bessel_identities():
    from scipy.special import kv
    rng = np.random.default_rng(5)
    a = 10 ** rng.uniform(-2, 1.3, 200)
    b = 10 ** rng.uniform(-3, 2, 200)
    K = A.incomplete_bessel_K4(a, b)
    Ks = A.incomplete_bessel_K4(b, a)
    # a K_{-1}(a,b) - b K_1(a,b) = e^{-a-b}   (Harris 2008, PAPER.md after 1p-QB-nonzero)
    lhs = a * K[:, 0] - b * K[:, 2]
    # relative to the terms (the difference cancels down to e^{-a-b})
    assert np.max(np.abs(lhs - np.exp(-a - b)) / (a * K[:, 0])) < 1e-13
    # K_1(a,b) + K_{-1}(b,a) = 2 sqrt(a/b) K_1(2 sqrt(ab))   (PAPER.md 1p-Bbar-R-limit)
    rhs = 2 * np.sqrt(a / b) * kv(1, 2 * np.sqrt(a * b))
    assert np.max(np.abs(K[:, 2] + Ks[:, 0] - rhs) / np.abs(rhs)) < 1e-12
    # K_nu(a, 0) = E_{nu+1}(a)
    from scipy.special import expn
    K0 = A.incomplete_bessel_K4(a[:50], np.zeros(50))
    for q, nu in ((1, 0), (2, 1), (3, 2)):
        assert np.max(np.abs(K0[:, q] - expn(nu + 1, a[:50])) / expn(nu + 1, a[:50])) < 1e-13
    assert np.max(np.abs(K0[:, 0] - np.exp(-a[:50]) / a[:50]) * a[:50] / np.exp(-a[:50])) < 1e-13


# ------------------------------------------------------- q tensors

@pytest.mark.parametrize("kind", KINDS)
def test_q2p_matches_fourier_quadrature(kind):
    """Q^{2P}(k1,k2,r3) = (1/2pi) int G^F(k1,k2,kappa3) e^{i kappa3 r3} dkappa3 (PAPER.md Qtilde-2p-def)."""
    xi = 4.0
    h = 0.01
    kap = np.arange(-40 * xi, 40 * xi + h / 2, h)
    for (k1, k2, r3) in [(2 * np.pi, 0.0, 0.3), (2 * np.pi, -4 * np.pi, -0.17), (-6 * np.pi, 2 * np.pi, 0.0)]:
        kk = np.stack([np.full_like(kap, k1), np.full_like(kap, k2), kap], -1)
        G = gf_hat_np(kind, kk, xi)
        ph = np.exp(1j * kap * r3)
        ref = h / (2 * np.pi) * np.tensordot(ph, G, axes=(0, 0))
        Q = A.q2p(kind, k1, k2, r3, xi)[0]
        Q = Q.reshape(ref.shape)
        err = np.max(np.abs(Q - ref)) / np.max(np.abs(ref))
        assert err < 1e-11, (k1, k2, r3, err)


@pytest.mark.parametrize("kind", KINDS)
def test_q1p_matches_fourier_quadrature(kind):
    """Q^{1P}(k1,r2,r3) = (2pi)^-2 int int G^F(k1,kappa2,kappa3) e^{i(kappa2 r2 + kappa3 r3)} (PAPER.md QA-1p-def)."""
    xi = 5.0
    h = 0.1
    kap = np.arange(-14 * xi, 14 * xi + h / 2, h)
    K2, K3 = np.meshgrid(kap, kap, indexing="ij")
    for (k1, r2, r3) in [(2 * np.pi, 0.1, 0.2), (-4 * np.pi, -0.05, 0.33), (2 * np.pi, 0.0, 0.0)]:
        kk = np.stack([np.full(K2.size, k1), K2.ravel(), K3.ravel()], -1)
        G = gf_hat_np(kind, kk, xi)
        ph = np.exp(1j * (K2.ravel() * r2 + K3.ravel() * r3))
        ref = h * h / (2 * np.pi) ** 2 * np.tensordot(ph, G, axes=(0, 0))
        Q = A.q1p(kind, k1, r2, r3, xi)[0].reshape(ref.shape)
        err = np.max(np.abs(Q - ref)) / np.max(np.abs(ref))
        assert err < 1e-10, (k1, r2, r3, err)


def test_q_tensor_structure_and_limits():
    rng = np.random.default_rng(3)
    k1, k2, r3 = rng.uniform(-20, 20, 8), rng.uniform(-20, 20, 8), rng.uniform(-0.5, 0.5, 8)
    Qs = A.q2p(S.Kernel.stokeslet, k1, k2, r3, 6.0)
    assert np.allclose(Qs, np.transpose(Qs, (0, 2, 1)), atol=0)
    Qr = A.q2p(S.Kernel.rotlet, k1, k2, r3, 6.0)
    assert np.allclose(Qr, -np.transpose(Qr, (0, 2, 1)), atol=0)
    Qt = A.q2p(S.Kernel.stresslet, k1, k2, r3, 6.0)
    for p in [(0, 2, 1, 3), (0, 3, 2, 1), (0, 1, 3, 2)]:
        assert np.allclose(Qt, np.transpose(Qt, p), atol=0)
    xi = 7.0
    # q2p_zero stokeslet at r3 = 0: -2 pi / (sqrt(pi) xi) diag(1, 1, 0)   (SPEC.md example)
    Z = A.q2p_zero(S.Kernel.stokeslet, 0.0, xi)[0]
    assert np.allclose(Z.real, -2 * np.pi / (math.sqrt(np.pi) * xi) * np.diag([1, 1, 0]), rtol=1e-15, atol=1e-15)
    # q1p_zero stokeslet as rho -> 0: (gamma + ln xi^2 - 1) diag(2, 1, 1)   (PAPER.md 1p-stokeslet-Q0-limit)
    lim = (np.euler_gamma + math.log(xi * xi) - 1) * np.diag([2, 1, 1])
    for rho in (0.0, 1e-9):
        Z = A.q1p_zero(S.Kernel.stokeslet, rho, 0.0, xi)[0]
        assert np.allclose(Z.real, lim, rtol=1e-12, atol=1e-12)
    # continuity of phi0 across the series / continued-fraction switch (V = 1)
    r = np.array([0.999999, 1.000001]) / xi
    Z = A.q1p_zero(S.Kernel.stokeslet, r, 0.0, xi)
    assert abs(Z[0, 1, 1].real - Z[1, 1, 1].real) < 1e-5
    # q1p_zero stresslet / rotlet at rho = 0: zero tensor (PAPER.md 1p-stresslet-Q0-limit)
    assert np.all(A.q1p_zero(S.Kernel.stresslet, 0.0, 0.0, xi) == 0)
    assert np.all(A.q1p_zero(S.Kernel.rotlet, 0.0, 0.0, xi) == 0)
    # zero-mode parity classes: rotlet (2P) odd in r3, stokeslet even
    a = A.q2p_zero(S.Kernel.rotlet, [0.2, -0.2], xi)
    assert np.allclose(a[0], -a[1])
    b = A.q2p_zero(S.Kernel.stokeslet, [0.2, -0.2], xi)
    assert np.allclose(b[0], b[1])
    with pytest.raises(S.DomainError):
        A.q2p(S.Kernel.stokeslet, 0.0, 0.0, 0.1, xi)


# --------------------------------------------------- whole oracles

def test_rms_error_examples():
    u = np.random.default_rng(1).standard_normal((7, 3))
    assert A.rms_error(u, u) == 0.0
    assert A.rel_rms_error(2 * u, u) == pytest.approx(1.0, rel=1e-15)
    assert A.rms_error([[3, 4, 0]], [[0, 0, 0]]) == 5.0
    assert A.rel_rms_error([[6, 8, 0]], [[3, 4, 0]]) == pytest.approx(1.0)
    with pytest.raises(S.InvalidArgument):
        A.rms_error(np.zeros((0, 3)), np.zeros((0, 3)))
    with pytest.raises(S.DomainError):
        A.rel_rms_error(u, np.zeros_like(u))


@pytest.mark.parametrize("kind", KINDS)
def test_direct_sum_0p(kind):
    rng = np.random.default_rng(11)
    # N = 1, target far away -> bare kernel value
    x = np.zeros((1, 3))
    f = np.array([[0.3, -1.2, 0.7]])
    nu = np.array([[0.0, 0.6, 0.8]]) if kind == S.Kernel.stresslet else None
    s1 = S.SourceSystem(kind, S.Cell((1, 1, 1)), 0, x, f, nu)
    xt = np.array([[3.0, -4.0, 12.0]])
    u = A.direct_sum_0p(s1, S.TargetSet(xt), False)[0]
    r = xt[0]
    rn = np.linalg.norm(r)
    if kind == S.Kernel.stokeslet:
        ref = f[0] / rn + r * (r @ f[0]) / rn ** 3
    elif kind == S.Kernel.rotlet:
        ref = np.cross(f[0], r) / rn ** 3
    else:
        ref = -6 * r * (r @ f[0]) * (r @ nu[0]) / rn ** 5
    assert np.allclose(u, ref, rtol=1e-15, atol=0)
    # superposition
    sys2 = rand_system(kind, 0, 2, 4, Q1=False)
    xt = rng.random((5, 3)) + 2.0
    ua = A.direct_sum_0p(S.SourceSystem(kind, sys2.cell, 0, sys2.x[:1], sys2.f[:1],
                                        None if sys2.nu is None else sys2.nu[:1]), S.TargetSet(xt), False)
    ub = A.direct_sum_0p(S.SourceSystem(kind, sys2.cell, 0, sys2.x[1:], sys2.f[1:],
                                        None if sys2.nu is None else sys2.nu[1:]), S.TargetSet(xt), False)
    uab = A.direct_sum_0p(sys2, S.TargetSet(xt), False)
    assert np.allclose(ua + ub, uab, rtol=1e-14, atol=1e-15)
    # coincident unstarred -> singularity error; starred skips the self pair
    with pytest.raises(S.DomainError):
        A.direct_sum_0p(sys2, S.TargetSet(sys2.x), False)
    us = A.direct_sum_0p(sys2, S.TargetSet.from_sources(sys2), True)
    assert np.allclose(us[0], A.direct_sum_0p(S.SourceSystem(kind, sys2.cell, 0, sys2.x[1:], sys2.f[1:],
                                                             None if sys2.nu is None else sys2.nu[1:]),
                                              S.TargetSet(sys2.x[:1]), False)[0], rtol=1e-15, atol=0)


def test_rotlet_antisymmetry_direct():
    # Omega(-r) = -Omega(r): swapping source and target with f fixed flips the field
    f = np.array([[0.2, 0.5, -0.9]])
    a, b = np.array([[0.1, 0.2, 0.3]]), np.array([[0.7, -0.4, 0.25]])
    u1 = A.direct_sum_0p(S.SourceSystem(S.Kernel.rotlet, S.Cell((1, 1, 1)), 0, a, f), S.TargetSet(b), False)
    u2 = A.direct_sum_0p(S.SourceSystem(S.Kernel.rotlet, S.Cell((1, 1, 1)), 0, b, f), S.TargetSet(a), False)
    assert np.allclose(u1, -u2, rtol=1e-15, atol=0)


def _se_params(system, tol=1e-8, xi=10.0):
    sel = S.select_parameters(system.kind, system.d, system.cell, S.source_quantity(system), xi,
                              S.ToleranceSpec(tol))
    return sel.params


@pytest.mark.parametrize("d", [3, 2, 1])
@pytest.mark.parametrize("kind", KINDS)
def test_fourier_oracle_vs_spectral_ewald(kind, d):
    """SPEC acceptance 1: uniform N = 1000, L = 1, Q = 1, xi = 10, tau = 1e-8:
    the Spectral Ewald Fourier part against the matching oracle lies in the
    paper's one-order-of-magnitude band [1e-9, 1e-7]."""
    system = rand_system(kind, d, 1000, 100 + 10 * d + int(kind))
    p = _se_params(system)
    T = S.TargetSet.from_sources(system)
    u_se = S.se_fourier_potential(system, T, p)
    u_or = A.fourier_reference_potential(system, T, 10.0)
    if kind == S.Kernel.stresslet and d == 3:
        # the oracle includes the zero mode; se_fourier_potential
        # leaves it to full_potential (kernels.cpp stresslet_zero_mode_3p)
        qn = np.sum(system.f * system.nu, 1)
        u_or = u_or + 8 * np.pi * (qn.sum() * system.x - qn @ system.x)
    err = A.rms_error(u_se, u_or)
    rms = math.sqrt(np.mean(np.sum(u_or ** 2, 1)))
    print(f"{kind.name} d={d}: rms(u_F)={rms:.3f} abs err={err:.2e}")
    assert 1e-10 <= err <= 1e-7


@pytest.mark.parametrize("kind", KINDS)
def test_direct_0p_vs_spectral_ewald(kind):
    """D = 0: the full SE potential against the direct sum (SPEC acceptance 1, D = 0)."""
    system = rand_system(kind, 0, 1000, 300 + int(kind))
    p = _se_params(system)
    T = S.TargetSet.from_sources(system)
    u = S.full_potential(system, T, p)
    ref = A.direct_sum_0p(system, T, True)
    err = A.rms_error(u, ref)
    print(f"{kind.name} d=0: rms(u)={math.sqrt(np.mean(np.sum(ref ** 2, 1))):.3f} abs err={err:.2e}")
    assert 1e-10 <= err <= 1e-7


def test_fourier_oracle_truncation_converges():
    """More modes change the oracle by less than the omitted tail."""
    system = rand_system(S.Kernel.stokeslet, 2, 200, 7)
    T = S.TargetSet(np.random.default_rng(8).random((50, 3)))
    a = A.fourier_reference_potential(system, T, 6.0, kmax=14)
    b = A.fourier_reference_potential(system, T, 6.0, kmax=20)
    assert A.rms_error(a, b) < 1e-13 * max(1.0, np.abs(b).max())


@pytest.mark.parametrize("d", [0, 1, 2, 3])
def test_stresslet_identity(d):
    """PAPER.md:1218 / SPEC acceptance 7: sphere of radius 0.2 in the unit cell,
    Gauss-Legendre order 32, tau = 1e-10: interior / exterior values."""
    center = np.array([0.5, 0.5, 0.5])
    x, n, w = A.sphere_quadrature(center, 0.2, 32)
    system = S.SourceSystem(S.Kernel.stresslet, S.Cell((1, 1, 1)), d, x, w[:, None] * np.array([[1.0, 0, 0]]), n)
    p = _se_params(system, tol=1e-10, xi=12.0)
    inner = np.array([[0.5, 0.5, 0.5], [0.55, 0.47, 0.52]])
    outer = np.array([[0.9, 0.5, 0.5], [0.5, 0.1, 0.85]])
    ri = A.stresslet_identity_check(d, center, 0.2, 32, inner, p, expected=8 * np.pi)
    ro = A.stresslet_identity_check(d, center, 0.2, 32, outer, p, expected=0.0)
    print(f"d={d}: interior {ri}, exterior {ro}")
    assert np.all(ri < 1e-5) and np.all(ro < 1e-5)
