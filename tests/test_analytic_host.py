"""CPU tests of the analytic-oracle host layer (paper_2210_01255_b200.analytic):
the rms errors (computed by the C-ABI on the host), the
sphere quadrature of the stresslet identity harness and the truncation rule.
The oracle sums themselves run on the GPU (tests/test_gpu_analytic.py)."""
import math

import numpy as np
import pytest


def test_rms_error_examples(S):
    from paper_2210_01255_b200 import analytic as A
    u = np.random.default_rng(2).standard_normal((9, 3))
    assert A.rms_error(u, u) == 0.0
    assert A.rel_rms_error(2 * u, u) == pytest.approx(1.0, rel=1e-15)
    # single target, u - u_ref = (3, 4, 0), |u_ref| = 5 -> abs 5, rel 1   (SPEC.md example)
    assert A.rms_error([[3.0, 4.0, 0.0]], [[0.0, 0.0, 0.0]]) == 5.0
    assert A.rel_rms_error([[6.0, 8.0, 0.0]], [[3.0, 4.0, 0.0]]) == pytest.approx(1.0, rel=1e-15)
    with pytest.raises(S.InvalidArgument):
        A.rms_error(np.zeros((0, 3)), np.zeros((0, 3)))
    with pytest.raises(S.InvalidArgument):
        A.rms_error(np.zeros((2, 3)), np.zeros((3, 3)))
    with pytest.raises(S.DomainError):
        A.rel_rms_error(u, np.zeros_like(u))


def test_sphere_quadrature_exact_moments(S):
    from paper_2210_01255_b200 import analytic as A
    c = np.array([0.3, 0.4, 0.5])
    x, n, w = A.sphere_quadrature(c, 0.2, 16)
    assert np.allclose(np.linalg.norm(x - c, axis=1), 0.2, rtol=1e-15)
    assert np.allclose(n, (x - c) / 0.2, atol=1e-15)
    assert w.sum() == pytest.approx(4 * math.pi * 0.04, rel=1e-14)
    # int n_i n_j dS = (4 pi R^2 / 3) delta_ij ; int n dS = 0
    assert np.allclose(np.einsum("n,ni,nj->ij", w, n, n), 4 * math.pi * 0.04 / 3 * np.eye(3), atol=1e-15)
    assert np.allclose(w @ n, 0, atol=1e-15)


def test_kmax_rule(S):
    from paper_2210_01255_b200 import analytic as A
    km = A.kmax_for(10.0, [1.0, 2.0, 0.5])
    for k, L in zip(km, [1.0, 2.0, 0.5]):
        kk = 2 * math.pi * (k - 1) / L
        assert math.exp(-kk * kk / 400.0) < math.exp(-39.0)
