"""Parity at the BASELINE sizes against the reference itself.

tests/golden/fullsize_<tag>.npz was written by oracle/make_fullsize_golden.py:
the unmodified reference (oracle/_ref) ran the config once on the seeded
inputs (full_potential as realspace.cpp:205-219 assembles it, with
se_fourier_potential (fourier.cpp:805-852) and the starred
realspace_potential (realspace.cpp:166-203) kept separately). The fixture
holds u, u_F, u_R at >= 10,240 sampled targets and, over ALL targets, sums
of squares and eight seeded random projections sum_i w_i . u_i.

Bar (BASELINE north_star): rms(u_gpu - u_ref) / rms(u_ref) <= 1e-12 on u, and
on u_F and u_R separately. A projection difference is a sum of the per-target
errors with N(0,1) weights, so its size is ~ rel_rms * sqrt(sum |u|^2): the
projections are held to 5e-12 of sqrt(sum |u|^2) (5 sigma at the 1e-12 bar),
which a wrong value at any single target would break.
"""
import glob
import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_rms

FIXTURES = sorted(glob.glob(os.path.join(GOLDEN, "fullsize_*.npz")))
TOL = 1e-12


def _inputs(cfg_index, N, Nt):
    from paper_2210_01255_b200.workloads import CONFIGS, generate
    cfg = CONFIGS[cfg_index]
    x, f, nu, xt = generate(cfg, N, Nt)
    return cfg, x, f, nu, xt


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        if a is not None:
            h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def _projections(u, seed, n=8):
    rng = np.random.default_rng(seed)
    return np.array([float(np.sum(rng.standard_normal(u.shape) * u)) for _ in range(n)])


def test_fixtures_present():
    tags = {os.path.basename(p)[len("fullsize_"):-4] for p in FIXTURES}
    assert "c2" in tags, tags


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p)[9:-4] for p in FIXTURES])
def test_fullsize_inputs_and_params(S, path):
    """CPU: the product's workload generator draws the fixture's exact input
    bytes, and the product's select_parameters picks the reference's exact
    parameter struct (bytes) for them."""
    g = np.load(path)
    N = int(g["N"])
    Nt = int(g["Nt"])
    cfg, x, f, nu, xt = _inputs(int(g["config"]), N, Nt if int(g["config"]) == 4 else None)
    assert _sha(x, f, nu, xt) == str(g["input_sha256"])
    sysm = S.SourceSystem(cfg.kind, S.Cell(cfg.L), cfg.d, x, f, nu)
    assert abs(S.source_quantity(sysm) - float(g["Q"])) <= 1e-12 * float(g["Q"])
    sel = S.select_parameters(cfg.kind, cfg.d, sysm.cell, float(g["Q_sel"]), cfg.xi, S.ToleranceSpec(cfg.tol),
                              S.SelectionOptions(4, cfg.window, True))
    assert bytes(sel.params.to_c()) == bytes(g["params"])


@pytest.mark.gpu
@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p)[9:-4] for p in FIXTURES])
def test_fullsize_parity(S, path):
    g = np.load(path)
    cfg_index = int(g["config"])
    cfg, x, f, nu, xt = _inputs(cfg_index, int(g["N"]), int(g["Nt"]) if cfg_index == 4 else None)
    assert _sha(x, f, nu, xt) == str(g["input_sha256"])
    p = S.EwaldParams.from_c(S.api.sewald_params_c.from_buffer_copy(bytes(g["params"])))
    sysm = S.SourceSystem(cfg.kind, S.Cell(cfg.L), cfg.d, x, f, nu)
    tg = S.TargetSet.from_sources(sysm) if xt is None else S.TargetSet(xt, False)
    u = S.full_potential(sysm, tg, p)
    uF = S.se_fourier_potential(sysm, tg, p)
    uR = S.realspace_potential(sysm, tg, p.xi, p.rc, tg.same_as_sources)
    idx = g["idx"]
    seed = int(g["proj_seed"])
    report = []
    for name, val in (("u", u), ("uF", uF), ("uR", uR)):
        r = rel_rms(val[idx], g[name])
        ss_ref = float(g["ss_" + name])
        pj = _projections(val, seed)
        pdev = float(np.max(np.abs(pj - g["proj_" + name]))) / np.sqrt(ss_ref)
        ssdev = abs(float(np.sum(val * val)) - ss_ref) / ss_ref
        report.append(f"{name}: sampled rel_rms={r:.2e} proj={pdev:.2e} ss={ssdev:.2e}")
        assert r < TOL, (name, r)
        assert pdev < 5 * TOL, (name, pdev)
        assert ssdev < 3 * TOL, (name, ssdev)
    print(f"{os.path.basename(path)}: " + "; ".join(report))
