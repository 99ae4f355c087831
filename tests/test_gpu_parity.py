"""GPU parity: the CUDA path (through the C-ABI) against the reference.

Bar (BASELINE.json north_star): rms(u_gpu - u_ref) / rms(u_ref) <= 1e-12 on
the full velocity, fp64. Fixtures in tests/golden were produced by the
reference itself (oracle/make_golden.py); the live cases call the compiled
reference (oracle/_ref) when it is present.
"""
import ctypes as C

import numpy as np
import pytest

from conftest import load_golden, rel_rms

pytestmark = pytest.mark.gpu

TOL = 1e-12


def params_from_bytes(S, raw):
    c = S.api.sewald_params_c.from_buffer_copy(bytes(raw))
    return S.EwaldParams.from_c(c)


def system_from(S, g):
    nu = g.get("nu")
    return S.SourceSystem(S.Kernel(int(g["kind"])), S.Cell(tuple(g["L"])), int(g["d"]), g["x"], g["f"], nu)


def targets_from(S, g, system):
    if "xt" in g:
        return S.TargetSet(g["xt"], False)
    return S.TargetSet.from_sources(system)


@pytest.mark.parametrize("name,tag", [
    ("c1_stokeslet_d3", ""), ("c1_stokeslet_d3", "_xi10"), ("stresslet_d3", ""), ("rotlet_d3", ""),
])
def test_golden_full_d3(S, name, tag):
    g = load_golden(name)
    sysm = system_from(S, g)
    tg = targets_from(S, g, sysm)
    params = params_from_bytes(S, g["params" + tag])
    # the product selects the identical parameter set
    sel = S.select_parameters(sysm.kind, sysm.d, sysm.cell, float(g["Q"]), params.xi,
                              S.ToleranceSpec(float(g["tol"])),
                              S.SelectionOptions(4, S.WindowKind(int(g["window"])), True))
    assert bytes(sel.params.to_c()) == bytes(params.to_c())
    u = S.full_potential(sysm, tg, params)
    uF = S.se_fourier_potential(sysm, tg, params)
    uR = S.realspace_potential(sysm, tg, params.xi, params.rc, tg.same_as_sources)
    assert rel_rms(uR, g["uR" + tag]) < TOL
    assert rel_rms(uF, g["uF" + tag]) < TOL
    assert rel_rms(u, g["u" + tag]) < TOL


@pytest.mark.parametrize("name", ["stresslet_d2", "stokeslet_d2", "rotlet_d1_tg", "stokeslet_d1", "stokeslet_d0"])
def test_golden_realspace_free_axes(S, name):
    g = load_golden(name)
    sysm = system_from(S, g)
    tg = targets_from(S, g, sysm)
    params = params_from_bytes(S, g["params"])
    uR = S.realspace_potential(sysm, tg, params.xi, params.rc, tg.same_as_sources)
    assert rel_rms(uR, g["uR"]) < TOL


@pytest.mark.parametrize("name", ["spread_kb_d3", "spread_pkb_d2_stresslet", "spread_tg_d0"])
def test_golden_spread_gather(S, name):
    g = load_golden(name)
    params = params_from_bytes(S, g["params"])
    kind = params.kind
    sysm = S.SourceSystem(kind, S.Cell(tuple(params.grid.L)), params.d, g["x"], g["f"], g.get("nu"))
    grid = S.spread(sysm, params)
    ref = g["grid"]
    assert np.max(np.abs(grid - ref)) <= 1e-14 * np.max(np.abs(ref))
    ug = S.gather(g["field"], params, S.TargetSet(g["xt"], False))
    assert np.max(np.abs(ug - g["ug"])) <= 1e-13 * np.max(np.abs(g["ug"]))


def test_smoke_entry():
    import __graft_entry__
    __graft_entry__.smoke()


# ---------------------------------------------------------------------------
# live comparisons against the compiled reference (skipped without oracle/_ref)
# ---------------------------------------------------------------------------

@pytest.mark.oracle
@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("window", [0, 1, 2])
def test_live_d3_windows(S, ref, kind, window):
    rng = np.random.default_rng(100 + 3 * kind + window)
    N = 300
    x = rng.random((N, 3))
    f = rng.standard_normal((N, 3))
    nu = rng.standard_normal((N, 3)) if kind == 1 else None
    sysm = S.SourceSystem(S.Kernel(kind), S.Cell((1, 1, 1)), 3, x, f, nu)
    sel = S.select_parameters(sysm.kind, 3, sysm.cell, S.source_quantity(sysm), 7.0, S.ToleranceSpec(1e-9),
                              S.SelectionOptions(4, S.WindowKind(window), True))
    rp = ref.params_from(sel.params.to_c())
    xt = rng.random((77, 3)) * 1.3 - 0.15  # targets outside the primary cell too
    for same in (True, False):
        tg = S.TargetSet.from_sources(sysm) if same else S.TargetSet(xt, False)
        u = S.full_potential(sysm, tg, sel.params)
        ur = ref.full_potential(rp, x, f, nu, None if same else xt, same)
        assert rel_rms(u, ur) < TOL, (kind, window, same)


@pytest.mark.oracle
@pytest.mark.parametrize("case", [
    # (kind, d, L, n, rc, own_targets) — test_realspace.cpp:328-336 shapes
    (0, 3, (1.0, 1.0, 1.0), 400, 0.2, True),
    (1, 3, (1.0, 1.0, 1.0), 400, 0.2, True),
    (2, 3, (1.0, 1.0, 1.0), 400, 0.2, True),
    (0, 3, (1.0, 1.0, 1.0), 60, 1.4, True),
    (1, 2, (1.0, 1.3, 0.8), 200, 0.35, False),
    (2, 1, (1.0, 0.7, 0.7), 150, 0.3, True),
    (0, 0, (1.0, 1.0, 1.0), 150, 0.45, False),
    (0, 3, (1.0, 1.0, 1.0), 40, 2e-3, True),
])
def test_live_realspace_cases(S, ref, case):
    kind, d, L, n, rc, own = case
    rng = np.random.default_rng(57120848 + n)
    x = np.empty((n, 3))
    for ax in range(3):
        x[:, ax] = (rng.random(n) if ax < d else rng.uniform(-0.4, 0.6, n)) * L[ax]
    f = rng.uniform(-1, 1, (n, 3))
    nu = rng.uniform(-1, 1, (n, 3)) if kind == 1 else None
    sysm = S.SourceSystem(S.Kernel(kind), S.Cell(L), d, x, f, nu)
    xt = rng.uniform(-0.6, 0.8, (40, 3)) * np.asarray(L)
    tg = S.TargetSet.from_sources(sysm) if own else S.TargetSet(xt, False)
    u = S.realspace_potential(sysm, tg, 3.0, rc, True)
    ur = ref.realspace_potential(kind, d, L, x, f, nu, None if own else xt, own, 3.0, rc, True)
    scale = max(np.max(np.abs(ur)), 1e-300)
    assert np.max(np.abs(u - ur)) / scale <= 1e-13


@pytest.mark.oracle
@pytest.mark.parametrize("M", [20, 24, 44, 60])
def test_live_d3_grid_sizes(S, ref, M):
    """Grid sizes not multiple of the spread tile, KB window P=14 (test_fourier.cpp:468-505 grid)."""
    rng = np.random.default_rng(M)
    N = 200
    x = rng.random((N, 3))
    f = rng.standard_normal((N, 3))
    p = S.EwaldParams(S.Kernel.stokeslet, 3, 6.0, 0.3)
    p.grid = S.GridSpec(3, 1.0 / M, (M, M, M), (M, M, M), (1, 1, 1), (1, 1, 1), (0, 0, 0), 4)
    p.window = S.WindowSpec.make(S.WindowKind.kb, 14, 1.0 / M)
    sysm = S.SourceSystem(S.Kernel.stokeslet, S.Cell((1, 1, 1)), 3, x, f)
    tg = S.TargetSet.from_sources(sysm)
    uF = S.se_fourier_potential(sysm, tg, p)
    ur = ref.fourier_potential(ref.params_from(p.to_c()), x, f)
    assert rel_rms(uF, ur) < TOL


# ---------------------------------------------------------------------------
# error behaviour (the reference's exception types)
# ---------------------------------------------------------------------------

def test_errors(S):
    sysm = S.SourceSystem(S.Kernel.stokeslet, S.Cell((1, 1, 1)), 3,
                          np.random.default_rng(0).random((5, 3)), np.ones((5, 3)))
    tg = S.TargetSet.from_sources(sysm)
    with pytest.raises(S.DomainError):  # test_realspace.cpp:429-435
        S.realspace_potential(sysm, tg, 3.0, 0.3, False)
    S.realspace_potential(sysm, tg, 3.0, 0.3, True)
    with pytest.raises(S.InvalidArgument):
        S.realspace_potential(sysm, tg, 0.0, 0.3, True)
    bad = S.TargetSet(np.array([[0.5, 0.5, 0.5], [np.nan, 0.0, 0.0]]), False)
    with pytest.raises(S.InvalidArgument):
        S.realspace_potential(sysm, bad, 1.0, 0.3, False)
    # spread outside the extended box on a free axis (test_fourier.cpp:174-187)
    h = 1 / 16
    p = S.EwaldParams(S.Kernel.stokeslet, 0, 5.0, 0.3)
    p.grid = S.GridSpec(0, h, (8, 8, 8), (16, 16, 16), (0.5, 0.5, 0.5), (1, 1, 1), (0.5, 0.5, 0.5), 4)
    p.window = S.WindowSpec.make(S.WindowKind.kb, 10, h)
    s0 = S.SourceSystem(S.Kernel.stokeslet, S.Cell((0.5, 0.5, 0.5)), 0, np.array([[0.49, 0.25, 0.25]]),
                        np.array([[1.0, 0, 0]]))
    with pytest.raises(S.InvalidArgument):
        S.spread(s0, p)


def test_zero_strengths_exact_zero(S):
    rng = np.random.default_rng(5)
    x = rng.random((50, 3))
    sysm = S.SourceSystem(S.Kernel.stokeslet, S.Cell((1, 1, 1)), 3, x, np.zeros((50, 3)))
    sel = S.select_parameters(S.Kernel.stokeslet, 3, sysm.cell, 1.0, 6.0)
    u = S.full_potential(sysm, S.TargetSet.from_sources(sysm), sel.params)
    assert np.all(u == 0.0)


def test_empty_inputs(S):
    sysm = S.SourceSystem(S.Kernel.stokeslet, S.Cell((1, 1, 1)), 3, np.zeros((0, 3)), np.zeros((0, 3)))
    sel = S.select_parameters(S.Kernel.stokeslet, 3, sysm.cell, 1.0, 6.0)
    u = S.full_potential(sysm, S.TargetSet.from_sources(sysm), sel.params)
    assert u.shape == (0, 3)
    xt = np.random.default_rng(1).random((10, 3))
    u = S.full_potential(sysm, S.TargetSet(xt, False), sel.params)
    assert np.all(u == 0.0)


# ---------------------------------------------------------------------------
# free directions (d = 2, 1, 0): mode classes, truncated kernels, D=0 table
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["stresslet_d2", "stokeslet_d2", "rotlet_d1_tg", "stokeslet_d1", "stokeslet_d0"])
def test_golden_full_free_axes(S, name):
    g = load_golden(name)
    sysm = system_from(S, g)
    tg = targets_from(S, g, sysm)
    params = params_from_bytes(S, g["params"])
    uF = S.se_fourier_potential(sysm, tg, params)
    assert rel_rms(uF, g["uF"]) < TOL
    if "uF_direct" in g:
        uFd = S.se_fourier_potential(sysm, tg, params, S.SePipelineOptions(precompute_0p=False))
        assert rel_rms(uFd, g["uF_direct"]) < TOL
    u = S.full_potential(sysm, tg, params)
    assert rel_rms(u, g["u"]) < TOL


def _test_grid(S, d, h, M, Mext):
    L = tuple(h * m for m in M)
    Le = tuple(h * m for m in Mext)
    return S.GridSpec(d, h, M, Mext, L, Le, tuple(a - b for a, b in zip(Le, L)), 4)


@pytest.mark.oracle
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_live_reference_test_grids(S, ref, kind):
    """The reference's own hand-built grids (test_fourier.cpp:507-724)."""
    cases = []
    # planar periodic: M=(8,8,4), M_ext=(8,8,12), s0=2, s*=1.5, k*=(2,2,0)
    g2 = _test_grid(S, 2, 1 / 8, (8, 8, 4), (8, 8, 12))
    cases.append((2, g2, (1.0, 1.0, 0.5), 2.5, 10, S.UpsamplingPlan(2.0, 1.5, (2, 2, 0)), 1.5, (0.2, 0.7), True))
    # singly periodic: M=(8,4,4), M_ext=(8,12,12), s0=8/3, s*=1.5, k*=(2,0,0)
    g1 = _test_grid(S, 1, 1 / 8, (8, 4, 4), (8, 12, 12))
    cases.append((1, g1, (1.0, 0.5, 0.5), 3.0, 10, S.UpsamplingPlan(8 / 3, 1.5, (2, 0, 0)), 1.5 * np.sqrt(2), (0.2, 0.7), True))
    # free space: M=(8,8,8), M_ext=(16,16,16), s0=3 (direct) and table path
    g0 = _test_grid(S, 0, 1 / 16, (8, 8, 8), (16, 16, 16))
    cases.append((0, g0, (0.5, 0.5, 0.5), 5.0, 12, S.UpsamplingPlan(3.0), np.sqrt(3.0), (0.3, 0.7), False))
    cases.append((0, g0, (0.5, 0.5, 0.5), 5.0, 12, S.UpsamplingPlan(3.0), np.sqrt(3.0), (0.3, 0.7), True))
    g0b = _test_grid(S, 0, 1 / 16, (8, 8, 8), (32, 32, 32))
    cases.append((0, g0b, (0.5, 0.5, 0.5), 5.0, 12, S.UpsamplingPlan(2.75), 2 * np.sqrt(3.0), (0.3, 0.7), True))
    rng = np.random.default_rng(71 + kind)
    for d, grid, L, xi, P, plan, R, (lo, hi), table in cases:
        if d == 1 and kind == 1:
            continue  # the reference's singly periodic test covers stokeslet and rotlet
        n = 6
        x = np.empty((n, 3))
        for ax in range(3):
            x[:, ax] = (rng.random(n) if ax < d else rng.uniform(lo, hi, n)) * L[ax]
        f = rng.uniform(-1, 1, (n, 3))
        nu = rng.uniform(-1, 1, (n, 3)) if kind == 1 else None
        p = S.EwaldParams(S.Kernel(kind), d, xi, 0.3, R, grid, S.WindowSpec.make(S.WindowKind.kb, P, grid.h), plan)
        sysm = S.SourceSystem(S.Kernel(kind), S.Cell(L), d, x, f, nu)
        tg = S.TargetSet.from_sources(sysm)
        opt = S.SePipelineOptions(precompute_0p=table)
        u = S.se_fourier_potential(sysm, tg, p, opt)
        rp = ref.params_from(p.to_c())
        ur = ref.fourier_potential(rp, x, f, nu, None, True, precompute_0p=table)
        assert rel_rms(u, ur) < TOL, (d, table)


@pytest.mark.oracle
@pytest.mark.parametrize("d", [0, 1, 2])
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_live_free_axes_selected(S, ref, d, kind):
    rng = np.random.default_rng(1000 + 10 * d + kind)
    N = 120
    L = (1.0, 1.0, 1.0) if d else (2.0, 1.0, 1.0)
    x = rng.random((N, 3)) * np.asarray(L)
    f = rng.standard_normal((N, 3))
    nu = rng.standard_normal((N, 3)) if kind == 1 else None
    sysm = S.SourceSystem(S.Kernel(kind), S.Cell(L), d, x, f, nu)
    window = S.WindowKind.tg if (d == 1 and kind == 2) else S.WindowKind.pkb
    sel = S.select_parameters(sysm.kind, d, sysm.cell, S.source_quantity(sysm), 6.0, S.ToleranceSpec(1e-8),
                              S.SelectionOptions(4, window, True))
    rp = ref.params_from(sel.params.to_c())
    xt = rng.random((50, 3)) * np.asarray(L)
    for same in (True, False):
        tg = S.TargetSet.from_sources(sysm) if same else S.TargetSet(xt, False)
        u = S.full_potential(sysm, tg, sel.params)
        ur = ref.full_potential(rp, x, f, nu, None if same else xt, same)
        assert rel_rms(u, ur) < TOL, (d, kind, same)


# ---------------------------------------------------------------------------
# device session: multi-part evaluation (the multi-GPU decomposition run on
# one GPU as sequential parts) must sum to the single-part result
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("kind,d,same", [(0, 3, True), (1, 2, True), (2, 1, False), (0, 0, True)])
def test_session_parts_sum_to_whole(S, kind, d, same):
    import torch
    from paper_2210_01255_b200.parallel import slice_bounds
    rng = np.random.default_rng(300 + kind + d)
    N = 2500
    L = (1.0, 1.0, 1.0) if d else (2.0, 1.0, 1.0)
    x = rng.random((N, 3)) * np.asarray(L)
    f = rng.standard_normal((N, 3))
    nu = rng.standard_normal((N, 3)) if kind == 1 else None
    xt = None if same else rng.random((1700, 3)) * np.asarray(L)
    sysm = S.SourceSystem(S.Kernel(kind), S.Cell(L), d, x, f, nu)
    sel = S.select_parameters(sysm.kind, d, sysm.cell, S.source_quantity(sysm), 9.0, S.ToleranceSpec(1e-8))
    tg = S.TargetSet.from_sources(sysm) if same else S.TargetSet(xt, False)
    u_ref = S.full_potential(sysm, tg, sel.params)
    dev = torch.device("cuda", 0)
    T = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    sess = S.Session(sel.params, sysm.cell)
    sess.set_sources(T(x), T(f), T(nu))
    sess.set_targets(T(xt), same)
    nt = N if same else xt.shape[0]
    for world in (1, 2, 3):
        grid = torch.zeros(sess.grid_size(), dtype=torch.float64, device=dev)
        total = torch.zeros((nt, 3), dtype=torch.float64, device=dev)
        grids = []
        for r in range(world):  # per-rank source slices, summed like the all-reduce
            g = torch.zeros_like(grid)
            i0, i1 = slice_bounds(N, r, world)
            sess.spread(i0, i1, g)
            grids.append(g)
        grid = sum(grids)
        sess.solve(grid)
        for r in range(world):
            u = torch.zeros((nt, 3), dtype=torch.float64, device=dev)
            sess.evaluate(u, r, world, 7)
            total += u
        torch.cuda.synchronize()
        assert rel_rms(total.cpu().numpy(), u_ref) < TOL, world
    sess.close()


def test_cpp_dropin_binary():
    """C++ user code against the reference header names (tests/cpp/test_dropin.cpp)."""
    import os
    import subprocess
    from conftest import ROOT
    exe = os.path.join(ROOT, "paper_2210_01255_b200", "lib", "test_dropin")
    assert os.path.exists(exe), "build() did not produce the drop-in test binary"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dropin: OK" in r.stdout


# ---------------------------------------------------------------------------
# BASELINE config 2 at full size (N = 1e6): size-independent properties
# ---------------------------------------------------------------------------

def test_full_size_c2_xi_invariance(S):
    """The full velocity does not depend on the split parameter beyond the
    tolerance (test_realspace.cpp:516-540 at the BASELINE size): xi = 37
    (pinned, M = 128) vs xi = 45."""
    from paper_2210_01255_b200.workloads import CONFIGS, generate
    cfg = CONFIGS[2]
    x, f, nu, xt = generate(cfg)
    sysm = S.SourceSystem(cfg.kind, S.Cell(cfg.L), cfg.d, x, f, nu)
    tg = S.TargetSet.from_sources(sysm)
    Q = S.source_quantity(sysm)
    pa = S.select_parameters(cfg.kind, cfg.d, sysm.cell, Q, 37.0, S.ToleranceSpec(cfg.tol)).params
    pb = S.select_parameters(cfg.kind, cfg.d, sysm.cell, Q, 45.0, S.ToleranceSpec(cfg.tol)).params
    ua = S.full_potential(sysm, tg, pa)
    ub = S.full_potential(sysm, tg, pb)
    rms = float(np.sqrt(np.mean(np.sum((ua - ub) ** 2, 1))))
    rms_u = float(np.sqrt(np.mean(np.sum(ua ** 2, 1))))
    print(f"c2 full size: rms(u)={rms_u:.6g} rms(u37-u45)={rms:.3e} (tau={cfg.tol})")
    assert rms <= 10.0 * (cfg.tol + cfg.tol)


@pytest.mark.parametrize("kind,d,N", [(0, 3, 300), (1, 3, 257), (2, 1, 2000), (0, 0, 50000)])
def test_small_systems_deterministic(S, kind, d, N):
    """Small systems (row-split non-symmetric real space, fixed-order sums):
    repeated real-space evaluations are bit-identical, as the reference's
    thread-count test requires (test_realspace.cpp:449-456). The full velocity
    also carries the spread, whose tensor-core tiles add into the grid with
    fp64 atomics (order-dependent last bits, accepted by the north_star)."""
    rng = np.random.default_rng(77 + kind + d)
    L = (1.0, 1.0, 1.0)
    x = rng.random((N, 3))
    f = rng.standard_normal((N, 3))
    nu = rng.standard_normal((N, 3)) if kind == 1 else None
    sysm = S.SourceSystem(S.Kernel(kind), S.Cell(L), d, x, f, nu)
    tg = S.TargetSet.from_sources(sysm)
    p = S.select_parameters(sysm.kind, d, sysm.cell, S.source_quantity(sysm), 10.0, S.ToleranceSpec(1e-8)).params
    ua = S.realspace_potential(sysm, tg, p.xi, p.rc, True)
    ub = S.realspace_potential(sysm, tg, p.xi, p.rc, True)
    assert np.array_equal(ua, ub)
    fa = S.full_potential(sysm, tg, p)
    fb = S.full_potential(sysm, tg, p)
    assert rel_rms(fa, fb) < 1e-14


@pytest.mark.parametrize("cfg_id,xi_b", [(3, 40.0), (4, 40.0), (5, 60.0)])
def test_full_size_xi_invariance(S, cfg_id, xi_b):
    """BASELINE configs 3-5 at full size (D = 2 stresslet 1e6, D = 1 rotlet 5e5 + 5e5
    separate targets with the TG window, D = 0 stokeslet 4e6): the full velocity
    at the pinned xi and at xi_b agree to the tolerance (test_realspace.cpp:516-540)."""
    from paper_2210_01255_b200.workloads import CONFIGS, generate
    cfg = CONFIGS[cfg_id]
    x, f, nu, xt = generate(cfg)
    sysm = S.SourceSystem(cfg.kind, S.Cell(cfg.L), cfg.d, x, f, nu)
    tg = S.TargetSet.from_sources(sysm) if xt is None else S.TargetSet(xt, False)
    Q = S.source_quantity(sysm)
    opt = S.SelectionOptions(4, cfg.window, True)
    pa = S.select_parameters(cfg.kind, cfg.d, sysm.cell, Q, cfg.xi, S.ToleranceSpec(cfg.tol), opt).params
    pb = S.select_parameters(cfg.kind, cfg.d, sysm.cell, Q, xi_b, S.ToleranceSpec(cfg.tol), opt).params
    ua = S.full_potential(sysm, tg, pa)
    ub = S.full_potential(sysm, tg, pb)
    rms = float(np.sqrt(np.mean(np.sum((ua - ub) ** 2, 1))))
    rms_u = float(np.sqrt(np.mean(np.sum(ua ** 2, 1))))
    print(f"{cfg.name}: rms(u)={rms_u:.6g} rms(u_a-u_b)={rms:.3e} (tau={cfg.tol})")
    assert rms <= 10.0 * (cfg.tol + cfg.tol)


@pytest.mark.oracle
def test_full_size_c2_realspace_subset(S, ref):
    """Real-space sum at N = 1e6 for a subset of targets against the reference
    (all sources; targets nudged off the source points, unstarred sum)."""
    from paper_2210_01255_b200.workloads import CONFIGS, generate
    cfg = CONFIGS[2]
    x, f, nu, _ = generate(cfg)
    rng = np.random.default_rng(5)
    xt = x[rng.choice(x.shape[0], 400, replace=False)] + 3.3e-7
    sysm = S.SourceSystem(cfg.kind, S.Cell(cfg.L), cfg.d, x, f, nu)
    p = S.select_parameters(cfg.kind, cfg.d, sysm.cell, S.source_quantity(sysm), cfg.xi, S.ToleranceSpec(cfg.tol)).params
    u = S.realspace_potential(sysm, S.TargetSet(xt, False), p.xi, p.rc, False)
    ur = ref.realspace_potential(0, 3, cfg.L, x, f, None, xt, False, p.xi, p.rc, False, 16)
    assert rel_rms(u, ur) < TOL


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("d,kind,table", [(0, 0, True), (0, 1, True), (0, 2, False),
                                          (3, 0, False), (3, 1, False), (3, 2, False)])
def test_slab_solve_emulated(S, world, d, kind, table):
    """Slab-distributed D = 0 and D = 3 solves (x-slabs -> all-to-all ->
    kz-slabs -> all-to-all back -> all-gather), ranks run in sequence in one
    process with the exchanges done by slicing: the Fourier velocity equals the
    single-GPU solve (D = 3 there: the D2Z / Z2D path of kspace.cu)."""
    import torch
    from paper_2210_01255_b200.parallel import (D0Slabs, d0_stage_forward, d0_stage_inverse, d0_stage_middle,
                                                emulate_all_to_all)
    rng = np.random.default_rng(900 + kind + 10 * world + d)
    N = 3000
    L = (2.0, 1.0, 1.0) if d == 0 else (1.0, 1.0, 1.0)
    x = rng.random((N, 3)) * np.asarray(L)
    f = rng.standard_normal((N, 3))
    nu = rng.standard_normal((N, 3)) if kind == 1 else None
    sysm = S.SourceSystem(S.Kernel(kind), S.Cell(L), d, x, f, nu)
    sel = S.select_parameters(sysm.kind, d, sysm.cell, S.source_quantity(sysm), 9.0, S.ToleranceSpec(1e-8))
    dev = torch.device("cuda", 0)
    T = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    sess = S.Session(sel.params, sysm.cell)
    sess.set_sources(T(x), T(f), T(nu))
    sess.set_targets(None, True)
    grid = torch.zeros(sess.grid_size(), dtype=torch.float64, device=dev)
    sess.spread(0, N, grid)
    sess.solve(grid, table)
    u_ref = torch.zeros((N, 3), dtype=torch.float64, device=dev)
    sess.evaluate(u_ref, 0, 1, 1)
    sl = D0Slabs(sess.d0_geometry(table), world)
    g = grid.view(sl.C, sl.m[0], sl.m[1], sl.m[2])
    sends = [d0_stage_forward(sess, sl, r, g[:, sl.xb[r]:sl.xb[r + 1]].contiguous(), table) for r in range(world)]
    recvs = emulate_all_to_all(sends, [sl.fwd_send_splits(r) for r in range(world)],
                               [sl.fwd_recv_splits(r) for r in range(world)])
    sends2 = [d0_stage_middle(sess, sl, r, recvs[r], table) for r in range(world)]
    recvs2 = emulate_all_to_all(sends2, [sl.inv_send_splits(r) for r in range(world)],
                                [sl.inv_recv_splits(r) for r in range(world)])
    flow = torch.cat([d0_stage_inverse(sess, sl, r, recvs2[r], table) for r in range(world)], dim=1).contiguous()
    sess.set_flow(flow)
    u = torch.zeros((N, 3), dtype=torch.float64, device=dev)
    sess.evaluate(u, 0, 1, 1)
    torch.cuda.synchronize()
    assert rel_rms(u.cpu().numpy(), u_ref.cpu().numpy()) < 1e-13
    sess.close()


@pytest.mark.oracle
@pytest.mark.parametrize("P", [8, 12, 14, 16, 18, 20, 24, 28, 32])
@pytest.mark.parametrize("d,kind,window", [(3, 0, 1), (1, 1, 2), (2, 2, 1)])
def test_live_spread_gather_widths(S, ref, P, d, kind, window):
    """Spread and gather stages across window widths: every kernel family
    (z-sweep, tensor-core tiles with L = 19 / 23 / 31-39, CUDA-core tiles) and
    periodic / free axes, against the reference's spread / gather."""
    rng = np.random.default_rng(4000 + P + 10 * d)
    L = (1.0, 1.0, 1.0)
    N = 700
    x = np.empty((N, 3))
    for ax in range(3):
        x[:, ax] = rng.random(N) if ax < d else rng.uniform(0.05, 0.95, N)
    f = rng.standard_normal((N, 3))
    nu = rng.standard_normal((N, 3)) if kind == 1 else None
    cell = S.Cell(L)
    grid = S.build_grid(cell, d, 1.0 / 40, P, S.Kernel(kind), 4)
    params = S.EwaldParams(S.Kernel(kind), d, 8.0, 0.2, 0.5, grid, S.WindowSpec.make(S.WindowKind(window), P, grid.h))
    sysm = S.SourceSystem(S.Kernel(kind), cell, d, x, f, nu)
    rp = ref.params_from(params.to_c())
    g_gpu = S.spread(sysm, params)
    g_ref = ref.spread(rp, x, f, nu)
    assert np.max(np.abs(g_gpu - g_ref)) <= 1e-13 * np.max(np.abs(g_ref)), P
    field = rng.standard_normal((3,) + tuple(grid.M_ext))
    xt = np.empty((500, 3))
    for ax in range(3):
        xt[:, ax] = rng.random(500) if ax < d else rng.uniform(0.05, 0.95, 500)
    u_gpu = S.gather(field, params, S.TargetSet(xt, False))
    u_ref = ref.gather(rp, field, xt)
    assert np.max(np.abs(u_gpu - u_ref)) <= 1e-13 * np.max(np.abs(u_ref)), P


@pytest.mark.oracle
@pytest.mark.parametrize("P,d", [(8, 3), (12, 3), (14, 0), (12, 2)])
def test_live_gather_dense_targets(S, ref, P, d):
    """Dense targets (>= 12 per tile): the L = 15 tensor-core gather tiles."""
    rng = np.random.default_rng(4100 + P + d)
    cell = S.Cell((1.0, 1.0, 1.0))
    grid = S.build_grid(cell, d, 1.0 / 24, P, S.Kernel.stokeslet, 4)
    params = S.EwaldParams(S.Kernel.stokeslet, d, 8.0, 0.2, 0.5, grid, S.WindowSpec.make(S.WindowKind.pkb, P, grid.h))
    cells = int(np.prod(grid.M_ext))
    B = 16 - P
    nt = int(16 * cells / B ** 3) + 1000
    xt = np.empty((nt, 3))
    for ax in range(3):
        xt[:, ax] = rng.random(nt) if ax < d else rng.uniform(0.1, 0.9, nt)
    field = rng.standard_normal((3,) + tuple(grid.M_ext))
    # the session's gather (Fourier part only, parts = 1) on an installed flow field
    import torch
    dev = torch.device("cuda", 0)
    T = lambda v: torch.from_numpy(np.ascontiguousarray(v)).to(dev)
    sess = S.Session(params, cell)
    sess.set_sources(T(xt[:100]), T(np.zeros((100, 3))))
    sess.set_targets(T(xt), False)
    sess.set_flow(T(field.ravel()))
    u = torch.zeros((nt, 3), dtype=torch.float64, device=dev)
    sess.evaluate(u, 0, 1, 1)
    torch.cuda.synchronize()
    u_gpu = u.cpu().numpy()
    sess.close()
    u_ref = ref.gather(ref.params_from(params.to_c()), field, xt)
    assert np.max(np.abs(u_gpu - u_ref)) <= 1e-13 * np.max(np.abs(u_ref)), (P, d, nt)


@pytest.mark.oracle
@pytest.mark.parametrize("P", [16, 18, 24])
def test_live_clustered_sources(S, ref, P):
    """Thousands of points inside a few grid cells: one tile holds many
    source / target groups (tensor-core spread and gather passes, dense cell
    rows in the real-space sum)."""
    rng = np.random.default_rng(777 + P)
    N = 3000
    x = 0.4 + 0.03 * rng.random((N, 3))
    f = rng.standard_normal((N, 3))
    cell = S.Cell((1.0, 1.0, 1.0))
    grid = S.build_grid(cell, 3, 1.0 / 48, P, S.Kernel.stokeslet, 4)
    params = S.EwaldParams(S.Kernel.stokeslet, 3, 10.0, 0.3, 0.5, grid,
                           S.WindowSpec.make(S.WindowKind.pkb, P, grid.h))
    sysm = S.SourceSystem(S.Kernel.stokeslet, cell, 3, x, f)
    rp = ref.params_from(params.to_c())
    g_gpu = S.spread(sysm, params)
    g_ref = ref.spread(rp, x, f, None)
    assert np.max(np.abs(g_gpu - g_ref)) <= 1e-13 * np.max(np.abs(g_ref))
    field = rng.standard_normal((3,) + tuple(grid.M_ext))
    u_gpu = S.gather(field, params, S.TargetSet(x, False))
    u_ref = ref.gather(rp, field, x)
    assert np.max(np.abs(u_gpu - u_ref)) <= 1e-13 * np.max(np.abs(u_ref))
    u = S.full_potential(sysm, S.TargetSet.from_sources(sysm), params)
    ur = ref.full_potential(rp, x, f, None, None, True)
    assert rel_rms(u, ur) < TOL


@pytest.mark.oracle
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_live_noncubic_d3(S, ref, kind):
    """Triply periodic, non-cubic box (grid, tiles and cell rows differ per axis)."""
    rng = np.random.default_rng(610 + kind)
    L = (1.0, 2.0, 0.5)  # M = (40, 80, 20): a tile region (L = 23) wraps the z axis
    N = 1500
    x = rng.random((N, 3)) * np.asarray(L)
    f = rng.standard_normal((N, 3))
    nu = rng.standard_normal((N, 3)) if kind == 1 else None
    sysm = S.SourceSystem(S.Kernel(kind), S.Cell(L), 3, x, f, nu)
    sel = S.select_parameters(sysm.kind, 3, sysm.cell, S.source_quantity(sysm), 11.0, S.ToleranceSpec(1e-9))
    rp = ref.params_from(sel.params.to_c())
    u = S.full_potential(sysm, S.TargetSet.from_sources(sysm), sel.params)
    ur = ref.full_potential(rp, x, f, nu, None, True)
    assert rel_rms(u, ur) < TOL
