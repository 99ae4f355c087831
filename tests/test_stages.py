"""Reference stage functions: aft_forward, scale (ModifiedKernelSpec
and PrecomputedKernel0P), aft_inverse, precompute_0p through the C-ABI,
against the reference's own stage functions (oracle/_ref) on the same
FourierField, stage by stage, plus the composed solve and the round trip.

Reference: fourier.h:30-74, fourier.cpp:311-803; the hand-built grids are the
ones of the reference's test_fourier.cpp:507-724.
"""
import numpy as np
import pytest

TOL = 1e-13


def _grid(S, d, h, M, Mext):
    L = tuple(h * m for m in M)
    Le = tuple(h * m for m in Mext)
    return S.GridSpec(d, h, M, Mext, L, Le, tuple(a - b for a, b in zip(Le, L)), 4)


def _cases(S):
    """(name, grid, plan, R) — reference test grids plus a periodic box."""
    return [
        ("d3", _grid(S, 3, 1 / 12, (12, 10, 8), (12, 10, 8)), S.UpsamplingPlan(), 1.0),
        ("d2", _grid(S, 2, 1 / 8, (8, 8, 4), (8, 8, 12)), S.UpsamplingPlan(2.0, 1.5, (2, 2, 0)), 1.5),
        ("d1", _grid(S, 1, 1 / 8, (8, 4, 4), (8, 12, 12)), S.UpsamplingPlan(8 / 3, 1.5, (2, 0, 0)),
         1.5 * np.sqrt(2)),
        ("d0", _grid(S, 0, 1 / 16, (8, 8, 8), (16, 16, 16)), S.UpsamplingPlan(3.0), np.sqrt(3.0)),
        ("d0_s2", _grid(S, 0, 1 / 16, (8, 8, 8), (16, 16, 16)), S.UpsamplingPlan(2.0), np.sqrt(3.0)),
    ]


def _close(a, b, tol=TOL):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    scale = np.max(np.abs(b)) if b.size else 0.0
    err = np.max(np.abs(a - b)) if b.size else 0.0
    assert err <= tol * max(scale, 1e-300), (err, scale)


def _to_ref(F):
    return {"d": F.d, "comps": F.comps, "n_per": tuple(F.n_per), "n_far": tuple(F.n_far),
            "n_near": tuple(F.n_near), "n_zero": tuple(F.n_zero), "near_rows": np.asarray(F.near_rows),
            "far": F.far, "near": F.near, "zero": F.zero}


def _from_ref(S, r):
    return S.FourierField(r["d"], r["comps"], r["n_per"], r["n_far"], r["n_near"], r["n_zero"], r["far"],
                          r["near_rows"].astype(np.int32), r["near"], r["zero"])


def _same_field(F, r, tol=TOL):
    assert (F.d, F.comps) == (r["d"], r["comps"])
    for k in ("n_per", "n_far", "n_near", "n_zero"):
        assert tuple(getattr(F, k)) == tuple(r[k]), k
    assert np.array_equal(np.asarray(F.near_rows), r["near_rows"])
    for k in ("far", "near", "zero"):
        _close(getattr(F, k), r[k], tol)


# d = 1 zero-row scale: the truncated 1P kernels need J0, J1 at x = R |k| up
# to ~75. The oracle build links the reference against a GSL shim that maps
# gsl_sf_bessel_J0/J1 to libstdc++ std::cyl_bessel_j (oracle/shims/gsl), whose
# relative error grows to ~1e-13 at such x (vs mpmath; GSL and CUDA j0/j1 stay
# near 1e-16), amplified by the bracket's cancellation to a few 1e-12 on the
# largest modes. The device path is the accurate side of that difference.
def _scale_tol(d):
    return 2e-11 if d == 1 else TOL


def _params(S, kind, grid, plan, R, xi=5.0, P=10, window=None):
    wk = S.WindowKind.kb if window is None else window
    return S.EwaldParams(S.Kernel(kind), grid.d, xi, 0.3, R, grid, S.WindowSpec.make(wk, P, grid.h), plan)


# ---------------------------------------------------------------------------
# host only: FourierField geometry and near rows (classify_rows)
# ---------------------------------------------------------------------------

@pytest.mark.oracle
@pytest.mark.parametrize("comps", [3, 9])
def test_geometry_matches_reference(S, ref, comps):
    import ctypes as C
    lib = S.api._abi.load()
    for name, grid, plan, R in _cases(S):
        p = _params(S, 0, grid, plan, R).to_c()
        g = S.api._abi.sewald_fourier_geom_c()
        rows = np.zeros(64, np.int32)
        assert lib.sewald_aft_geometry(C.byref(p), comps, C.byref(g),
                                       rows.ctypes.data_as(C.POINTER(C.c_int32))) == 0
        field = np.zeros((comps,) + tuple(grid.M_ext))
        r = ref.aft_forward(ref.params_from(p), field)
        assert (g.d, g.comps) == (r["d"], r["comps"])
        for k in ("n_per", "n_far", "n_near", "n_zero"):
            assert tuple(getattr(g, k)) == tuple(r[k]), (name, k)
        assert np.array_equal(rows[:g.n_near_rows], r["near_rows"]), name
        assert (g.far_len, g.near_len, g.zero_len) == (r["far"].size, r["near"].size, r["zero"].size), name


def test_modspec_optimal(S):
    m = S.ModifiedKernelSpec.optimal(S.Kernel.stresslet, 0, 2.0)
    assert (m.a_B, m.b_B, m.ell_H, m.c_B) == (-1.0, -0.25, 2.0, -2.0)
    assert abs(m.ell_B - 2.0 * np.exp(0.5)) < 1e-15


def test_geometry_errors(S):
    import ctypes as C
    grid = _grid(S, 0, 1 / 16, (8, 8, 8), (16, 16, 16))
    lib = S.api._abi.load()
    g = S.api._abi.sewald_fourier_geom_c()
    p = S.api._stage_params(grid, S.UpsamplingPlan(2.03))
    with pytest.raises(S.InvalidArgument, match="integer grid size"):
        S.api._host_call(lib.sewald_aft_geometry(C.byref(p), 3, C.byref(g), None))
    p = S.api._stage_params(grid, S.UpsamplingPlan(2.0))
    with pytest.raises(S.InvalidArgument, match="inconsistent"):
        S.api._host_call(lib.sewald_aft_geometry(C.byref(p), 0, C.byref(g), None))


# ---------------------------------------------------------------------------
# GPU stage parity
# ---------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.oracle
@pytest.mark.parametrize("window", [0, 1, 2])
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_stages_against_reference(S, ref, kind, window):
    """Each stage for every kernel, periodicity class and window (the scale
    divides by the window's transform: exact KB for KB / PKB, Gaussian for TG)."""
    rng = np.random.default_rng(500 + kind + 7 * window)
    comps = S.strength_components(S.Kernel(kind))
    for name, grid, plan, R in _cases(S):
        p = _params(S, kind, grid, plan, R, window=S.WindowKind(window))
        rp = ref.params_from(p.to_c())
        phi = rng.standard_normal((comps,) + tuple(grid.M_ext))
        # aft_forward
        F = S.aft_forward(phi, grid, plan)
        r = ref.aft_forward(rp, phi)
        _same_field(F, r)
        # scale with the optimal modified kernel, fed the reference's own modes
        spec = S.ModifiedKernelSpec.optimal(S.Kernel(kind), grid.d, 1.0 if grid.d == 3 else R)
        Fs = S.scale(_from_ref(S, r), spec, p.xi, p.window, grid)
        rs = ref.scale(rp, r, (kind, grid.d, spec.R, spec.a_B, spec.b_B, spec.ell_H, spec.ell_B, spec.c_B), p.xi)
        _same_field(Fs, rs, _scale_tol(grid.d))
        # aft_inverse of the reference's scaled field
        u = S.aft_inverse(_from_ref(S, rs), grid, plan)
        ur = ref.aft_inverse(rp, rs)
        _close(u, ur)
        # composed on the device only: forward -> scale -> inverse
        u2 = S.aft_inverse(S.scale(F, spec, p.xi, p.window, grid), grid, plan)
        _close(u2, ur, max(1e-12, _scale_tol(grid.d)))


@pytest.mark.gpu
@pytest.mark.oracle
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_nonoptimal_gauge(S, ref, kind):
    """scale with user gauge constants (ModifiedKernelSpec fields, modified_kernels.h:10-19)."""
    rng = np.random.default_rng(520 + kind)
    comps = S.strength_components(S.Kernel(kind))
    for name, grid, plan, R in _cases(S)[1:4]:
        p = _params(S, kind, grid, plan, R)
        rp = ref.params_from(p.to_c())
        phi = rng.standard_normal((comps,) + tuple(grid.M_ext))
        r = ref.aft_forward(rp, phi)
        spec = S.ModifiedKernelSpec(S.Kernel(kind), grid.d, R, -0.3 * R, -0.7 / R, 1.3 * R, 2.1 * R, -0.2 * R * R)
        Fs = S.scale(_from_ref(S, r), spec, p.xi, p.window, grid)
        rs = ref.scale(rp, r, (kind, grid.d, spec.R, spec.a_B, spec.b_B, spec.ell_H, spec.ell_B, spec.c_B), p.xi)
        _same_field(Fs, rs, _scale_tol(grid.d))


@pytest.mark.gpu
@pytest.mark.oracle
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_precompute_0p_and_table_scale(S, ref, kind):
    rng = np.random.default_rng(540 + kind)
    comps = S.strength_components(S.Kernel(kind))
    grid = _grid(S, 0, 1 / 16, (8, 8, 8), (16, 16, 16))
    plan = S.UpsamplingPlan(2.0)
    R = np.sqrt(3.0)
    p = _params(S, kind, grid, plan, R)
    rp = ref.params_from(p.to_c())
    pre = S.precompute_0p(S.Kernel(kind), grid, R)
    assert tuple(pre.n) == (32, 32, 32)
    rtab = ref.precompute_0p(rp)
    _close(pre.table.reshape(rtab.shape), rtab, 1e-12)
    phi = rng.standard_normal((comps,) + tuple(grid.M_ext))
    r = ref.aft_forward(rp, phi)
    Fs = S.scale(_from_ref(S, r), pre, p.xi, p.window, grid)
    rs = ref.scale_table(rp, r, kind, R, p.xi)
    _same_field(Fs, rs, 1e-12)
    # the table-scaled field (default n_per / n_far) inverts like the reference's
    _close(S.aft_inverse(Fs, grid, plan), ref.aft_inverse(rp, rs), 1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("case", [0, 1, 2, 3])
def test_forward_inverse_round_trip(S, case):
    """aft_inverse(aft_forward(phi)) == phi (size-independent property)."""
    name, grid, plan, R = _cases(S)[case]
    rng = np.random.default_rng(560 + case)
    phi = rng.standard_normal((9,) + tuple(grid.M_ext))
    back = S.aft_inverse(S.aft_forward(phi, grid, plan), grid, plan)
    _close(back, phi, 1e-13)


@pytest.mark.gpu
def test_stage_errors(S):
    name, grid, plan, R = _cases(S)[1]
    p = _params(S, 0, grid, plan, R)
    phi = np.zeros((3,) + tuple(grid.M_ext))
    F = S.aft_forward(phi, grid, plan)
    spec = S.ModifiedKernelSpec.optimal(S.Kernel.stokeslet, 2, R)
    with pytest.raises(S.InvalidArgument, match="periodicity"):
        S.scale(F, S.ModifiedKernelSpec.optimal(S.Kernel.stokeslet, 1, R), p.xi, p.window, grid)
    with pytest.raises(S.InvalidArgument, match="component count"):
        S.scale(F, S.ModifiedKernelSpec.optimal(S.Kernel.stresslet, 2, R), p.xi, p.window, grid)
    with pytest.raises(S.InvalidArgument, match="xi must be positive"):
        S.scale(F, spec, 0.0, p.window, grid)
    with pytest.raises(S.InvalidArgument, match="grid spacing"):
        S.scale(F, spec, p.xi, S.WindowSpec.make(S.WindowKind.kb, 10, grid.h * 2), grid)
    with pytest.raises(S.InvalidArgument, match="d = 0 only"):
        S.precompute_0p(S.Kernel.stokeslet, grid, R)
    g0 = _cases(S)[3][1]
    with pytest.raises(S.InvalidArgument, match="truncation radius"):
        S.precompute_0p(S.Kernel.stokeslet, g0, 0.0)
    pre = S.precompute_0p(S.Kernel.stokeslet, g0, np.sqrt(3.0))
    F0 = S.aft_forward(np.zeros((3,) + tuple(g0.M_ext)), g0, S.UpsamplingPlan(3.0))
    with pytest.raises(S.InvalidArgument, match="different padded grid"):
        S.scale(F0, pre, 5.0, S.WindowSpec.make(S.WindowKind.kb, 10, g0.h), g0)
    bad = S.FourierField(**{**F.__dict__, "d": 1})
    with pytest.raises(S.InvalidArgument, match="periodicity differ"):
        S.aft_inverse(bad, grid, plan)


@pytest.mark.gpu
@pytest.mark.oracle
def test_pipeline_uses_caller_table(S, ref):
    """SePipelineOptions::table (fourier.h:76-79, fourier.cpp:822-829): the
    caller's table replaces the engine's own. With the engine's own R the
    result is unchanged; with a table built for another R it follows that
    table, as the reference's stage composition with the same table does."""
    rng = np.random.default_rng(580)
    N = 200
    L = (0.5, 0.5, 0.5)
    x = rng.uniform(0.15, 0.35, (N, 3))
    f = rng.standard_normal((N, 3))
    sysm = S.SourceSystem(S.Kernel.rotlet, S.Cell(L), 0, x, f, None)
    tg = S.TargetSet.from_sources(sysm)
    p = S.select_parameters(S.Kernel.rotlet, 0, sysm.cell, S.source_quantity(sysm), 12.0, S.ToleranceSpec(1e-9)).params
    u0 = S.se_fourier_potential(sysm, tg, p)
    own = S.precompute_0p(S.Kernel.rotlet, p.grid, p.R)
    u1 = S.se_fourier_potential(sysm, tg, p, S.SePipelineOptions(True, own))
    _close(u1, u0, 1e-14)
    R2 = 0.1 * p.R  # shorter than the source spread: truncates real interactions
    other = S.precompute_0p(S.Kernel.rotlet, p.grid, R2)
    u2 = S.se_fourier_potential(sysm, tg, p, S.SePipelineOptions(True, other))
    # reference stages with the same table (fourier.cpp:816-846)
    plan2 = S.UpsamplingPlan(2.0, p.upsampling.s_star, tuple(p.upsampling.k_star))
    rp = ref.params_from(S.EwaldParams(p.kind, 0, p.xi, p.rc, p.R, p.grid, p.window, plan2).to_c())
    phi = ref.spread(rp, x, f, None)
    F = ref.scale_table(rp, ref.aft_forward(rp, phi), 2, R2, p.xi)
    ur = ref.gather(rp, ref.aft_inverse(rp, F), x)
    _close(u2, ur, 1e-12)
    assert np.max(np.abs(u2 - u0)) > 1e-10 * np.max(np.abs(u0))  # the table made a difference
    # back to the engine's own table
    _close(S.se_fourier_potential(sysm, tg, p), u0, 1e-14)


@pytest.mark.gpu
def test_stage_empty_and_zero_inputs(S):
    """Empty source / target sets and all-zero fields through the stage API:
    exact zeros out, shapes as the reference's."""
    for name, grid, plan, R in _cases(S):
        d = grid.d
        p = _params(S, 0, grid, plan, R)
        sysm = S.SourceSystem(S.Kernel.stokeslet, S.Cell(tuple(grid.L)), d, np.zeros((0, 3)), np.zeros((0, 3)))
        phi = S.spread(sysm, p)
        assert phi.shape == (3,) + tuple(grid.M_ext) and not np.any(phi)
        F = S.aft_forward(phi, grid, plan)
        for k in ("far", "near", "zero"):
            assert not np.any(getattr(F, k))
        spec = S.ModifiedKernelSpec.optimal(S.Kernel.stokeslet, d, 1.0 if d == 3 else R)
        Fs = S.scale(F, spec, p.xi, p.window, grid)
        back = S.aft_inverse(Fs, grid, plan)
        assert back.shape == (3,) + tuple(grid.M_ext) and not np.any(back)
        u = S.gather(back, p, S.TargetSet(np.zeros((0, 3)), False))
        assert u.shape == (0, 3)
