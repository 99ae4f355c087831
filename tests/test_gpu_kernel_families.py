"""GPU parity of every kernel family, each forced through the kernel-choice
switches (include/sewald_gpu.h SEWALD_OPT_*), against the reference.

The engine picks kernels by size: the pair-symmetric real-space kernel
(csrc/realspace_sym.cu) only for >= 75,776 targets, the tensor-core
spread/gather tiles by window width and target density. Small oracle cases
would otherwise only reach the small-system kernels, so each test here forces
one family and compares it with the reference's own stage:
  real space  realspace.cpp:30-93 / :166-203 (starred sum), bar 1e-13
              max-relative (the reference's own bar is 1e-14 against
              all-pairs, test_realspace.cpp:319-352; fp64 reaction atomics
              change the summation order);
  spread      fourier.cpp:237-274, bar 1e-13 of max |grid|;
  gather      fourier.cpp:276-309, bar 1e-13 of max |u|.
"""
import numpy as np
import pytest

from conftest import load_golden, rel_rms

pytestmark = pytest.mark.gpu


def _params(S, raw):
    return S.EwaldParams.from_c(S.api.sewald_params_c.from_buffer_copy(bytes(raw)))


def _maxrel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-300))


# ---------------------------------------------------------------------------
# pair-symmetric real space (RS_SYM = 2 forces it at any size)
# ---------------------------------------------------------------------------

GOLDEN_SAME = ["c1_stokeslet_d3", "stresslet_d3", "rotlet_d3", "stresslet_d2", "stokeslet_d2",
               "stokeslet_d1", "stokeslet_d0"]


@pytest.mark.parametrize("name", GOLDEN_SAME)
def test_sym_realspace_golden(S, name):
    """Forced pair-symmetric kernel vs the reference's starred real-space sum
    stored in the golden fixtures (all three kernels, D = 3/2/1/0)."""
    g = load_golden(name)
    assert "xt" not in g
    sysm = S.SourceSystem(S.Kernel(int(g["kind"])), S.Cell(tuple(g["L"])), int(g["d"]), g["x"], g["f"], g.get("nu"))
    tg = S.TargetSet.from_sources(sysm)
    p = _params(S, g["params"])
    with S.kernel_options(RS_SYM=2):
        u = S.realspace_potential(sysm, tg, p.xi, p.rc, True)
        uf = S.full_potential(sysm, tg, p)
    assert _maxrel(u, g["uR"]) <= 1e-13
    assert rel_rms(uf, g["u"]) < 1e-12


def _points(rng, n, d, L, lo=0.0, hi=1.0):
    x = np.empty((n, 3))
    for ax in range(3):
        x[:, ax] = (rng.random(n) if ax < d else rng.uniform(lo, hi, n)) * L[ax]
    return x


SYM_CASES = [
    # (kind, d, L, N, xi, rc)
    (0, 3, (1.0, 1.0, 1.0), 3000, 10.0, 0.25),
    (1, 3, (1.0, 1.0, 1.0), 3000, 10.0, 0.25),
    (2, 3, (1.0, 1.0, 1.0), 3000, 10.0, 0.25),
    (0, 3, (1.0, 1.0, 1.0), 200, 3.0, 0.9),    # rc > L/2: several images of one pair
    (1, 3, (0.6, 1.0, 0.8), 150, 3.0, 1.4),    # rc > L on every axis, non-cubic
    (2, 3, (1.0, 1.0, 1.0), 40, 3.0, 2e-3),    # bucket capping (test_realspace.cpp:469-540 shape)
    (0, 2, (1.0, 1.3, 0.8), 2500, 8.0, 0.3),
    (1, 2, (1.0, 1.0, 1.0), 2000, 6.0, 0.55),  # rc > L/2 on the periodic axes
    (2, 2, (1.0, 1.0, 1.0), 2500, 8.0, 0.3),
    (0, 1, (1.0, 0.7, 0.7), 2000, 8.0, 0.3),
    (1, 1, (0.5, 1.0, 1.0), 1500, 6.0, 0.4),   # periodic axis shorter than 2 rc
    (2, 1, (1.0, 1.0, 1.0), 2500, 8.0, 0.3),
    (0, 0, (2.0, 1.0, 1.0), 3000, 8.0, 0.3),
    (1, 0, (1.0, 1.0, 1.0), 2500, 8.0, 0.3),
    (2, 0, (1.0, 1.0, 1.0), 2500, 8.0, 0.3),
]


@pytest.mark.oracle
@pytest.mark.parametrize("case", SYM_CASES)
def test_sym_realspace_live(S, ref, case):
    """Forced pair-symmetric kernel vs the live reference, covering its half
    rule (each unordered pair once, b > a or a positive image shift), image
    shifts with rc above half the period, free axes and capped buckets."""
    kind, d, L, n, xi, rc = case
    rng = np.random.default_rng(8100 + 7 * kind + 3 * d + n)
    x = _points(rng, n, d, L, -0.3, 1.3)
    f = rng.standard_normal((n, 3))
    nu = rng.standard_normal((n, 3)) if kind == 1 else None
    sysm = S.SourceSystem(S.Kernel(kind), S.Cell(L), d, x, f, nu)
    tg = S.TargetSet.from_sources(sysm)
    with S.kernel_options(RS_SYM=2):
        u = S.realspace_potential(sysm, tg, xi, rc, True)
    ur = ref.realspace_potential(kind, d, L, x, f, nu, None, True, xi, rc, True, 8)
    assert _maxrel(u, ur) <= 1e-13, case


@pytest.mark.oracle
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_sym_realspace_clustered(S, ref, kind):
    """Clustered sources (dense cells, long row pieces, many j-blocks per row)."""
    rng = np.random.default_rng(8200 + kind)
    centers = rng.random((6, 3))
    x = (centers[rng.integers(0, 6, 4000)] + 0.03 * rng.standard_normal((4000, 3))) % 1.0
    f = rng.standard_normal((4000, 3))
    nu = rng.standard_normal((4000, 3)) if kind == 1 else None
    sysm = S.SourceSystem(S.Kernel(kind), S.Cell((1, 1, 1)), 3, x, f, nu)
    with S.kernel_options(RS_SYM=2):
        u = S.realspace_potential(sysm, S.TargetSet.from_sources(sysm), 12.0, 0.2, True)
    ur = ref.realspace_potential(kind, 3, (1, 1, 1), x, f, nu, None, True, 12.0, 0.2, True, 8)
    assert _maxrel(u, ur) <= 1e-13


def test_sym_matches_nonsym(S):
    """The two real-space kernels agree with each other (and the forced
    symmetric kernel with the small-system kernel) at 1e-13."""
    rng = np.random.default_rng(8300)
    x = rng.random((6000, 3))
    f = rng.standard_normal((6000, 3))
    sysm = S.SourceSystem(S.Kernel.stokeslet, S.Cell((1, 1, 1)), 3, x, f)
    tg = S.TargetSet.from_sources(sysm)
    with S.kernel_options(RS_SYM=0):
        a = S.realspace_potential(sysm, tg, 14.0, 0.18, True)
    with S.kernel_options(RS_SYM=2):
        b = S.realspace_potential(sysm, tg, 14.0, 0.18, True)
    assert _maxrel(b, a) <= 1e-13


def test_partition_kernel_choice_consistent(S):
    """with nparts > 1 and a cluster count just above
    nparts x resident warps, every part must run the same real-space kernel;
    the parts' sum equals the single-part result. 4735 clusters of 32 split in
    two parts of 2367 / 2368 clusters straddle the 2368-warp threshold."""
    import torch
    from paper_2210_01255_b200.parallel import slice_bounds  # noqa: F401
    N = 4735 * 32
    rng = np.random.default_rng(8400)
    x = rng.random((N, 3))
    f = rng.standard_normal((N, 3))
    sysm = S.SourceSystem(S.Kernel.stokeslet, S.Cell((1, 1, 1)), 3, x, f)
    p = S.select_parameters(sysm.kind, 3, sysm.cell, S.source_quantity(sysm), 20.0, S.ToleranceSpec(1e-8)).params
    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    sess = S.Session(p, sysm.cell)
    sess.set_sources(T(x), T(f))
    sess.set_targets(None, True)
    one = torch.zeros((N, 3), dtype=torch.float64, device=dev)
    sess.evaluate(one, 0, 1, 2)
    for world in (2, 3, 4):
        tot = torch.zeros_like(one)
        for r in range(world):
            u = torch.zeros_like(one)
            sess.evaluate(u, r, world, 2)
            tot += u
        torch.cuda.synchronize()
        assert _maxrel(tot.cpu().numpy(), one.cpu().numpy()) <= 1e-13, world
    sess.close()


# ---------------------------------------------------------------------------
# spread / gather families
# ---------------------------------------------------------------------------

SPREAD_FAMILIES = {
    "mma": dict(SPREAD_MMA=1, SPREAD_SWEEP=-1),
    "mma_taps_kernel": dict(SPREAD_MMA=1, SPREAD_SWEEP=-1, SPREAD_FUSED=0),
    "mma_unsorted": dict(SPREAD_MMA=1, SPREAD_SWEEP=-1, SPREAD_SORT=0),
    "mma_taps_unsorted": dict(SPREAD_MMA=1, SPREAD_SWEEP=-1, SPREAD_FUSED=0, SPREAD_SORT=0),
    "mma_rowsweep": dict(SPREAD_MMA=1, SPREAD_SWEEP=-1, SPREAD_ROWSWEEP=1),
    "mma_rowsweep_unsorted": dict(SPREAD_MMA=1, SPREAD_SWEEP=-1, SPREAD_ROWSWEEP=1, SPREAD_SORT=0),
    "mma_L19": dict(SPREAD_MMA=1, SPREAD_MMA_L=19, SPREAD_SWEEP=-1),
    "mma_pergroup": dict(SPREAD_MMA=1, SPREAD_CACHED=0, SPREAD_SWEEP=-1),
    "sweep": dict(SPREAD_MMA=0, SPREAD_SWEEP=1),
    "tile": dict(SPREAD_MMA=0, SPREAD_SWEEP=0),
}

GATHER_FAMILIES = {
    "warp": dict(GATHER=0),
    "sweep": dict(GATHER=1),
    "tile_mma": dict(GATHER=2, GATHER_MMA=1),
    "tile_mma_L15": dict(GATHER=2, GATHER_MMA=1, GATHER_L=15),
    "tile_cuda": dict(GATHER=2, GATHER_MMA=0),
    "tile_smem_region": dict(GATHER=2, GATHER_WIDE=0),
    "tile_fused_taps": dict(GATHER=2, GATHER_FUSED=1),
    "tile_regA_wide_only": dict(GATHER=2, GATHER_WIDE=1),
    "tile_regA_unsorted": dict(GATHER=2, GATHER_SORT=0),
    "tile_fused_unsorted": dict(GATHER=2, GATHER_FUSED=1, GATHER_SORT=0),
    "sweep_wide_off": dict(GATHER=-1, GATHER_WIDE=0),
}


def _stage_case(S, rng, P, d, kind, window, M=40):
    cell = S.Cell((1.0, 1.0, 1.0))
    grid = S.build_grid(cell, d, 1.0 / M, P, S.Kernel(kind), 4)
    params = S.EwaldParams(S.Kernel(kind), d, 8.0, 0.2, 0.5, grid, S.WindowSpec.make(S.WindowKind(window), P, grid.h))
    return cell, grid, params


@pytest.mark.oracle
@pytest.mark.parametrize("family", list(SPREAD_FAMILIES))
@pytest.mark.parametrize("P", [8, 14, 16, 18, 20, 24, 32])
@pytest.mark.parametrize("d,kind,window", [(3, 0, 1), (2, 1, 1), (1, 2, 2)])
def test_spread_family(S, ref, family, P, d, kind, window):
    rng = np.random.default_rng(8500 + P + 10 * d)
    cell, grid, params = _stage_case(S, rng, P, d, kind, window)
    N = 900
    x = _points(rng, N, d, (1, 1, 1), 0.05, 0.95)
    f = rng.standard_normal((N, 3))
    nu = rng.standard_normal((N, 3)) if kind == 1 else None
    sysm = S.SourceSystem(S.Kernel(kind), cell, d, x, f, nu)
    with S.kernel_options(**SPREAD_FAMILIES[family]):
        g_gpu = S.spread(sysm, params)
    g_ref = ref.spread(ref.params_from(params.to_c()), x, f, nu)
    assert np.max(np.abs(g_gpu - g_ref)) <= 1e-13 * np.max(np.abs(g_ref)), (family, P)


@pytest.mark.oracle
@pytest.mark.parametrize("family", list(GATHER_FAMILIES))
@pytest.mark.parametrize("P", [8, 12, 14, 16, 18, 20, 24, 32])
@pytest.mark.parametrize("d", [3, 2, 1, 0])
def test_gather_family(S, ref, family, P, d):
    """sewald_gpu_gather runs the kernel the pipeline would pick (or the
    forced family; families that do not apply to a width fall back to the
    next one, as in the pipeline) against the reference gather."""
    rng = np.random.default_rng(8600 + P + 10 * d)
    cell, grid, params = _stage_case(S, rng, P, d, 0, 1 if P <= 24 else 2)
    nt = 3000
    xt = _points(rng, nt, d, (1, 1, 1), 0.05, 0.95)
    field = rng.standard_normal((3,) + tuple(grid.M_ext))
    with S.kernel_options(**GATHER_FAMILIES[family]):
        u_gpu = S.gather(field, params, S.TargetSet(xt, False))
    u_ref = ref.gather(ref.params_from(params.to_c()), field, xt)
    assert np.max(np.abs(u_gpu - u_ref)) <= 1e-13 * np.max(np.abs(u_ref)), (family, P, d)


@pytest.mark.parametrize("family", list(GATHER_FAMILIES))
def test_gather_family_golden(S, family):
    """Same, against the stored reference gather of the stage fixtures."""
    for name in ["spread_kb_d3", "spread_pkb_d2_stresslet", "spread_tg_d0"]:
        g = load_golden(name)
        params = _params(S, g["params"])
        with S.kernel_options(**GATHER_FAMILIES[family]):
            ug = S.gather(g["field"], params, S.TargetSet(g["xt"], False))
        assert np.max(np.abs(ug - g["ug"])) <= 1e-13 * np.max(np.abs(g["ug"])), (family, name)


@pytest.mark.parametrize("family", list(SPREAD_FAMILIES))
def test_spread_family_golden(S, family):
    for name in ["spread_kb_d3", "spread_pkb_d2_stresslet", "spread_tg_d0"]:
        g = load_golden(name)
        params = _params(S, g["params"])
        sysm = S.SourceSystem(params.kind, S.Cell(tuple(params.grid.L)), params.d, g["x"], g["f"], g.get("nu"))
        with S.kernel_options(**SPREAD_FAMILIES[family]):
            grid = S.spread(sysm, params)
        assert np.max(np.abs(grid - g["grid"])) <= 1e-14 * np.max(np.abs(g["grid"])), (family, name)


def test_partition_pair_balance(S):
    """Multi-part pair-symmetric real space takes interleaved clusters: every
    part gets the same share of the pairs (contiguous ranges gave the first
    part the periodic-wrap pairs of both ends), and the parts' pairs add up to
    the single-part count."""
    import torch
    N = 300_000
    rng = np.random.default_rng(8450)
    x = rng.random((N, 3))
    f = rng.standard_normal((N, 3))
    sysm = S.SourceSystem(S.Kernel.stokeslet, S.Cell((1, 1, 1)), 3, x, f)
    p = S.select_parameters(sysm.kind, 3, sysm.cell, S.source_quantity(sysm), 25.0, S.ToleranceSpec(1e-8)).params
    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    sess = S.Session(p, sysm.cell)
    sess.set_sources(T(x), T(f))
    sess.set_targets(None, True)
    u = torch.zeros((N, 3), dtype=torch.float64, device=dev)
    with S.kernel_options(RS_SYM=2):
        sess.pair_count(reset=True)
        sess.evaluate(u, 0, 1, 2)
        total = sess.pair_count(reset=True)
        counts = []
        for r in range(8):
            sess.evaluate(u, r, 8, 2)
            counts.append(sess.pair_count(reset=True))
    sess.close()
    assert sum(counts) == total
    assert max(counts) / min(counts) < 1.05, counts
