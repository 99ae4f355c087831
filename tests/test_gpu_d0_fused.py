"""D = 0 solve, fused y path (aft_d0.cu d0_yfused_kernel: x transforms over
the data rows only; y transform, scale and inverse y transform in one kernel)
against the batched 2-D transforms + scale kernel, for every kernel and both
the table and the direct modified-kernel paths, on grids whose padded y
length is a power of two (the fused path's domain). Seeded systems with the
BASELINE c5 selection options; xi chosen so that M_ext(1) = 128 (n1 = 256).
The c5 full-size fixture (tests/test_fullsize_parity.py) covers n1 = 512."""
import numpy as np
import pytest

from conftest import rel_rms

pytestmark = pytest.mark.gpu

CASES = [(0, 32.5), (1, 27.5), (2, 35.0)]  # (kernel, xi) with M_ext(1) = 128 for N = 4000 below


def _fourier(S, params, cell, x, f, nu, table, fused):
    import torch
    dev = torch.device("cuda", 0)
    T = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    with S.kernel_options(D0_YFUSED=int(fused)):
        sess = S.Session(params, cell)
        try:
            sess.set_sources(T(x), T(f), T(nu))
            sess.set_targets(None, True)
            grid = torch.zeros(sess.grid_size(), dtype=torch.float64, device=dev)
            sess.spread(0, x.shape[0], grid)
            sess.solve(grid, table)
            u = torch.zeros((x.shape[0], 3), dtype=torch.float64, device=dev)
            sess.evaluate(u, 0, 1, 1)
            torch.cuda.synchronize()
            return u.cpu().numpy()
        finally:
            sess.close()


@pytest.mark.parametrize("table", [True, False])
@pytest.mark.parametrize("kind,xi", CASES)
def test_d0_fused_y_matches_2d(S, kind, xi, table):
    from paper_2210_01255_b200.workloads import CONFIGS
    rng = np.random.default_rng(7)
    L = (2.0, 1.0, 1.0)
    N = 4000
    x = rng.random((N, 3)) * np.asarray(L)
    f = rng.standard_normal((N, 3))
    nu = rng.standard_normal((N, 3)) if kind == 1 else None
    sysm = S.SourceSystem(S.Kernel(kind), S.Cell(L), 0, x, f, nu)
    sel = S.select_parameters(sysm.kind, 0, sysm.cell, S.source_quantity(sysm), xi, S.ToleranceSpec(1e-6),
                              S.SelectionOptions(4, CONFIGS[5].window, True))
    assert sel.params.grid.M_ext[1] == 128  # padded y = 256: the fused path applies
    u1 = _fourier(S, sel.params, sysm.cell, x, f, nu, table, True)
    u0 = _fourier(S, sel.params, sysm.cell, x, f, nu, table, False)
    assert rel_rms(u1, u0) < 1e-13
