"""Regression: the host-buffer entry points keep a cached session whose cuFFT
plans were created on the context's stream at the time. A device Session
switches the context to torch's current stream; every later cuFFT execution
must follow (plans are re-bound to the context's stream before each exec),
otherwise the transforms race the engine's kernels on the other stream."""
import numpy as np
import pytest

from conftest import load_golden, rel_rms

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["stokeslet_d0", "stresslet_d2", "c1_stokeslet_d3"])
def test_cached_session_after_stream_change(S, name):
    import torch
    import test_gpu_parity as T
    g = load_golden(name)
    sysm = T.system_from(S, g)
    tg = T.targets_from(S, g, sysm)
    params = T.params_from_bytes(S, g["params"])
    assert rel_rms(S.full_potential(sysm, tg, params), g["u"]) < 1e-12
    # a device session on torch's stream (different parameters)
    rng = np.random.default_rng(5)
    x = rng.random((500, 3))
    f = rng.standard_normal((500, 3))
    other = S.SourceSystem(S.Kernel.stokeslet, S.Cell((1.0, 1.0, 1.0)), 3, x, f, None)
    sel = S.select_parameters(other.kind, 3, other.cell, S.source_quantity(other), 9.0, S.ToleranceSpec(1e-8))
    sess = S.Session(sel.params, other.cell)
    dev = torch.device("cuda", 0)
    sess.set_sources(torch.from_numpy(x).to(dev), torch.from_numpy(f).to(dev), None)
    sess.set_targets(None, True)
    grid = torch.zeros(sess.grid_size(), dtype=torch.float64, device=dev)
    sess.spread(0, 500, grid)
    sess.solve(grid, True)
    torch.cuda.synchronize()
    sess.close()
    assert rel_rms(S.full_potential(sysm, tg, params), g["u"]) < 1e-12
    assert rel_rms(S.se_fourier_potential(sysm, tg, params), g["uF"]) < 1e-12
