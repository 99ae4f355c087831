"""CPU: the independent numpy restatement (oracle/restatement.py) against the
golden fixtures produced by the compiled reference — pins the oracle pair."""
import numpy as np
import pytest

from conftest import load_golden, rel_rms


def _params(g, R):
    import ctypes as C
    raw = bytes(g["params"])
    # struct layout of include/sewald_gpu.h (oracle/sewald_ref.RefParams)
    import sewald_ref
    p = sewald_ref.RefParams.from_buffer_copy(raw)
    return dict(kind=p.kind, d=p.d, xi=p.xi, rc=p.rc, h=p.h, M=list(p.M), P=p.P, beta=p.beta, nu=p.nu,
                L=list(p.L))


@pytest.mark.parametrize("name", ["rotlet_d3", "stresslet_d3"])
def test_restatement_matches_golden(name):
    import restatement as R
    g = load_golden(name)
    p = _params(g, R)
    kind = int(g["kind"])
    nu = g.get("nu")
    # parameter chain restated (D = 3)
    q = R.select_parameters_d3(kind, tuple(g["L"]), float(g["Q"]), p["xi"], float(g["tol"]))
    assert q["M"] == p["M"] and q["P"] == p["P"] and abs(q["rc"] - p["rc"]) <= 1e-14 * p["rc"]
    uR = R.realspace_potential(kind, p["L"], g["x"], g["f"], nu, None, p["xi"], p["rc"], True)
    assert rel_rms(uR, g["uR"]) < 1e-13
    uF = R.fourier_potential(p, g["x"], g["f"], nu)
    assert rel_rms(uF, g["uF"]) < 1e-11
    u = R.full_potential_d3(p, g["x"], g["f"], nu)
    assert rel_rms(u, g["u"]) < 1e-11


def test_restatement_spread_gather_stage():
    import restatement as R
    import sewald_ref
    g = load_golden("spread_kb_d3")
    raw = sewald_ref.RefParams.from_buffer_copy(bytes(g["params"]))
    # the restatement implements the PKB window; compare on a PKB grid built the same way
    p = dict(kind=0, d=3, xi=5.0, rc=0.3, h=raw.h, M=list(raw.M), P=raw.P, beta=2.5 * raw.P,
             nu=min(raw.P // 2 + 2, 10), L=list(raw.L))
    tab = R.pkb_table(p)
    # PKB reproduces KB closely (test_window.cpp:123-155: <1e-7 at P=10)
    r = np.linspace(-0.24, 0.24, 97)
    assert np.max(np.abs(R.pkb_value(p, tab, r) - R.kb_value(p, r))) < 1e-5
    grid = R.spread(p, g["x"], g["f"])
    assert np.isfinite(grid).all() and abs(grid.sum()) > 0
