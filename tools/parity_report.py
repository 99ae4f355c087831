"""Print the measured parity (rms(u_gpu - u_ref) / rms(u_ref)) of every golden
fixture: the margin under the 1e-12 bar that tests/test_gpu_parity.py checks."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2210_01255_b200 as S  # noqa: E402
from conftest import load_golden, rel_rms  # noqa: E402
from test_gpu_parity import params_from_bytes, system_from, targets_from  # noqa: E402

cases = [("c1_stokeslet_d3", ""), ("c1_stokeslet_d3", "_xi10"), ("stresslet_d3", ""), ("rotlet_d3", ""),
         ("stresslet_d2", ""), ("stokeslet_d2", ""), ("rotlet_d1_tg", ""), ("stokeslet_d1", ""), ("stokeslet_d0", "")]
print(f"{'fixture':24s} {'u_R':>10s} {'u_F':>10s} {'u':>10s}")
for name, tag in cases:
    g = load_golden(name)
    sysm = system_from(S, g)
    tg = targets_from(S, g, sysm)
    p = params_from_bytes(S, g["params" + tag])
    u = S.full_potential(sysm, tg, p)
    uF = S.se_fourier_potential(sysm, tg, p)
    uR = S.realspace_potential(sysm, tg, p.xi, p.rc, tg.same_as_sources)
    print(f"{name + tag:24s} {rel_rms(uR, g['uR' + tag]):10.2e} {rel_rms(uF, g['uF' + tag]):10.2e} "
          f"{rel_rms(u, g['u' + tag]):10.2e}")
