import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2210_01255_b200 as S
from conftest import load_golden, rel_rms
me = S.MultiEngine([0, 0])
for name in ["c1_stokeslet_d3", "stresslet_d2", "stokeslet_d0", "c1_stokeslet_d3", "rotlet_d1_tg"]:
    g = load_golden(name)
    sysm = S.SourceSystem(S.Kernel(int(g["kind"])), S.Cell(tuple(g["L"])), int(g["d"]), g["x"], g["f"], g.get("nu"))
    tg = S.TargetSet(g["xt"], False) if "xt" in g else S.TargetSet.from_sources(sysm)
    p = S.EwaldParams.from_c(S.api.sewald_params_c.from_buffer_copy(bytes(g["params"])))
    u = me.full_potential(sysm, tg, p)
    one = S.full_potential(sysm, tg, p)
    print(name, rel_rms(u, one), rel_rms(u, g["u"]))
