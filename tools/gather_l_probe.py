"""Gather-only timing (Fourier part, parts = 1) for dense targets, to compare
tile regions (SEWALD_GATHER_L=15 / 19). D = 3 stokeslet, M = 128, P = 14."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_01255_b200 as S

N = int(os.environ.get("NPTS", "4000000"))
rng = np.random.default_rng(5)
x = rng.random((N, 3))
f = rng.standard_normal((N, 3))
cell = S.Cell((1.0, 1.0, 1.0))
sysm = S.SourceSystem(S.Kernel.stokeslet, cell, 3, x, f, None)
sel = S.select_parameters(S.Kernel.stokeslet, 3, cell, S.source_quantity(sysm), 37.0, S.ToleranceSpec(float(os.environ.get("TOL", "1e-6"))))
p = sel.params
sess = S.Session(p, cell)
T = lambda a: torch.from_numpy(a).cuda()
sess.set_sources(T(x), T(f))
sess.set_targets(None, True)
grid = torch.zeros(sess.grid_size(), dtype=torch.float64, device="cuda")
sess.spread(0, N, grid)
sess.solve(grid)
u = torch.zeros((N, 3), dtype=torch.float64, device="cuda")
sess.evaluate(u, 0, 1, 1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    sess.evaluate(u, 0, 1, 1)
e1.record()
torch.cuda.synchronize()
print(f"L={os.environ.get('SEWALD_GATHER_L', 'auto')} N={N} M={p.grid.M_ext} P={p.window.P} gather ms {e0.elapsed_time(e1) / 5:.3f} u0={u[0].tolist()}")
