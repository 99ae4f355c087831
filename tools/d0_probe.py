"""Time Session.solve for BASELINE config 5 (D = 0) in isolation."""
import os, sys, time
import numpy as np
import torch
if os.environ.get("TORCH_CUFFT_FIRST"):
    torch.fft.fft(torch.zeros(8, dtype=torch.complex128, device="cuda"))  # load torch's cuFFT first
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_01255_b200 as S
from paper_2210_01255_b200.workloads import CONFIGS, generate

cfg = CONFIGS[int(os.environ.get("CFG", "5"))]
x, f, nu, xt = generate(cfg)
cell = S.Cell(cfg.L)
sysm = S.SourceSystem(cfg.kind, cell, cfg.d, x, f, nu)
sel = S.select_parameters(cfg.kind, cfg.d, cell, S.source_quantity(sysm), cfg.xi, S.ToleranceSpec(cfg.tol),
                          S.SelectionOptions(4, cfg.window, True))
sess = S.Session(sel.params, cell)
T = lambda a: None if a is None else torch.from_numpy(a).cuda()
sess.set_sources(T(x), T(f), T(nu))
sess.set_targets(T(xt), xt is None)
grid = torch.zeros(sess.grid_size(), dtype=torch.float64, device="cuda")
sess.spread(0, x.shape[0], grid)
sess.solve(grid)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    sess.solve(grid)
e1.record()
torch.cuda.synchronize()
import subprocess
maps = open("/proc/self/maps").read()
print("cufft libs:", sorted({l.split()[-1] for l in maps.splitlines() if "cufft" in l}))
print(cfg.name, "solve ms", e0.elapsed_time(e1) / 5, "M_ext", sel.params.grid.M_ext)
