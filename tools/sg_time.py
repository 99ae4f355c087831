"""Time the spread and the gather (Session.spread / Session.evaluate(parts=1))
of a BASELINE config under kernel-choice options, and check each variant's
grid / velocity against the default kernels of the same session.

    python tools/sg_time.py [config] [reps] [OPT=VAL,OPT=VAL ...]...
e.g. python tools/sg_time.py 2 5 "" SPREAD_ROWSWEEP=1
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2210_01255_b200 as S  # noqa: E402
from paper_2210_01255_b200.workloads import CONFIGS, generate  # noqa: E402

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
variants = sys.argv[3:] or [""]
if os.environ.get("SG_XI"):  # another split parameter (bench.py --xi)
    import dataclasses
    cfg = dataclasses.replace(cfg, xi=float(os.environ["SG_XI"]))
x, f, nu, xt = generate(cfg)
sysm = S.SourceSystem(cfg.kind, S.Cell(cfg.L), cfg.d, x, f, nu)
p = S.select_parameters(cfg.kind, cfg.d, sysm.cell, S.source_quantity(sysm), cfg.xi, S.ToleranceSpec(cfg.tol),
                        S.SelectionOptions(4, cfg.window, True)).params
dev = torch.device("cuda", 0)
T = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
sess = S.Session(p, sysm.cell)
sess.set_sources(T(x), T(f), T(nu))
sess.set_targets(T(xt), xt is None)
nt = x.shape[0] if xt is None else xt.shape[0]
grid = torch.zeros(sess.grid_size(), dtype=torch.float64, device=dev)
u = torch.zeros((nt, 3), dtype=torch.float64, device=dev)


def timed(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


ref_grid = ref_u = None
for v in variants:
    opts = dict(kv.split("=") for kv in v.split(",") if kv)
    opts = {k: int(val) for k, val in opts.items()}
    with S.kernel_options(**opts):
        t_sp = timed(lambda: sess.spread(0, x.shape[0], grid))
        g = grid.cpu().numpy()
        sess.solve(grid, True)
        t_ga = timed(lambda: sess.evaluate(u, 0, 1, 1))
        uu = u.cpu().numpy()
    if ref_grid is None:
        ref_grid, ref_u = g, uu
    out = {"config": cfg.name, "variant": v or "default", "spread_ms": round(t_sp, 4), "gather_ms": round(t_ga, 4),
           "grid_maxrel": float(np.max(np.abs(g - ref_grid)) / np.max(np.abs(ref_grid))),
           "u_maxrel": float(np.max(np.abs(uu - ref_u)) / np.max(np.abs(ref_u)))}
    print(json.dumps(out), flush=True)
