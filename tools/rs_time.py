"""Time the real-space kernel alone (Session.evaluate(parts=2), cell order
cached) at a BASELINE config and check it against the reference's own full-size
fixture (u_R at the sampled targets). SEWALD_LIB selects a variant build.

    SEWALD_LIB=paper_2210_01255_b200/lib/var_x/libsewald_gpu.so python tools/rs_time.py [config] [reps]
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
u = torch.zeros((nt, 3), dtype=torch.float64, device=dev)
sess.evaluate(u, 0, 1, 2)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sess.evaluate(u, 0, 1, 2)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
out = {"lib": os.environ.get("SEWALD_LIB", "default"), "config": cfg.name, "rs_ms": sorted(ts)[len(ts) // 2],
       "rs_ms_all": [round(t, 3) for t in ts]}
fx = os.path.join(ROOT, "tests", "golden", f"fullsize_c{cfg.index}.npz")
if os.path.exists(fx):
    g = np.load(fx)
    uu = u.cpu().numpy()[g["idx"]]
    ref = g["uR"]
    out["uR_rel_rms"] = float(np.sqrt(np.mean(np.sum((uu - ref) ** 2, 1)) / np.mean(np.sum(ref ** 2, 1))))
print(json.dumps(out))
