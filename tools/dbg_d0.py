import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import paper_2210_01255_b200 as S
from conftest import load_golden, rel_rms
import test_gpu_parity as T
from paper_2210_01255_b200.parallel import (D0Slabs, d0_stage_forward, d0_stage_inverse, d0_stage_middle, emulate_all_to_all)
g = load_golden("stokeslet_d0")
sysm = T.system_from(S, g); tg = T.targets_from(S, g, sysm); params = T.params_from_bytes(S, g["params"])
def chk(tag): print(tag, rel_rms(S.full_potential(sysm, tg, params), g["u"]), flush=True)
chk("u0")
rng = np.random.default_rng(900)
N = 3000; L = (2.0, 1.0, 1.0); d = 0; kind = 0; world = 2; table = True
x = rng.random((N, 3)) * np.asarray(L); f = rng.standard_normal((N, 3))
sy = S.SourceSystem(S.Kernel(kind), S.Cell(L), d, x, f, None)
sel = S.select_parameters(sy.kind, d, sy.cell, S.source_quantity(sy), 9.0, S.ToleranceSpec(1e-8))
dev = torch.device("cuda", 0)
sess = S.Session(sel.params, sy.cell)
sess.set_sources(torch.from_numpy(x).to(dev), torch.from_numpy(f).to(dev), None)
sess.set_targets(None, True)
chk("after session create")
grid = torch.zeros(sess.grid_size(), dtype=torch.float64, device=dev)
sess.spread(0, N, grid); chk("after spread")
sess.solve(grid, table); chk("after solve")
u_ref = torch.zeros((N, 3), dtype=torch.float64, device=dev)
sess.evaluate(u_ref, 0, 1, 1); chk("after evaluate")
sl = D0Slabs(sess.d0_geometry(table), world); chk("after geometry")
gg = grid.view(sl.C, sl.m[0], sl.m[1], sl.m[2])
sends = [d0_stage_forward(sess, sl, r, gg[:, sl.xb[r]:sl.xb[r + 1]].contiguous(), table) for r in range(world)]
chk("after fwd")
recvs = emulate_all_to_all(sends, [sl.fwd_send_splits(r) for r in range(world)], [sl.fwd_recv_splits(r) for r in range(world)])
sends2 = [d0_stage_middle(sess, sl, r, recvs[r], table) for r in range(world)]
chk("after middle")
recvs2 = emulate_all_to_all(sends2, [sl.inv_send_splits(r) for r in range(world)], [sl.inv_recv_splits(r) for r in range(world)])
flow = torch.cat([d0_stage_inverse(sess, sl, r, recvs2[r], table) for r in range(world)], dim=1).contiguous()
chk("after inverse")
sess.close(); chk("after close")
