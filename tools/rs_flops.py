"""Real-space kernel probe: one real-space-only evaluation per (kernel,
symmetric) variant on a uniform periodic system, printing the accepted pair
count. Run under `ncu -k regex:realspace --metrics <fp64 op counters>` to
obtain executed fp64 flops per pair (bench.py FLOPS_PER_PAIR).

    python tools/rs_flops.py            # all six variants, N = 2e5
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_01255_b200 as S  # noqa: E402


def main():
    N = int(os.environ.get("RS_N", "200000"))
    eng = S.Engine(0)
    rng = np.random.default_rng(5)
    out = []
    for kind in (S.Kernel.stokeslet, S.Kernel.stresslet, S.Kernel.rotlet):
        x = rng.random((N, 3))
        f = rng.standard_normal((N, 3))
        nu = None
        if kind == S.Kernel.stresslet:
            g = rng.standard_normal((N, 3))
            nu = g / np.linalg.norm(g, axis=1, keepdims=True)
        cell = S.Cell((1.0, 1.0, 1.0))
        sysm = S.SourceSystem(kind, cell, 3, x, f, nu)
        xi = 37.0 * (N / 1e6) ** (1 / 3)
        sel = S.select_parameters(kind, 3, cell, S.source_quantity(sysm), xi, S.ToleranceSpec(1e-8),
                                  S.SelectionOptions(4, S.WindowKind.pkb, True))
        for sym in (True, False):
            sess = S.Session(sel.params, cell, eng)
            dx = torch.from_numpy(x).cuda()
            sess.set_sources(dx, torch.from_numpy(f).cuda(), torch.from_numpy(nu).cuda() if nu is not None else None)
            if sym:
                sess.set_targets(None, True)
            else:
                sess.set_targets(dx + 1e-13, False)  # distinct target array: non-symmetric kernel
            u = torch.zeros((N, 3), dtype=torch.float64, device="cuda")
            sess.pair_count(reset=True)
            sess.evaluate(u, 0, 1, 2)
            torch.cuda.synchronize()
            out.append({"kernel": kind.name, "symmetric": sym, "N": N, "xi": xi, "rc": sel.params.rc,
                        "pairs": sess.pair_count(reset=True)})
            print(json.dumps(out[-1]), flush=True)
            sess.close()


if __name__ == "__main__":
    main()
