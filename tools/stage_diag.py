"""Per-mode scale differences GPU vs reference (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import paper_2210_01255_b200 as S
import sewald_ref as ref
from test_stages import _cases, _params, _from_ref

for kind in (0, 1, 2):
    comps = S.strength_components(S.Kernel(kind))
    rng = np.random.default_rng(1)
    for name, grid, plan, R in _cases(S):
        p = _params(S, kind, grid, plan, R)
        rp = ref.params_from(p.to_c())
        phi = rng.standard_normal((comps,) + tuple(grid.M_ext))
        r = ref.aft_forward(rp, phi)
        F = S.aft_forward(phi, grid, plan)
        spec = S.ModifiedKernelSpec.optimal(S.Kernel(kind), grid.d, 1.0 if grid.d == 3 else R)
        Fs = S.scale(_from_ref(S, r), spec, p.xi, p.window, grid)
        rs = ref.scale(rp, r, (kind, grid.d, spec.R, spec.a_B, spec.b_B, spec.ell_H, spec.ell_B, spec.c_B), p.xi)
        for k in ("far", "near", "zero"):
            a, b = getattr(F, k), r[k]
            fe = np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300) if b.size else 0
            a, b = getattr(Fs, k), rs[k]
            if not b.size:
                continue
            d = np.abs(a - b)
            i = int(np.argmax(d))
            print(f"kind={kind} {name:6s} {k:4s} fwd={fe:.1e} scale={d[i]/np.max(np.abs(b)):.2e} at {i} "
                  f"val={b[i]:.6e} pointwise={d[i]/max(abs(b[i]),1e-300):.2e} n={b.size}")
