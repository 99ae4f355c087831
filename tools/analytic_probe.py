"""Timing probe of the GPU analytic oracles (csrc/analytic.cu) at small sizes."""
import sys, time, math
import numpy as np
sys.path.insert(0, ".")
import paper_2210_01255_b200 as S
from paper_2210_01255_b200 import analytic as A

def sysm(kind, d, N, seed=1):
    rng = np.random.default_rng(seed)
    x = rng.random((N, 3)); f = rng.standard_normal((N, 3)); nu = None
    if kind == S.Kernel.stresslet:
        g = rng.standard_normal((N, 3)); nu = g / np.linalg.norm(g, axis=1, keepdims=True)
    return S.SourceSystem(kind, S.Cell((1, 1, 1)), d, x, f, nu)

t = time.time(); K = A.incomplete_bessel_K4([0.1, 1.0], [0.0, 3.0]); print("K4", K, time.time() - t, flush=True)
for N in (50, 200, 1000):
    for d in (3, 2, 1, 0):
        for kind in (S.Kernel.stokeslet, S.Kernel.rotlet, S.Kernel.stresslet):
            s = sysm(kind, d, N)
            T = S.TargetSet.from_sources(s)
            t = time.time()
            if d == 0:
                u = A.direct_sum_0p(s, T, True)
            else:
                u = A.fourier_reference_potential(s, T, 10.0)
            print(f"N={N} d={d} {kind.name}: {time.time() - t:.3f} s rms {math.sqrt(np.mean(u**2)):.3e}", flush=True)
