"""ORACLE TEST INFRASTRUCTURE — full-size parity fixtures for the BASELINE
configs, produced by the reference itself (oracle/_ref/libsewald_ref.so, the
unmodified reference sources compiled with the committed shims).

    make -C oracle lib && python oracle/make_fullsize_golden.py c2 [c3 c4 c5 ...]

For each config the seeded inputs of oracle/baseline_inputs.py (the same
bytes the product's workloads.generate draws; the fixture stores their
SHA-256 so a test can prove it) are run once through the reference at the
pinned xi, with the parameters the reference's select_parameters picks
(estimates.cpp:211-268):
  u   = full_potential as realspace.cpp:205-219 assembles it,
  u_F = se_fourier_potential (fourier.cpp:805-852),
  u_R = realspace_potential(starred when targets are the sources,
        realspace.cpp:166-203) on all host threads (realspace.h:40-41).
The fixture keeps u, u_F, u_R at >= 10,240 sampled target indices, plus, over
ALL targets, the sums of squares and eight seeded random projections
sum_i w_i . u_i per field: a wrong value at any target moves a projection by
its error times |w_i|, so matching projections to ~1e-12 relative pins every
target, not only the sampled ones.

Reduced sizes ("c5n1e6" etc.) keep the config's parameters (pinned xi, box,
and the grid / P / rc selected for the full N: Q is scaled to the config's N)
and only lower N; the tag names the reduction.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import baseline_inputs as BI  # noqa: E402
import sewald_ref as R  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")
N_SAMPLE = 10240
N_PROJ = 8


def projections(u: np.ndarray, seed: int) -> np.ndarray:
    """Eight seeded random projections sum_i w_i . u_i (w ~ N(0,1)^{Nt x 3})."""
    rng = np.random.default_rng(seed)
    out = np.empty(N_PROJ)
    for k in range(N_PROJ):
        w = rng.standard_normal(u.shape)
        out[k] = float(np.sum(w * u))
    return out


def run(tag: str, n_threads: int) -> None:
    cfg_index, N, Nt = BI.parse_tag(tag)
    cfg = BI.CONFIGS[cfg_index]
    x, f, nu, xt = BI.generate(cfg_index, N, Nt)
    same = xt is None
    Q = BI.source_quantity(cfg.kind, f, nu)
    # A reduced N keeps the full workload's parameters (grid, P, rc): select
    # with Q scaled to the config's N (Q is a sum over sources, domain.cpp:53-62).
    Q_sel = Q * (cfg.N / x.shape[0])
    p, _ = R.select_parameters(cfg.kind, cfg.d, cfg.L, Q_sel, cfg.xi, cfg.tol, False, 4, cfg.window, True)
    t0 = time.time()
    u, uf, ur, secs = R.full_parts(p, x, f, nu, xt, same, precompute_0p=True, n_threads=n_threads)
    wall = time.time() - t0
    nt = u.shape[0]
    rng = np.random.default_rng(4242 + cfg_index)
    idx = np.sort(rng.choice(nt, size=min(N_SAMPLE, nt), replace=False)).astype(np.int64)
    out = dict(
        tag=tag, config=cfg_index, N=x.shape[0], Nt=nt, kind=cfg.kind, d=cfg.d,
        L=np.asarray(cfg.L, float), xi=cfg.xi, tol=cfg.tol, window=cfg.window, Q=Q, Q_sel=Q_sel,
        params=np.frombuffer(bytes(p), dtype=np.uint8),
        input_sha256=BI.input_hash(x, f, nu, xt),
        idx=idx, u=u[idx], uF=uf[idx], uR=ur[idx],
        ss_u=float(np.sum(u * u)), ss_uF=float(np.sum(uf * uf)), ss_uR=float(np.sum(ur * ur)),
        proj_seed=777 + cfg_index,
        proj_u=projections(u, 777 + cfg_index), proj_uF=projections(uf, 777 + cfg_index),
        proj_uR=projections(ur, 777 + cfg_index),
        ref_seconds=np.array([secs["fourier"], secs["realspace"], secs["terms"], secs["total"]]),
        ref_threads=n_threads,
    )
    path = os.path.join(OUT, f"fullsize_{tag}.npz")
    np.savez_compressed(path, **out)
    info = dict(tag=tag, N=int(x.shape[0]), Nt=int(nt), M=list(p.M), M_ext=list(p.M_ext), P=p.P,
                rc=p.rc, wall_s=wall, **secs,
                u_rms=float(np.sqrt(out["ss_u"] / nt)))
    print(json.dumps(info), flush=True)


if __name__ == "__main__":
    threads = int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1))
    for t in sys.argv[1:] or ["c2"]:
        run(t, threads)
