"""World-size-2 gloo test of the multi-GPU decomposition (parallel.sharded_step)
on CPU. The device session is replaced by a CPU test double with the same
stage interface built on the reference itself (oracle/_ref), so the test
checks the product's orchestration: source slices spread separately and
summed by the all-reduce, replicated k-space solve, disjoint target parts
summed into the full result. Compared against the single-process reference."""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class RefSession:
    """CPU stand-in for paper_2210_01255_b200.Session (tests only)."""

    def __init__(self, R, p, kind, d, L, x, f, nu):
        self.R, self.p, self.kind, self.d, self.L = R, p, kind, d, L
        self.x, self.f, self.nu = x, f, nu
        self.shape = (9 if kind == 1 else 3, p.M_ext[0], p.M_ext[1], p.M_ext[2])

    def spread(self, i0, i1, grid):
        nu = None if self.nu is None else self.nu[i0:i1]
        g = self.R.spread(self.p, self.x[i0:i1], self.f[i0:i1], nu)
        grid.copy_(__import__("torch").from_numpy(g.ravel()))

    def solve(self, grid, precompute_0p=True):
        self.flow = self.R.solve_grid(self.p, grid.numpy().reshape(self.shape), precompute_0p)

    def evaluate(self, u, part, nparts, parts=7):
        import torch
        from paper_2210_01255_b200.parallel import slice_bounds
        ncl = (self.x.shape[0] + 31) // 32  # cluster-aligned parts, as the device session
        c0, c1 = slice_bounds(ncl, part, nparts)
        t0, t1 = min(32 * c0, self.x.shape[0]), min(32 * c1, self.x.shape[0])
        u.zero_()
        uF = self.R.gather(self.p, self.flow, self.x[t0:t1])
        uR = self.R.realspace_potential(self.kind, self.d, self.L, self.x, self.f, self.nu, None, True,
                                        self.p.xi, self.p.rc, True)[t0:t1]
        out = uF + uR
        if self.kind == 0:
            out += -4.0 * self.p.xi / np.sqrt(np.pi) * self.f[t0:t1]
        u[t0:t1] = torch.from_numpy(out)


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist
    import sewald_ref as R
    from paper_2210_01255_b200.parallel import sharded_step
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(9)
    N = 300
    x = rng.random((N, 3))
    f = rng.standard_normal((N, 3))
    p, _ = R.select_parameters(0, 3, (1, 1, 1), float(np.sum(f * f)), 8.0, 1e-8)
    sess = RefSession(R, p, 0, 3, (1.0, 1.0, 1.0), x, f, None)
    grid = torch.zeros(3 * p.M_ext[0] * p.M_ext[1] * p.M_ext[2], dtype=torch.float64)
    u = torch.zeros((N, 3), dtype=torch.float64)
    sharded_step(sess, N, grid, u, rank, world, all_reduce=dist.all_reduce)
    if rank == 0:
        np.save(os.path.join(outdir, "u.npy"), u.numpy())
        np.save(os.path.join(outdir, "uref.npy"), R.full_potential(p, x, f))
    dist.destroy_process_group()


def test_sharded_step_gloo_world2(tmp_path, ref):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    u = np.load(tmp_path / "u.npy")
    ur = np.load(tmp_path / "uref.npy")
    rel = np.sqrt(np.mean(np.sum((u - ur) ** 2, 1)) / np.mean(np.sum(ur ** 2, 1)))
    assert rel < 1e-13, rel


def test_slice_bounds_partition():
    from paper_2210_01255_b200.parallel import slice_bounds
    for n in (0, 1, 7, 1000, 1_000_003):
        for w in (1, 2, 3, 8):
            parts = [slice_bounds(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1
    with pytest.raises(ValueError):
        slice_bounds(10, 2, 2)
