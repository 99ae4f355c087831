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


def test_d0_slab_splits_are_consistent():
    """All-to-all split sizes of the slab-distributed D = 0 solve: what rank p
    sends to r is what r expects from p, and the buffers tile the data."""
    from paper_2210_01255_b200.parallel import D0Slabs
    for world in (1, 2, 3, 5, 8):
        for m0, m1, m2, h2, C in ((480, 256, 256, 257, 3), (37, 20, 23, 24, 9)):
            sl = D0Slabs({"m": (m0, m1, m2), "n": (2 * m0, 2 * m1, 2 * m2), "h2": h2, "C": C}, world)
            assert sl.xb[0] == 0 and sl.xb[-1] == m0 and sl.kb[-1] == h2
            for r in range(world):
                for p in range(world):
                    assert sl.fwd_send_splits(p)[r] == sl.fwd_recv_splits(r)[p]
                    assert sl.inv_send_splits(p)[r] == sl.inv_recv_splits(r)[p]
                assert sum(sl.fwd_send_splits(r)) == C * sl.nx(r) * m1 * h2
                assert sum(sl.inv_send_splits(r)) == 3 * sl.nk(r) * m0 * m1
            assert sum(sum(sl.fwd_send_splits(r)) for r in range(world)) == C * m0 * m1 * h2


class FakeD0Session:
    """numpy stand-in for the slab-distributed D = 0 stages (same buffer
    layouts as include/sewald_gpu.h) with a fixed real, even k-space
    operator, so d0_sharded_solve's collectives can run on gloo (tests only)."""

    def __init__(self, m, C, pad=2):
        self.m, self.C = m, C
        self.n = tuple(pad * v for v in m)  # pad 2: D = 0 box; pad 1: the periodic D = 3 box
        self.h2 = self.n[2] // 2 + 1
        k = [np.fft.fftfreq(v) * v for v in self.n]
        kz = np.arange(self.h2)
        self.H = 1.0 / (1.0 + k[0][None, :, None] ** 2 + k[1][None, None, :] ** 2 + kz[:, None, None] ** 2)

    def d0_geometry(self, precompute_0p=True):
        return {"m": self.m, "n": self.n, "h2": self.h2, "C": self.C}

    def full_flow(self, grid):
        g = grid.reshape(self.C, *self.m)[:3]
        F = np.fft.rfftn(g, s=self.n, axes=(1, 2, 3))  # [3][kx][ky][kz]
        F *= np.transpose(self.H, (1, 2, 0))[None]
        return np.fft.irfftn(F, s=self.n, axes=(1, 2, 3))[:, :self.m[0], :self.m[1], :self.m[2]]

    def d0_forward(self, grid_slab, xa, xb, kb, send, precompute_0p=True):
        import torch
        Z = np.fft.rfft(grid_slab.numpy(), n=self.n[2], axis=-1)
        send.copy_(torch.from_numpy(np.concatenate([Z[..., kb[q]:kb[q + 1]].ravel() for q in range(len(kb) - 1)])))

    def d0_middle(self, recv, xbd, ka, kb, send, precompute_0p=True):
        import torch
        nk, m0, m1 = kb - ka, self.m[0], self.m[1]
        r = recv.numpy()
        parts, o = [], 0
        for p in range(len(xbd) - 1):
            sz = self.C * (xbd[p + 1] - xbd[p]) * m1 * nk
            parts.append(r[o:o + sz].reshape(self.C, xbd[p + 1] - xbd[p], m1, nk))
            o += sz
        A = np.transpose(np.concatenate(parts, axis=1), (0, 3, 1, 2))[:3]  # [3][nk][m0][m1]
        F = np.fft.fft2(A, s=self.n[:2], axes=(2, 3)) * self.H[ka:kb][None]
        B = np.fft.ifft2(F, axes=(2, 3))[:, :, :m0, :m1]
        send.copy_(torch.from_numpy(np.concatenate([B[:, :, xbd[q]:xbd[q + 1], :].ravel()
                                                    for q in range(len(xbd) - 1)])))

    def d0_inverse(self, recv, xa, xb, kb, flow_slab, precompute_0p=True):
        import torch
        nxs, m1 = xb - xa, self.m[1]
        r = recv.numpy()
        parts, o = [], 0
        for p in range(len(kb) - 1):
            sz = 3 * (kb[p + 1] - kb[p]) * nxs * m1
            parts.append(r[o:o + sz].reshape(3, kb[p + 1] - kb[p], nxs, m1))
            o += sz
        Z = np.transpose(np.concatenate(parts, axis=1), (0, 2, 3, 1))  # [3][nxs][m1][h2]
        flow_slab.copy_(torch.from_numpy(np.fft.irfft(Z, n=self.n[2], axis=-1)[..., :self.m[2]]))

    def set_flow(self, flow):
        self.flow = flow.numpy().copy()


def _d0_worker(rank, world, port, outdir, pad=2):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_2210_01255_b200.parallel import d0_sharded_solve
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, C = ((11, 6, 5), 9) if pad == 2 else ((12, 6, 8), 3)
    sess = FakeD0Session(m, C, pad)
    rng = np.random.default_rng(40 + rank)  # per-rank partial grids, summed by the solve
    grid = torch.from_numpy(rng.standard_normal(C * m[0] * m[1] * m[2]))
    d0_sharded_solve(sess, grid, rank, world, dist)
    total = grid.clone()
    dist.all_reduce(total)
    if rank == 0:
        np.save(os.path.join(outdir, "flow.npy"), sess.flow)
        np.save(os.path.join(outdir, "ref.npy"), sess.full_flow(total.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,pad", [(2, 2), (3, 2), (2, 1), (3, 1)])
def test_sharded_solve_gloo(tmp_path, world, pad):
    """d0_sharded_solve with real collectives (gloo, world 2 and 3): grid
    reduction to x-slabs, two all-to-alls, all-gather of the flow slabs; on the
    zero-padded D = 0 box (pad 2) and the unpadded periodic D = 3 box (pad 1)."""
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_d0_worker, args=(world, port, str(tmp_path), pad), nprocs=world, join=True,
                       start_method="spawn")
    flow = np.load(tmp_path / "flow.npy")
    ref = np.load(tmp_path / "ref.npy")
    assert np.max(np.abs(flow - ref)) < 1e-12 * np.max(np.abs(ref))
