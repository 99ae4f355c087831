"""Multi-process run of the product's distributed step on the GPU box:
world size 2, both ranks on cuda:0 with the gloo backend (a functional check
of the multi-GPU code path on a one-GPU box; NCCL needs one GPU per rank).
Each rank runs parallel.sharded_step with a real device Session; the summed
result must equal the single-process full_potential. Covers the replicated
solve (D = 3, grid all-reduce + symmetric real-space reactions) and the
slab-distributed D = 0 and D = 3 solves (reduce -> all-to-all -> all-to-all ->
all-gather), world sizes 2 and 3."""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT, rel_rms

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _system(d, kind, N):
    rng = np.random.default_rng(77 + d + 10 * kind)
    L = (1.0, 1.0, 1.0) if d else (2.0, 1.0, 1.0)
    x = rng.random((N, 3)) * np.asarray(L)
    f = rng.standard_normal((N, 3))
    nu = rng.standard_normal((N, 3)) if kind == 1 else None
    return L, x, f, nu


def _worker(rank, world, port, outdir, d, kind, N, slab=None):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import paper_2210_01255_b200 as S
    from paper_2210_01255_b200.parallel import sharded_step
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, x, f, nu = _system(d, kind, N)
    sysm = S.SourceSystem(S.Kernel(kind), S.Cell(L), d, x, f, nu)
    sel = S.select_parameters(sysm.kind, d, sysm.cell, S.source_quantity(sysm), 9.0, S.ToleranceSpec(1e-8))
    dev = torch.device("cuda", 0)
    T = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    sess = S.Session(sel.params, sysm.cell)
    sess.set_sources(T(x), T(f), T(nu))
    sess.set_targets(None, True)
    grid = torch.zeros(sess.grid_size(), dtype=torch.float64, device=dev)
    u = torch.zeros((N, 3), dtype=torch.float64, device=dev)
    use_slab = (d == 0) if slab is None else slab
    sharded_step(sess, N, grid, u, rank, world, all_reduce=dist.all_reduce,
                 slab_dist=dist if use_slab else None)
    torch.cuda.synchronize()
    if rank == 0:
        np.save(os.path.join(outdir, "u.npy"), u.cpu().numpy())
        np.save(os.path.join(outdir, "uref.npy"), S.full_potential(sysm, S.TargetSet.from_sources(sysm), sel.params))
    sess.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("d,kind,slab,world", [(3, 0, False, 2), (0, 0, True, 2), (0, 1, True, 2), (2, 2, False, 2),
                                               (3, 0, True, 2), (3, 1, True, 3), (3, 2, True, 3)])
def test_sharded_step_ranks_gpu(tmp_path, d, kind, slab, world):
    """slab: the k-space step slab-distributed (reduce-scatter, two all-to-alls,
    all-gather) instead of a grid all-reduce and a replicated solve."""
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path), d, kind, 3000, slab), nprocs=world, join=True,
                       start_method="spawn")
    u = np.load(tmp_path / "u.npy")
    uref = np.load(tmp_path / "uref.npy")
    assert rel_rms(u, uref) < 1e-12
