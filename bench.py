#!/usr/bin/env python3
"""Benchmark of the Spectral Ewald hot path (BASELINE.json metric: targets/s,
N=1e6 triply periodic stokeslets, fp64, tol 1e-8) on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

A step = one full-potential evaluation (sources -> spread -> FFT -> k-space
scale -> IFFT -> gather, plus the real-space cell-list sum and the self
term) over the whole synthetic workload. `value` is measured with inputs
resident in HBM through the device session (sort/bucketing included every
step, as positions change in time stepping); `e2e` through the public API
(full_potential on 1 GPU, parallel.full_potential_sharded on N) with pinned
host buffers (H2D of the inputs and D2H of u inside the timed region).
`--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU, NCCL). Multi-GPU: every
rank spreads 1/N of the sources, the grid is summed with an NCCL all-reduce
(D = 0: slab-distributed solve), every rank evaluates 1/N of the targets
(strong scaling: the workload is fixed as N grows).

`--impl reference` runs the reference's own CPU implementation
(oracle/_ref: the unmodified reference sources compiled with shims) over the
WHOLE workload once, on rank 0 only: se_fourier_potential single-threaded as
shipped and realspace_potential on all host threads (its only parallel
knob, realspace.h:40-41), assembled as realspace.cpp:205-219. That run is
the measurement (steps = 1, warmup = 0); it imports only oracle/ modules.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# DRAM bytes (read + write) per launch of the dominant kernel from one
# `ncu --set full` capture of the kernel at the same workload (profiles/r2_ncu_realspace_sym_v6.txt).
TRAFFIC_BYTES = {"c2_stokeslet_d3_N1e6": 97_504_768 + 4_602_624}

# Algorithmic fp64 flops per accepted (directed) real-space pair of the
# implemented evaluation, keyed (kernel, symmetric): ncu thread-level
# 2*DFMA + DMUL + DADD of the kernel divided by the kernel's own pair counter
# (tools/gpu_probe3.sh: branchy kernel variant so idle lanes execute nothing;
# profiles/r1_realspace_flops_v2.txt; DESIGN.md "real-space
# roofline"). The symmetric kernel (targets == sources) evaluates each
# unordered pair once and charges half of it to each direction.
FLOPS_PER_PAIR = {
    (0, True): 62.0, (1, True): 80.8, (2, True): 57.4,
    (0, False): 111.5, (1, False): 139.4, (2, False): 105.4,
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2)
    # split parameter override (not the BASELINE workload: BASELINE.md §3 pins xi
    # per config): the paper's N_rc balancing of real-space vs Fourier work
    # applied on the B200; parity is then reported as
    # xi-invariance against the pinned-xi fixture (tau level, not 1e-12)
    ap.add_argument("--xi", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    # supplementary: the same workload at the split parameter balanced for the
    # B200 (PAPER.md:3790-3800 applied on this GPU; not the BASELINE-pinned xi)
    ap.add_argument("--no-balanced", action="store_true")
    ap.add_argument("--profile-stages", action="store_true", default=True)
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1].split()[0]))
                smax.append(float(parts[2].split()[0]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def select(S, cfg, x, f, nu):
    cell = S.Cell(cfg.L)
    sysm = S.SourceSystem(cfg.kind, cell, cfg.d, x, f, nu)
    sel = S.select_parameters(cfg.kind, cfg.d, cell, S.source_quantity(sysm), cfg.xi,
                              S.ToleranceSpec(cfg.tol), S.SelectionOptions(4, cfg.window, True))
    return sysm, sel


KERNEL_NAMES = {0: "stokeslet", 1: "stresslet", 2: "rotlet"}
WINDOW_NAMES = {0: "kb", 1: "pkb", 2: "tg"}


def config_dict(name, N, Nt, kind, d, xi, tol, M_ext, P, window, rc, ws):
    """The `config` of both arms (identical for the same workload and N)."""
    par = (f"targets+source-slices x{ws}, NCCL all-reduce of the grid" if d != 0 or ws == 1 else
           f"targets+source-slices x{ws}, slab FFT (NCCL reduce-scatter, 2 all-to-all, all-gather)")
    return {"workload": name, "N": int(N), "Nt": int(Nt), "kernel": KERNEL_NAMES[int(kind)], "d": int(d),
            "xi": float(xi), "tol": float(tol), "M_ext": [int(v) for v in M_ext], "P": int(P),
            "window": WINDOW_NAMES[int(window)], "rc": float(rc), "parallelism": par,
            "l2": "GPU arm: flushed between steps (256 MB write inside the timed loop)"}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def fixture_parity(u, cfg_index, xi_override=False):
    """rel-RMS of u against the reference's own full-size run stored in
    tests/golden/fullsize_c<k>.npz (sampled targets) and the worst
    all-target projection deviation (see tests/test_fullsize_parity.py)."""
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_c{cfg_index}.npz")
    if not os.path.exists(path):
        return None
    g = np.load(path)
    if int(g["Nt"]) != u.shape[0]:
        return None
    idx = g["idx"]
    ref = g["u"]
    rel = float(np.sqrt(np.mean(np.sum((u[idx] - ref) ** 2, 1)) / np.mean(np.sum(ref ** 2, 1))))
    rng = np.random.default_rng(int(g["proj_seed"]))
    pj = np.array([float(np.sum(rng.standard_normal(u.shape) * u)) for _ in range(len(g["proj_u"]))])
    pdev = float(np.max(np.abs(pj - g["proj_u"])) / np.sqrt(float(g["ss_u"])))
    out = {"fixture": os.path.relpath(path, ROOT), "rel_rms_sampled": rel, "n_sampled": int(len(idx)),
           "proj_dev_all_targets": pdev, "bar": 1e-12}
    if xi_override:  # another xi: same sum to the tolerance, not to rounding
        out.update({"bar": 1e-7, "note": "xi differs from the fixture's pinned xi: xi-invariance at the tau level"})
    return out


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref)
# ---------------------------------------------------------------------------

def cpu_reference_sample(cfg, params_c, x, f, nu, xt, n_threads, sample=10000, seed=7):
    """cpu_baseline of the GPU arm (rank 0, N = 1; ~10-30 s of CPU work): the
    reference's per-unit costs measured on `sample` sources / targets of the
    SAME workload and combined into the whole workload's time
        T = T_fixed + N t_spread + Nt t_gather + Nt t_realspace.
    T_fixed is one reference flow_field call on a single source (grid zero,
    FFT, scale, IFFT) plus the real-space cell-list build over all N sources;
    the per-unit rates have those fixed costs subtracted (a 1-point call of
    the same stage is timed and removed), so they are not inflated by the
    sample size. Real space runs for the sampled targets against all N
    sources on `n_threads` threads. This is a model of the full run, which
    `bench.py --impl reference` measures directly."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import sewald_ref as R

    p = R.params_from(params_c)
    rng = np.random.default_rng(seed)
    N = x.shape[0]
    same = xt is None
    tx = x if same else xt
    Nt = tx.shape[0]
    si = rng.choice(N, size=min(sample, N), replace=False)
    ti = rng.choice(Nt, size=min(sample, Nt), replace=False)
    nus = lambda idx: None if nu is None else nu[idx]
    clock = time.perf_counter
    t0 = clock()
    R.flow_field(p, x[:1], f[:1], nus(slice(0, 1)))
    t_fft = clock() - t0
    t0 = clock()
    R.spread(p, x[:1], f[:1], nus(slice(0, 1)))
    t_sp1 = clock() - t0
    t0 = clock()
    R.spread(p, x[si], f[si], nus(si))
    t_spread = max(clock() - t0 - t_sp1, 0.0) / len(si)
    field = np.zeros((3, p.M_ext[0], p.M_ext[1], p.M_ext[2]))
    t0 = clock()
    R.gather(p, field, tx[:1])
    t_g1 = clock() - t0
    t0 = clock()
    R.gather(p, field, tx[ti])
    t_gather = max(clock() - t0 - t_g1, 0.0) / len(ti)
    # same-point targets are nudged by 1e-9 so the (skipped) self pair is not r = 0
    tt = tx[ti] + (1e-9 if same else 0.0)
    t0 = clock()
    R.realspace_potential(int(cfg.kind), cfg.d, cfg.L, x, f, nu, tt[:1], False, float(params_c.xi),
                          float(params_c.rc), False, 1)
    t_cells = clock() - t0
    t0 = clock()
    R.realspace_potential(int(cfg.kind), cfg.d, cfg.L, x, f, nu, tt, False, float(params_c.xi),
                          float(params_c.rc), False, n_threads)
    t_rs = max(clock() - t0 - t_cells, 0.0) / len(ti)
    total = t_fft + t_cells + N * t_spread + Nt * t_gather + Nt * t_rs
    detail = dict(fixed_fft_s=t_fft, cell_list_build_s=t_cells, spread_us_per_source=t_spread * 1e6,
                  gather_us_per_target=t_gather * 1e6, realspace_us_per_target=t_rs * 1e6,
                  modelled_full_workload_s=total, sample_sources=len(si), sample_targets=len(ti))
    return Nt / total, detail


def run_reference(args, cfg_index):
    """The reference arm: the unmodified reference (oracle/_ref) runs the whole
    workload once on this host. Only oracle/ modules are imported (inputs:
    oracle/baseline_inputs.py, the same bytes the GPU arm draws; parameters:
    the reference's own select_parameters)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import baseline_inputs as BI
    import sewald_ref as R
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libsewald_ref.so not built"}))
        return
    if cfg_index not in BI.CONFIGS:
        print(json.dumps({"impl": "reference", "unavailable": f"config {cfg_index} is not a BASELINE config"}))
        return
    wall0 = time.perf_counter()
    cfg = BI.CONFIGS[cfg_index]
    x, f, nu, xt = BI.generate(cfg_index)
    same = xt is None
    Nt = x.shape[0] if same else xt.shape[0]
    Q = BI.source_quantity(cfg.kind, f, nu)
    p, _ = R.select_parameters(cfg.kind, cfg.d, cfg.L, Q, cfg.xi, cfg.tol, False, 4, cfg.window, True)
    nthreads = os.cpu_count() or 1
    t0 = time.perf_counter()
    u, _, _, secs = R.full_parts(p, x, f, nu, xt, same, precompute_0p=True, n_threads=nthreads)
    run_s = time.perf_counter() - t0
    value = Nt / run_s
    line = {
        "impl": "reference", "metric": "targets/sec", "value": value, "unit": "targets/s",
        "n_gpus": ws, "steps": 1, "warmup": 0, "requested": {"steps": args.steps, "warmup": args.warmup},
        "ms_per_step": 1e3 * run_s, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded uniform positions, N(0,1) strengths; BASELINE config)",
        "config": config_dict(cfg.name, x.shape[0], Nt, cfg.kind, cfg.d, cfg.xi, cfg.tol, list(p.M_ext), p.P,
                              p.win_kind, p.rc, ws),
        "cpu_baseline": {"value": value, "unit": "targets/s", "cores": nthreads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": ("the whole workload, measured once: reference C++ (oracle/_ref) "
                                    "se_fourier_potential single-threaded as shipped + realspace_potential on "
                                    f"{nthreads} threads + self/zero-mode/gauge terms (realspace.cpp:205-219)"),
                         "stage_s": secs},
        "e2e": {"value": value, "unit": "targets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "parity_vs_fixture": fixture_parity(u, cfg_index),
        "wall_s": time.perf_counter() - wall0,
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# our engine
# ---------------------------------------------------------------------------

# profiles/r2_xi_balance_c2.txt (c2: 57.6 ms at the pinned xi 37 ... 24.3 at 63-71) and
# profiles/r2_xi_balance_c3_c4_c5.txt (c3: 117 -> 62.5 ms at 61; c4: 56.8 -> 41.6 at 46; c5's
# pinned 68.5 is already the fastest measured)
BALANCED_XI = {2: 63.0, 3: 61.0, 4: 46.0}


def balanced_probe(S, cfg, x, f, nu, xt, engine, stream, dev, l2, steps=5, warmup=2):
    """Same inputs, tolerance and window at the B200-balanced split parameter
    (device-resident, L2 flushed, CUDA events): a supplementary figure, not the
    headline (BASELINE.md §3 pins xi)."""
    import dataclasses
    import torch
    cb = dataclasses.replace(cfg, xi=BALANCED_XI[cfg.index])
    _, sel = select(S, cb, x, f, nu)
    p = sel.params
    same = xt is None
    Nt = x.shape[0] if same else xt.shape[0]
    sess = S.Session(p, S.Cell(cb.L), engine)
    dx, df = torch.from_numpy(x).to(dev), torch.from_numpy(f).to(dev)
    dnu = torch.from_numpy(nu).to(dev) if nu is not None else None
    dxt = torch.from_numpy(xt).to(dev) if xt is not None else None
    grid = torch.empty(sess.grid_size(), dtype=torch.float64, device=dev)
    u = torch.zeros((Nt, 3), dtype=torch.float64, device=dev)

    def step():
        sess.set_sources(dx, df, dnu)
        sess.set_targets(dxt, same)
        sess.spread(0, x.shape[0], grid)
        sess.solve(grid, True)
        sess.evaluate(u, 0, 1, 7)

    for _ in range(warmup):
        l2.fill_(1.0)
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        l2.fill_(1.0)
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(stream)
    sess.spread(0, x.shape[0], grid)
    ev[1].record(stream)
    sess.solve(grid, True)
    ev[2].record(stream)
    sess.evaluate(u, 0, 1, 2)
    ev[3].record(stream)
    torch.cuda.synchronize()
    st = {"spread(incl. bucket sort)": ev[0].elapsed_time(ev[1]), "fft+scale+ifft": ev[1].elapsed_time(ev[2]),
          "realspace": ev[2].elapsed_time(ev[3])}
    u.zero_()
    step()
    uu = u.cpu().numpy()
    out = {"note": "supplementary, not the headline: same inputs / tolerance / window at the split parameter "
                   "balanced for the B200 (PAPER.md:3790-3800); BASELINE.md pins xi per config",
           "xi": cb.xi, "M_ext": [int(v) for v in p.grid.M_ext], "P": int(p.window.P), "rc": float(p.rc),
           "ms_per_step": ms, "value": Nt / (ms * 1e-3), "unit": "targets/s", "steps": steps, "warmup": warmup,
           "stages_ms": {k: round(v, 4) for k, v in st.items()},
           "parity_vs_fixture": fixture_parity(uu, cfg.index, True)}
    del sess, grid, u
    torch.cuda.empty_cache()
    return out


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2210_01255_b200 as S
    from paper_2210_01255_b200.workloads import generate

    ws, rank, local = dist_env()
    # SEWALD_DIST_BACKEND=gloo: functional multi-rank check on a box with fewer GPUs
    # than ranks (ranks share devices; not a timing configuration)
    backend = os.environ.get("SEWALD_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    x, f, nu, xt = generate(cfg)
    sysm, sel = select(S, cfg, x, f, nu)
    params = sel.params
    same = xt is None
    N = x.shape[0]
    Nt = N if same else xt.shape[0]

    engine = S.Engine(local)
    # A dedicated (non-default) torch stream shared with the engine, so CUDA
    # events, NCCL collectives and the engine's kernels are stream-ordered.
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    engine.set_stream(stream.cuda_stream)
    sess = S.Session(params, S.Cell(cfg.L), engine)
    dx = torch.from_numpy(x).to(dev)
    df = torch.from_numpy(f).to(dev)
    dnu = torch.from_numpy(nu).to(dev) if nu is not None else None
    dxt = torch.from_numpy(xt).to(dev) if xt is not None else None
    grid = torch.empty(sess.grid_size(), dtype=torch.float64, device=dev)
    u = torch.zeros((Nt, 3), dtype=torch.float64, device=dev)
    l2 = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    i0, i1 = N * rank // ws, N * (rank + 1) // ws

    from paper_2210_01255_b200.parallel import sharded_step, use_slabs

    def step():
        sess.set_sources(dx, df, dnu)
        sess.set_targets(dxt, same)
        sharded_step(sess, N, grid, u, rank, ws, all_reduce=dist.all_reduce if ws > 1 else None,
                     slab_dist=dist if use_slabs(cfg.d, ws) else None)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 0)):
        l2.fill_(1.0)
        step()
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    launches0 = engine.launch_count()
    sess.pair_count(reset=True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        l2.fill_(1.0)
        step()
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    launches = engine.launch_count() - launches0
    ms_total = e0.elapsed_time(e1)
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    value = Nt / (ms_per_step * 1e-3)
    pairs = sess.pair_count(reset=True) / max(args.steps, 1)
    u_step = u.cpu().numpy() if rank == 0 else None  # the last timed step's velocity (all targets)

    # per-stage device times (one instrumented step on the same stream)
    stages = {}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    torch.cuda.synchronize()
    ev[0].record(stream)
    sess.set_sources(dx, df, dnu)
    sess.set_targets(dxt, same)
    ev[1].record(stream)
    sess.spread(i0, i1, grid)
    ev[2].record(stream)
    if ws > 1:
        dist.all_reduce(grid)
    ev[3].record(stream)
    sess.solve(grid, True)
    ev[4].record(stream)
    sess.evaluate(u, rank, ws, 2)  # real space alone (includes the cell sort)
    ev[5].record(stream)
    sess.evaluate(u, rank, ws, 1 | 4)  # gather + terms
    ev[6].record(stream)
    torch.cuda.synchronize()
    names = ["upload+validate", "spread(incl. bucket sort)", "allreduce", "fft+scale+ifft",
             "realspace(incl. cell sort)", "gather+terms"]
    for i, nm in enumerate(names):
        stages[nm] = round(ev[i].elapsed_time(ev[i + 1]), 4)
    # isolate the real-space kernel (cell sort already cached now)
    ev[0].record(stream)
    sess.pair_count(reset=True)
    ev[0].record(stream)
    sess.evaluate(u, rank, ws, 2)
    ev[1].record(stream)
    torch.cuda.synchronize()
    rs_ms = ev[0].elapsed_time(ev[1])
    rs_pairs = sess.pair_count(reset=True)
    ev[0].record(stream)
    sess.spread(i0, i1, grid)
    ev[1].record(stream)
    sess.evaluate(u, rank, ws, 1)
    ev[2].record(stream)
    torch.cuda.synchronize()
    spread_ms = ev[0].elapsed_time(ev[1])
    gather_ms = ev[1].elapsed_time(ev[2])
    stages["realspace_kernel"] = round(rs_ms, 4)
    stages["spread_kernel"] = round(spread_ms, 4)
    stages["gather(+terms)_kernel"] = round(gather_ms, 4)

    line = None
    if rank == 0:
        peak64 = engine.fp64_peak_tflops()
        import json as _j
        mp = {}
        try:
            mp = _j.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        hbm_peak = mp.get("hbm_gbs", 6650.0)
        fl = FLOPS_PER_PAIR[(int(cfg.kind), bool(same and S.get_kernel_option(S.KernelOption.RS_SYM) != 0))]
        achieved = rs_pairs * fl / (rs_ms * 1e-3) / 1e12
        C = 9 if cfg.kind == S.Kernel.stresslet else 3
        vol = int(np.prod(params.grid.M_ext))
        spread_bytes = 8 * (3 + (6 if C == 9 else 3)) * N + 8 * C * vol
        gather_bytes = 8 * 6 * Nt + 8 * 3 * vol
        line = {
            "metric": "targets/sec", "value": value, "unit": "targets/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded uniform positions, N(0,1) strengths; BASELINE config)",
            "config": config_dict(cfg.name, N, Nt, cfg.kind, cfg.d, cfg.xi, cfg.tol, params.grid.M_ext,
                                  params.window.P, params.window.kind, params.rc, ws),
            "roofline": {"kernel": "realspace", "bound": "fp64", "achieved": achieved, "peak": peak64,
                         "unit": "TFLOP/s", "frac": achieved / peak64,
                         "peak_source": "measured DFMA microbenchmark (sewald_gpu_fp64_peak)",
                         "traffic": TRAFFIC_BYTES.get(cfg.name), "traffic_unit": "bytes/launch (ncu dram read+write)",
                         "pairs_per_launch": rs_pairs, "flops_per_pair": fl,
                         "kernel_ms": rs_ms},
            "stages_ms": stages,
            "spread_gather": {"spread_GBps": spread_bytes / (spread_ms * 1e-3) / 1e9,
                              "gather_GBps": gather_bytes / (gather_ms * 1e-3) / 1e9,
                              "hbm_peak_GBps": hbm_peak,
                              "spread_frac_hbm": spread_bytes / (spread_ms * 1e-3) / 1e9 / hbm_peak,
                              "gather_frac_hbm": gather_bytes / (gather_ms * 1e-3) / 1e9 / hbm_peak,
                              "spread_fp64_frac": 2 * C * params.window.P ** 3 * N / (spread_ms * 1e-3) / 1e12 / peak64,
                              "gather_fp64_frac": 2 * 3 * params.window.P ** 3 * Nt / (gather_ms * 1e-3) / 1e12 / peak64},
            "pairs_per_step": pairs,
            "gpu_launches": int(launches),
            "clocks": clocks,
        }

    # parity of the device-resident result against the reference's own run
    if rank == 0 and line is not None:
        torch.cuda.synchronize()
        line["parity_vs_fixture"] = fixture_parity(u_step, cfg.index, args.xi is not None)
        if ws == 1 and cfg.index in BALANCED_XI and args.xi is None and not args.no_balanced:
            try:  # supplementary: never costs the headline line
                line["balanced_xi"] = balanced_probe(S, cfg, x, f, nu, xt, engine, stream, dev, l2)
            except Exception as ex:  # pragma: no cover - reported, not fatal
                line["balanced_xi"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}

    # end-to-end through the public API with pinned host buffers: full_potential
    # on 1 GPU, parallel.full_potential_sharded on N (max over ranks)
    if not args.no_e2e:
        from paper_2210_01255_b200.parallel import full_potential_sharded
        pin = lambda a: torch.from_numpy(a).pin_memory().numpy() if a is not None else None
        px, pf, pnu = pin(x), pin(f), pin(nu)
        pxt = pin(xt)
        psys = S.SourceSystem(cfg.kind, S.Cell(cfg.L), cfg.d, px, pf, pnu)
        ptg = S.TargetSet.from_sources(psys) if same else S.TargetSet(pxt, False)
        pout = torch.empty((Nt, 3), dtype=torch.float64).pin_memory().numpy()
        if ws == 1:
            eng2 = S.default_engine(local)
            call = lambda: S.full_potential(psys, ptg, params, engine=eng2, out=pout)
            api = "paper_2210_01255_b200.full_potential (pinned host numpy in/out)"
        else:
            call = lambda: full_potential_sharded(psys, ptg, params, rank, ws, dist=dist, engine=engine, out=pout)
            api = "paper_2210_01255_b200.parallel.full_potential_sharded (pinned host numpy in, rank 0 out)"
        call()  # warm (plans, buffers)
        ts = []
        for _ in range(max(1, min(args.steps, 5))):
            barrier()
            t0 = time.perf_counter()
            uo = call()
            torch.cuda.synchronize()
            dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
            if ws > 1:
                dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            ts.append(float(dt.item()))
        e2e_s = float(np.median(ts))
        h2d = x.nbytes + f.nbytes + (nu.nbytes if nu is not None else 0) + (xt.nbytes if xt is not None else 0)
        if rank == 0:
            line["e2e"] = {"value": Nt / e2e_s, "unit": "targets/s", "h2d_bytes_per_step": int(h2d) * ws,
                           "d2h_bytes_per_step": int(pout.nbytes), "ms_per_call": e2e_s * 1e3,
                           "api": api, "timing": "host wall clock per call, max over ranks, median of calls"}
            par = fixture_parity(uo, cfg.index, args.xi is not None)
            if par is not None:
                line["e2e"]["parity_vs_fixture"] = par

    # the C++ drop-in path (sewald::full_potential, pageable std::vector in/out), config 2 only
    exe = os.path.join(ROOT, "paper_2210_01255_b200", "lib", "bench_dropin")
    if ws == 1 and rank == 0 and not args.no_e2e and cfg.index == 2 and os.path.exists(exe):
        try:
            r = subprocess.run([exe, str(N), str(max(1, min(args.steps, 5)))], capture_output=True, text=True,
                               timeout=600)
            line["e2e_cpp"] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as e:  # pragma: no cover
            line["e2e_cpp"] = {"unavailable": str(e)[:200]}

    if ws == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            v, det = cpu_reference_sample(cfg, params.to_c(), x, f, nu, xt, os.cpu_count() or 1, sample=10000)
            line["cpu_baseline"] = {
                "value": v, "unit": "targets/s", "cores": os.cpu_count() or 1, "kind": "reference",
                "cpu_model": cpu_model(), "modelled": True,
                "sample": ("reference C++ (oracle/_ref) per-unit costs on 10000 sampled sources/targets of this "
                           "workload, fixed costs removed; T = T_fixed + N t_spread + Nt t_gather + Nt t_realspace "
                           "(real space on all cores). bench.py --impl reference measures the whole run."),
                "detail": det}
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unit": "targets/s", "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line))
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def relaunch_distributed(n: int) -> int:
    """`--gpus N` outside torchrun: run this script under torch.distributed.run
    with N ranks on this node (rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args.gpus))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus and int(os.environ.get("RANK", "0")) == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; using {ws} ranks", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, args.config)
    else:
        from paper_2210_01255_b200.workloads import CONFIGS
        cfg = CONFIGS[args.config]
        if args.xi is not None:
            import dataclasses
            cfg = dataclasses.replace(cfg, xi=float(args.xi), name=f"{cfg.name}_xi{args.xi:g}")
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
