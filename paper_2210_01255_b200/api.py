"""Python mirror of the reference's host API for the Spectral Ewald hot path.

Same names, argument meaning and error behaviour as the reference C++
library (/root/reference/proj/include/sewald/*.h); every numeric call goes
through the C-ABI (include/sewald_gpu.h) into sm_100a kernels.

    estimates.h:106-107  select_parameters(kind, d, cell, Q, xi, tol, opt)
    realspace.h:46-47    full_potential(system, targets, params, opt)
    fourier.h:81-82      se_fourier_potential(system, targets, params, opt)
    realspace.h:40-41    realspace_potential(system, targets, xi, rc, starred, n_threads)
    fourier.h:59, 71-72  spread(system, params) / gather(field, params, targets)
    domain.h:78-79       source_quantity(system)

Exceptions: InvalidArgument (std::invalid_argument), DomainError
(std::domain_error), SewaldRuntimeError (std::runtime_error).
"""
from __future__ import annotations

import contextlib
import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _abi
from ._abi import (DomainError, InvalidArgument, SewaldError, SewaldRuntimeError, DeviceError,
                   sewald_params_c, sewald_report_c, sewald_timings_c)


class Kernel(enum.IntEnum):
    """enum class Kernel (domain.h:26)."""
    stokeslet = _abi.STOKESLET
    stresslet = _abi.STRESSLET
    rotlet = _abi.ROTLET


class WindowKind(enum.IntEnum):
    """enum class WindowKind (window.h:9)."""
    kb = _abi.WIN_KB
    pkb = _abi.WIN_PKB
    tg = _abi.WIN_TG


def strength_components(kind: Kernel) -> int:
    """domain.h:34 — 9 for the stresslet outer product, else 3."""
    return 9 if Kernel(kind) == Kernel.stresslet else 3


@dataclass
class Cell:
    """struct Cell (domain.h:36-39)."""
    L: Sequence[float] = (1.0, 1.0, 1.0)

    def volume(self) -> float:
        return float(self.L[0]) * float(self.L[1]) * float(self.L[2])


def _vec3(a, name: str) -> np.ndarray:
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if arr.size == 0:
        return arr.reshape(0, 3)
    if arr.ndim != 2 or arr.shape[1] != 3:
        raise InvalidArgument(f"{name} must have shape (n, 3)")
    return arr


@dataclass
class SourceSystem:
    """struct SourceSystem (domain.h:47-56): AoS positions and strengths."""
    kind: Kernel = Kernel.stokeslet
    cell: Cell = field(default_factory=Cell)
    d: int = 3
    x: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    f: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    nu: Optional[np.ndarray] = None

    def size(self) -> int:
        return int(np.asarray(self.x).shape[0])


@dataclass
class TargetSet:
    """struct TargetSet (domain.h:58-64)."""
    x: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    same_as_sources: bool = False

    @staticmethod
    def from_sources(s: SourceSystem) -> "TargetSet":
        return TargetSet(np.asarray(s.x), True)


@dataclass
class ToleranceSpec:
    """struct ToleranceSpec (estimates.h:13-18)."""
    value: float = 1e-8
    relative: bool = False


@dataclass
class SelectionOptions:
    """struct SelectionOptions (estimates.h:92-96)."""
    f_m: int = 4
    window: WindowKind = WindowKind.pkb
    pollution_fix: bool = True


@dataclass
class SePipelineOptions:
    """struct SePipelineOptions (fourier.h:76-79). Without `table` the device
    session builds the D=0 kernel table once per parameter set and keeps it;
    a caller-built `table` (precompute_0p) is used instead."""
    precompute_0p: bool = True
    table: Optional["PrecomputedKernel0P"] = None


@dataclass
class GridSpec:
    """struct GridSpec (grid.h:13-24)."""
    d: int = 3
    h: float = 0.0
    M: Sequence[int] = (0, 0, 0)
    M_ext: Sequence[int] = (0, 0, 0)
    L: Sequence[float] = (0.0, 0.0, 0.0)
    L_ext: Sequence[float] = (0.0, 0.0, 0.0)
    pad: Sequence[float] = (0.0, 0.0, 0.0)
    f_m: int = 4


@dataclass
class WindowSpec:
    """struct WindowSpec (window.h:15-29)."""
    kind: WindowKind = WindowKind.pkb
    P: int = 8
    h: float = 1.0
    beta: float = 20.0
    nu: int = 6
    alpha: float = 0.0

    @staticmethod
    def make(kind: WindowKind, P: int, h: float) -> "WindowSpec":
        """WindowSpec::make (window.cpp:76-86), computed by the C-ABI."""
        c = sewald_params_c()
        _host_call(_abi.load().sewald_window_make(int(kind), int(P), float(h), C.byref(c)))
        return WindowSpec(WindowKind(c.win_kind), c.P, c.win_h, c.beta, c.nu, c.alpha)


@dataclass
class UpsamplingPlan:
    """struct UpsamplingPlan (grid.h:29-35)."""
    s0: float = 1.0
    s_star: float = 1.0
    k_star: Sequence[int] = (0, 0, 0)
    s0_raw: float = 1.0
    s_star_raw: float = 1.0


@dataclass
class EwaldParams:
    """struct EwaldParams (estimates.h:62-71)."""
    kind: Kernel = Kernel.stokeslet
    d: int = 3
    xi: float = 1.0
    rc: float = 0.0
    R: float = 0.0
    grid: GridSpec = field(default_factory=GridSpec)
    window: WindowSpec = field(default_factory=WindowSpec)
    upsampling: UpsamplingPlan = field(default_factory=UpsamplingPlan)

    def to_c(self) -> sewald_params_c:
        c = sewald_params_c()
        c.kind, c.d = int(self.kind), int(self.d)
        c.xi, c.rc, c.R = float(self.xi), float(self.rc), float(self.R)
        g = self.grid
        c.h = float(g.h)
        for i in range(3):
            c.M[i], c.M_ext[i] = int(g.M[i]), int(g.M_ext[i])
            c.L[i], c.L_ext[i], c.pad[i] = float(g.L[i]), float(g.L_ext[i]), float(g.pad[i])
            c.k_star[i] = int(self.upsampling.k_star[i])
        c.f_m = int(g.f_m)
        w = self.window
        c.win_kind, c.P, c.win_h = int(w.kind), int(w.P), float(w.h)
        c.beta, c.nu, c.alpha = float(w.beta), int(w.nu), float(w.alpha)
        u = self.upsampling
        c.s0, c.s_star, c.s0_raw, c.s_star_raw = float(u.s0), float(u.s_star), float(u.s0_raw), float(u.s_star_raw)
        return c

    @staticmethod
    def from_c(c: sewald_params_c) -> "EwaldParams":
        g = GridSpec(c.d, c.h, tuple(c.M), tuple(c.M_ext), tuple(c.L), tuple(c.L_ext), tuple(c.pad), c.f_m)
        w = WindowSpec(WindowKind(c.win_kind), c.P, c.win_h, c.beta, c.nu, c.alpha)
        u = UpsamplingPlan(c.s0, c.s_star, tuple(c.k_star), c.s0_raw, c.s_star_raw)
        return EwaldParams(Kernel(c.kind), c.d, c.xi, c.rc, c.R, g, w, u)


@dataclass
class EstimateReport:
    """struct EstimateReport (estimates.h:73-90)."""
    tau_abs: float = 0.0
    U: float = 0.0
    kinf: float = 0.0
    fourier_trunc: float = 0.0
    realspace_trunc: float = 0.0
    window_err: float = 0.0
    h_estimate: float = 0.0
    P_estimate: int = 0
    h_target: float = 0.0
    P_target: int = 0
    rc_clamped: bool = False
    kinf_clamped: bool = False
    window_saturated: bool = False
    tg_support_from_pkb: bool = False


@dataclass
class ParameterSelection:
    params: EwaldParams
    report: EstimateReport


def _host_call(code: int):
    if code != _abi.OK:
        _abi.raise_for(code, _abi.load().sewald_last_error().decode())


def _dp(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(_abi.DP)


def select_parameters(kind: Kernel, d: int, cell: Cell, Q: float, xi: float,
                      tol: ToleranceSpec = ToleranceSpec(),
                      opt: SelectionOptions = SelectionOptions()) -> ParameterSelection:
    """select_parameters (estimates.h:106-107, estimates.cpp:211-268)."""
    lib = _abi.load()
    c, r = sewald_params_c(), sewald_report_c()
    L = (C.c_double * 3)(*[float(v) for v in cell.L])
    _host_call(lib.sewald_select_parameters(int(kind), int(d), L, float(Q), float(xi), float(tol.value),
                                            int(bool(tol.relative)), int(opt.f_m), int(opt.window),
                                            int(bool(opt.pollution_fix)), C.byref(c), C.byref(r)))
    rep = EstimateReport(r.tau_abs, r.U, r.kinf, r.fourier_trunc, r.realspace_trunc, r.window_err,
                         r.h_estimate, r.P_estimate, r.h_target, r.P_target, bool(r.rc_clamped),
                         bool(r.kinf_clamped), bool(r.window_saturated), bool(r.tg_support_from_pkb))
    return ParameterSelection(EwaldParams.from_c(c), rep)


def build_grid(cell: Cell, d: int, h_target: float, P: int, kind: Kernel, f_m: int) -> GridSpec:
    """build_grid (grid.h:38, grid.cpp:35-77)."""
    c = sewald_params_c()
    L = (C.c_double * 3)(*[float(v) for v in cell.L])
    _host_call(_abi.load().sewald_build_grid(L, int(d), float(h_target), int(P), int(kind), int(f_m), C.byref(c)))
    return EwaldParams.from_c(c).grid


def pkb_coefficients(window: WindowSpec) -> np.ndarray:
    """pkb_build (window.cpp:112-138): (P, nu+1) monomial coefficients."""
    p = EwaldParams(window=window).to_c()
    out = np.zeros((window.P, window.nu + 1))
    _host_call(_abi.load().sewald_pkb_coefficients(C.byref(p), _dp(out)))
    return out


def window_eval(window: WindowSpec, r) -> np.ndarray:
    """Window::eval1d (window.cpp:171-178) on the host."""
    r = np.ascontiguousarray(np.asarray(r, dtype=np.float64).ravel())
    out = np.zeros_like(r)
    p = EwaldParams(window=window).to_c()
    _host_call(_abi.load().sewald_window_eval(C.byref(p), _dp(r), r.size, _dp(out)))
    return out


def window_hat(window: WindowSpec, k) -> np.ndarray:
    """Window::hat1d (window.cpp:180-182) on the host."""
    k = np.ascontiguousarray(np.asarray(k, dtype=np.float64).ravel())
    out = np.zeros_like(k)
    p = EwaldParams(window=window).to_c()
    _host_call(_abi.load().sewald_window_hat(C.byref(p), _dp(k), k.size, _dp(out)))
    return out


def source_quantity(system: SourceSystem) -> float:
    """source_quantity (domain.cpp:53-62)."""
    f = _vec3(system.f, "f")
    nu = _vec3(system.nu, "nu") if Kernel(system.kind) == Kernel.stresslet else None
    return float(_abi.load().sewald_source_quantity(int(system.kind), _dp(f), _dp(nu), f.shape[0]))


# ---------------------------------------------------------------------------
# device engine
# ---------------------------------------------------------------------------


class KernelOption(enum.IntEnum):
    """Kernel-choice switches (include/sewald_gpu.h SEWALD_OPT_*): defaults
    are the measured best; tests set them to pin every kernel family."""
    RS_SYM = 0          # 0 never pair-symmetric, 1 auto, 2 always (targets == sources)
    GATHER = 1          # -1 auto, 0 warp per target, 1 z-sweep, 2 tiles
    GATHER_MMA = 2      # tiled gather: 1 tensor-core form, 0 CUDA-core form
    GATHER_L = 3        # tiled gather region edge: 0 auto, 15, 19
    SPREAD_SWEEP = 4    # -1 auto, 0 off, 1 on
    SPREAD_MMA = 5      # 1 tensor-core spread (15 <= P <= 32), 0 off
    SPREAD_MMA_L = 6    # 23 or 19
    SPREAD_CACHED = 7   # 1 staged tables per chunk, 0 per group
    SPREAD_ROWSWEEP = 8  # 1 row-sweep tensor-core spread CTAs for P <= 20
    SPREAD_FUSED = 9    # 1 tensor-core spread tiles evaluate their taps in the kernel
    GATHER_WIDE = 10    # register-A gather tiles: 2 every width, 1 only 20 < P <= 32, 0 never
    GATHER_FUSED = 11   # register-A gather tiles evaluate their taps in the kernel
    SPREAD_SORT = 12    # tensor-core spread tiles: points ordered by (x, y) offset, unreachable MMA steps skipped
    GATHER_SORT = 13    # register-A gather tiles: the same for targets
    D0_YFUSED = 14      # D = 0 solve: fused y transform + scale + inverse y transform (read at plan build)


def get_kernel_option(which: KernelOption) -> int:
    v = C.c_int()
    _abi.raise_for(_abi.load().sewald_gpu_get_option(int(which), C.byref(v)), f"unknown option {which}")
    return v.value


def set_kernel_option(which: KernelOption, value: int) -> None:
    code = _abi.load().sewald_gpu_set_option(int(which), int(value))
    _abi.raise_for(code, f"bad value {value} for option {KernelOption(which).name}")


@contextlib.contextmanager
def kernel_options(**kw):
    """with kernel_options(RS_SYM=2, GATHER=1): ... — set, then restore."""
    old = {k: get_kernel_option(KernelOption[k]) for k in kw}
    try:
        for k, v in kw.items():
            set_kernel_option(KernelOption[k], v)
        yield
    finally:
        for k, v in old.items():
            set_kernel_option(KernelOption[k], v)


class Engine:
    """One device context (stream, cached cuFFT plans and resident buffers)."""

    def __init__(self, device: int = 0):
        self._lib = _abi.load()
        h = C.c_void_p()
        code = self._lib.sewald_gpu_create(int(device), C.byref(h))
        if code != _abi.OK:
            _abi.raise_for(code, f"sewald_gpu_create(device={device}) failed (no usable CUDA device?)")
        self.ctx = h
        self.device = device
        self._lock = threading.Lock()

    def close(self):
        if getattr(self, "ctx", None):
            self._lib.sewald_gpu_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, code: int):
        if code != _abi.OK:
            _abi.raise_for(code, self._lib.sewald_gpu_last_error(self.ctx).decode())

    def set_profiling(self, on: bool):
        self.check(self._lib.sewald_gpu_set_profiling(self.ctx, int(bool(on))))

    def set_stream(self, stream_ptr: int):
        self.check(self._lib.sewald_gpu_set_stream(self.ctx, C.c_void_p(stream_ptr)))

    def launch_count(self) -> int:
        return int(self._lib.sewald_gpu_launch_count(self.ctx))

    def fp64_peak_tflops(self) -> float:
        v = C.c_double()
        self.check(self._lib.sewald_gpu_fp64_peak(self.ctx, C.byref(v)))
        return float(v.value)

    def timings(self) -> dict:
        t = sewald_timings_c()
        self.check(self._lib.sewald_gpu_get_timings(self.ctx, C.byref(t)))
        return {n: getattr(t, n) for n, _ in sewald_timings_c._fields_}


_engines: dict = {}
_elock = threading.Lock()


class MultiEngine:
    """Several GPUs of this node driven from one process (sewald_gpu_multi_*):
    sources spread in 1/W slices, grids summed over NVLink peer memory, each
    GPU evaluates 1/W of the targets. `devices` may repeat a device (tests on
    one GPU). full_potential / se_fourier_potential take the same arguments as
    the module functions."""

    def __init__(self, devices: Sequence[int]):
        self._lib = _abi.load()
        devs = [int(d) for d in devices]
        if not devs:
            raise InvalidArgument("at least one device")
        arr = (C.c_int * len(devs))(*devs)
        h = C.c_void_p()
        code = self._lib.sewald_gpu_multi_create(len(devs), arr, C.byref(h))
        if code != _abi.OK:
            _abi.raise_for(code, f"sewald_gpu_multi_create({devs}) failed (devices or peer access unavailable)")
        self.m = h
        self.devices = devs
        self._lock = threading.Lock()

    def close(self):
        if getattr(self, "m", None):
            self._lib.sewald_gpu_multi_destroy(self.m)
            self.m = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _run(self, entry, system, targets, params, opt, out):
        x, f, nu = _system_arrays(system, params)
        if not (float(params.xi) > 0.0):
            raise InvalidArgument("xi must be positive")
        same = bool(targets.same_as_sources)
        xt = x if same else _vec3(targets.x, "targets")
        nt = xt.shape[0]
        u = _out_array(out, nt)
        c = _params_for(system, params)
        with self._lock:
            if int(params.d) == 0 and opt.precompute_0p:
                tab = opt.table
                for d in range(len(self.devices)):
                    ctx = self._lib.sewald_gpu_multi_context(self.m, d)
                    if tab is None:
                        code = self._lib.sewald_gpu_set_table0p(ctx, C.byref(c), None, None)
                    else:
                        tb = np.ascontiguousarray(np.asarray(tab.table, dtype=np.complex128).ravel())
                        tn = (C.c_int32 * 3)(*[int(v) for v in tab.n])
                        code = self._lib.sewald_gpu_set_table0p(ctx, C.byref(c), tn, _cdp(tb))
                    _abi.raise_for(code, self._lib.sewald_gpu_last_error(ctx).decode())
            code = getattr(self._lib, entry)(self.m, C.byref(c), _dp(x), _dp(f), _dp(nu), x.shape[0], _dp(xt), nt,
                                             int(same), int(bool(opt.precompute_0p)), _dp(u))
            _abi.raise_for(code, self._lib.sewald_gpu_multi_last_error(self.m).decode())
        return u

    def full_potential(self, system, targets, params, opt=None, out=None):
        return self._run("sewald_gpu_multi_full_potential", system, targets, params, opt or SePipelineOptions(), out)

    def se_fourier_potential(self, system, targets, params, opt=None, out=None):
        return self._run("sewald_gpu_multi_fourier_potential", system, targets, params, opt or SePipelineOptions(),
                         out)


def default_engine(device: int = 0) -> Engine:
    with _elock:
        e = _engines.get(device)
        if e is None:
            e = Engine(device)
            _engines[device] = e
        return e


def _system_arrays(system: SourceSystem, params: Optional[EwaldParams] = None):
    kind = Kernel(system.kind)
    if params is not None and (kind != Kernel(params.kind) or int(system.d) != int(params.d)):
        raise InvalidArgument("parameter set was built for a different system")
    x = _vec3(system.x, "x")
    f = _vec3(system.f, "f")
    if f.shape[0] != x.shape[0]:
        raise InvalidArgument("strength count does not match position count")
    nu = None
    if kind == Kernel.stresslet:
        nu = _vec3(system.nu if system.nu is not None else np.zeros((0, 3)), "nu")
        if nu.shape[0] != x.shape[0]:
            raise InvalidArgument("stresslet needs one orientation per source")
    elif system.nu is not None and np.asarray(system.nu).size:
        raise InvalidArgument("orientations only apply to the stresslet")
    if not (0 <= int(system.d) <= 3):
        raise InvalidArgument("periodicity d must be in 0..3")
    if any(not (float(v) > 0.0) for v in system.cell.L):
        raise InvalidArgument("cell lengths must be positive")
    # non-finite positions are rejected on the device (finite_check_kernel,
    # InvalidArgument "non-finite source position"), not by a host pass
    return x, f, nu


def _params_for(system: SourceSystem, params: EwaldParams) -> sewald_params_c:
    c = params.to_c()
    for i in range(3):
        c.L[i] = float(system.cell.L[i])
    return c


def _out_array(out, nt: int) -> np.ndarray:
    if out is None:
        return np.empty((nt, 3))
    if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.shape == (nt, 3)
            and out.flags.c_contiguous and out.flags.writeable):
        raise InvalidArgument("out must be a writeable C-contiguous float64 array of shape (n_targets, 3)")
    return out


def _pipeline(entry: str, system: SourceSystem, targets: TargetSet, params: EwaldParams,
              opt: SePipelineOptions, engine: Optional[Engine], out=None) -> np.ndarray:
    x, f, nu = _system_arrays(system, params)
    if not (float(params.xi) > 0.0):
        raise InvalidArgument("xi must be positive")
    same = bool(targets.same_as_sources)
    xt = x if same else _vec3(targets.x, "targets")
    nt = xt.shape[0]
    u = _out_array(out, nt)
    eng = engine or default_engine()
    c = _params_for(system, params)
    tab = opt.table
    if tab is not None and Kernel(tab.kind) != Kernel(params.kind):
        raise InvalidArgument("kernel table was built for a different kernel")
    with eng._lock:
        if int(params.d) == 0 and opt.precompute_0p:
            if tab is None:
                eng.check(eng._lib.sewald_gpu_set_table0p(eng.ctx, C.byref(c), None, None))
            else:
                tb = np.ascontiguousarray(np.asarray(tab.table, dtype=np.complex128).ravel())
                if tb.size != int(np.prod(tab.n)):
                    raise InvalidArgument("kernel table storage is inconsistent")
                tn = (C.c_int32 * 3)(*[int(v) for v in tab.n])
                eng.check(eng._lib.sewald_gpu_set_table0p(eng.ctx, C.byref(c), tn, _cdp(tb)))
        fn = getattr(eng._lib, entry)
        eng.check(fn(eng.ctx, C.byref(c), _dp(x), _dp(f), _dp(nu), x.shape[0], _dp(xt), nt,
                     int(same), int(bool(opt.precompute_0p)), _dp(u)))
    return u


def full_potential(system: SourceSystem, targets: TargetSet, params: EwaldParams,
                   opt: SePipelineOptions = SePipelineOptions(), engine: Optional[Engine] = None,
                   out: Optional[np.ndarray] = None) -> np.ndarray:
    """full_potential (realspace.h:46-47): u_R + u_F + self + zero-mode terms, (Nt, 3).
    `out` (optional, e.g. pinned host memory) receives the result and is returned."""
    return _pipeline("sewald_gpu_full_potential", system, targets, params, opt, engine, out)


def se_fourier_potential(system: SourceSystem, targets: TargetSet, params: EwaldParams,
                         opt: SePipelineOptions = SePipelineOptions(),
                         engine: Optional[Engine] = None, out: Optional[np.ndarray] = None) -> np.ndarray:
    """se_fourier_potential (fourier.h:81-82)."""
    return _pipeline("sewald_gpu_fourier_potential", system, targets, params, opt, engine, out)


def realspace_potential(system: SourceSystem, targets: TargetSet, xi: float, rc: float,
                        starred: bool, n_threads: int = 1, engine: Optional[Engine] = None) -> np.ndarray:
    """realspace_potential (realspace.h:40-41). n_threads is accepted for API
    compatibility; the sum always runs on the GPU."""
    del n_threads
    if not (float(xi) > 0.0):
        raise InvalidArgument("split parameter must be positive")
    x, f, nu = _system_arrays(system)
    same = bool(targets.same_as_sources)
    xt = x if same else _vec3(targets.x, "targets")
    if xt.size and not np.all(np.isfinite(xt)):
        raise InvalidArgument("target coordinates must be finite")
    if not (float(rc) > 0.0):
        raise InvalidArgument("cell list cutoff must be positive")
    u = np.zeros((xt.shape[0], 3))
    eng = engine or default_engine()
    L = (C.c_double * 3)(*[float(v) for v in system.cell.L])
    with eng._lock:
        eng.check(eng._lib.sewald_gpu_realspace_potential(
            eng.ctx, int(system.kind), int(system.d), L, _dp(x), _dp(f), _dp(nu), x.shape[0], _dp(xt),
            xt.shape[0], int(same), float(xi), float(rc), int(bool(starred)), _dp(u)))
    return u


def spread(system: SourceSystem, params: EwaldParams, engine: Optional[Engine] = None) -> np.ndarray:
    """spread (fourier.h:59): RealField values, shape (C, n0, n1, n2)."""
    x, f, nu = _system_arrays(system)
    if int(system.d) != int(params.d):
        raise InvalidArgument("system and grid periodicity differ")
    n = tuple(int(v) for v in params.grid.M_ext)
    Cc = strength_components(system.kind)
    out = np.zeros((Cc,) + n)
    eng = engine or default_engine()
    c = params.to_c()
    c.kind = int(system.kind)
    with eng._lock:
        eng.check(eng._lib.sewald_gpu_spread(eng.ctx, C.byref(c), _dp(x), _dp(f), _dp(nu), x.shape[0], _dp(out)))
    return out


def gather(field: np.ndarray, params: EwaldParams, targets: TargetSet,
           engine: Optional[Engine] = None) -> np.ndarray:
    """gather (fourier.h:71-72): field shape (3, n0, n1, n2) -> (Nt, 3)."""
    fld = np.ascontiguousarray(np.asarray(field, dtype=np.float64))
    n = tuple(int(v) for v in params.grid.M_ext)
    if fld.shape != (3,) + n:
        raise InvalidArgument("gather expects a 3-component field on the extended grid")
    xt = _vec3(targets.x, "targets")
    u = np.zeros((xt.shape[0], 3))
    eng = engine or default_engine()
    c = params.to_c()
    with eng._lock:
        eng.check(eng._lib.sewald_gpu_gather(eng.ctx, C.byref(c), _dp(fld), _dp(xt), xt.shape[0], _dp(u)))
    return u


# ---------------------------------------------------------------------------
# reference stage functions (fourier.h:30-74)
# ---------------------------------------------------------------------------


@dataclass
class ModifiedKernelSpec:
    """struct ModifiedKernelSpec (modified_kernels.h:10-21)."""
    kind: Kernel = Kernel.stokeslet
    d: int = 0
    R: float = 1.0
    a_B: float = 0.0
    b_B: float = 0.0
    ell_H: float = 1.0
    ell_B: float = 1.0
    c_B: float = 0.0

    @staticmethod
    def optimal(kind: Kernel, d: int, R: float) -> "ModifiedKernelSpec":
        """ModifiedKernelSpec::optimal (modified_kernels.cpp:52-63), via the C-ABI."""
        m = _abi.sewald_modspec_c()
        _host_call(_abi.load().sewald_modspec_optimal(int(kind), int(d), float(R), C.byref(m)))
        return ModifiedKernelSpec(Kernel(m.kind), m.d, m.R, m.a_B, m.b_B, m.ell_H, m.ell_B, m.c_B)

    def to_c(self):
        return _abi.sewald_modspec_c(int(self.kind), int(self.d), float(self.R), float(self.a_B), float(self.b_B),
                                     float(self.ell_H), float(self.ell_B), float(self.c_B))


@dataclass
class FourierField:
    """struct FourierField (fourier.h:35-46). far / near / zero are flat
    complex128 arrays in the reference's vector order; near_rows int32."""
    d: int = 3
    comps: int = 0
    n_per: Sequence[int] = (1, 1, 1)
    n_far: Sequence[int] = (1, 1, 1)
    n_near: Sequence[int] = (1, 1, 1)
    n_zero: Sequence[int] = (1, 1, 1)
    far: np.ndarray = field(default_factory=lambda: np.zeros(0, np.complex128))
    near_rows: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    near: np.ndarray = field(default_factory=lambda: np.zeros(0, np.complex128))
    zero: np.ndarray = field(default_factory=lambda: np.zeros(0, np.complex128))

    def geom(self):
        g = _abi.sewald_fourier_geom_c()
        g.d, g.comps = int(self.d), int(self.comps)
        for i in range(3):
            g.n_per[i], g.n_far[i] = int(self.n_per[i]), int(self.n_far[i])
            g.n_near[i], g.n_zero[i] = int(self.n_near[i]), int(self.n_zero[i])
        g.n_near_rows = int(np.asarray(self.near_rows).size)
        g.far_len, g.near_len, g.zero_len = (int(np.asarray(a).size) for a in (self.far, self.near, self.zero))
        return g


@dataclass
class PrecomputedKernel0P:
    """struct PrecomputedKernel0P (fourier.h:52-57)."""
    kind: Kernel = Kernel.stokeslet
    n: Sequence[int] = (0, 0, 0)
    R: float = 0.0
    table: np.ndarray = field(default_factory=lambda: np.zeros(0, np.complex128))


def _stage_params(grid: GridSpec, plan: Optional[UpsamplingPlan] = None,
                  window: Optional[WindowSpec] = None) -> sewald_params_c:
    return EwaldParams(d=int(grid.d), grid=grid, window=window if window is not None else WindowSpec(h=grid.h),
                       upsampling=plan if plan is not None else UpsamplingPlan()).to_c()


def _cplx_buf(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.complex128).ravel())
    return a


def _cdp(a: np.ndarray):
    return a.view(np.float64).ctypes.data_as(_abi.DP) if a.size else None


def _rows_ptr(rows: np.ndarray):
    return rows.ctypes.data_as(C.POINTER(C.c_int32)) if rows.size else None


def _empty_like_geom(g, comps: int):
    per = lambda n: np.zeros(n // max(g.comps, 1) * comps, np.complex128)  # noqa: E731
    return per(g.far_len), per(g.near_len), per(g.zero_len)


def aft_forward(rfield: np.ndarray, grid: GridSpec, plan: UpsamplingPlan,
                engine: Optional[Engine] = None) -> FourierField:
    """aft_forward (fourier.h:61, fourier.cpp:311-416): RealField values
    (comps, *M_ext) -> FourierField, transforms on the GPU."""
    fld = np.ascontiguousarray(np.asarray(rfield, dtype=np.float64))
    n = tuple(int(v) for v in grid.M_ext)
    if fld.ndim != 4 or fld.shape[1:] != n:
        raise InvalidArgument("field shape does not match the extended grid")
    comps = fld.shape[0]
    c = _stage_params(grid, plan)
    lib = _abi.load()
    g = _abi.sewald_fourier_geom_c()
    rows = np.zeros(max(1, int(np.prod([grid.M[i] for i in range(int(grid.d)) if i < 2] or [1]))), np.int32)
    _host_call(lib.sewald_aft_geometry(C.byref(c), comps, C.byref(g), _rows_ptr(rows)))
    far, near, zero = (np.zeros(k, np.complex128) for k in (g.far_len, g.near_len, g.zero_len))
    eng = engine or default_engine()
    with eng._lock:
        eng.check(lib.sewald_gpu_aft_forward(eng.ctx, C.byref(c), _dp(fld), C.byref(g), _cdp(far), _cdp(near),
                                             _cdp(zero)))
    return FourierField(g.d, g.comps, tuple(g.n_per), tuple(g.n_far), tuple(g.n_near), tuple(g.n_zero),
                        far, rows[:g.n_near_rows].copy(), near, zero)


def aft_inverse(F: FourierField, grid: GridSpec, plan: Optional[UpsamplingPlan] = None,
                engine: Optional[Engine] = None) -> np.ndarray:
    """aft_inverse (fourier.h:62, fourier.cpp:418-520): -> (comps, *M_ext)."""
    c = _stage_params(grid, plan)
    g = F.geom()
    far, near, zero = _cplx_buf(F.far), _cplx_buf(F.near), _cplx_buf(F.zero)
    rows = np.ascontiguousarray(F.near_rows, dtype=np.int32)
    out = np.zeros((int(F.comps),) + tuple(int(v) for v in grid.M_ext))
    eng = engine or default_engine()
    with eng._lock:
        eng.check(eng._lib.sewald_gpu_aft_inverse(eng.ctx, C.byref(c), C.byref(g), _rows_ptr(rows), _cdp(far),
                                                  _cdp(near), _cdp(zero), _dp(out)))
    return out


def scale(F: FourierField, spec, xi: float, window: WindowSpec, grid: GridSpec,
          engine: Optional[Engine] = None) -> FourierField:
    """scale (fourier.h:66-69, fourier.cpp:522-720): `spec` is a
    ModifiedKernelSpec or a PrecomputedKernel0P. Output has 3 components."""
    c = _stage_params(grid, None, window)
    g = F.geom()
    far, near, zero = _cplx_buf(F.far), _cplx_buf(F.near), _cplx_buf(F.zero)
    rows = np.ascontiguousarray(F.near_rows, dtype=np.int32)
    ofar, onear, ozero = _empty_like_geom(g, 3)
    eng = engine or default_engine()
    with eng._lock:
        if isinstance(spec, PrecomputedKernel0P):
            tn = (C.c_int32 * 3)(*[int(v) for v in spec.n])
            tab = _cplx_buf(spec.table)
            if tab.size != int(np.prod(spec.n)):
                raise InvalidArgument("kernel table storage is inconsistent")
            eng.check(eng._lib.sewald_gpu_scale_table(eng.ctx, C.byref(c), int(spec.kind), tn, _cdp(tab), float(xi),
                                                      C.byref(g), _cdp(zero), _cdp(ozero)))
        else:
            m = spec.to_c()
            eng.check(eng._lib.sewald_gpu_scale(eng.ctx, C.byref(c), C.byref(m), float(xi), C.byref(g),
                                                _rows_ptr(rows), _cdp(far), _cdp(near), _cdp(zero), _cdp(ofar),
                                                _cdp(onear), _cdp(ozero)))
    if isinstance(spec, PrecomputedKernel0P):  # fourier.cpp:688-692: only d, comps, n_zero carried over
        return FourierField(0, 3, n_zero=tuple(F.n_zero), zero=ozero)
    return FourierField(F.d, 3, tuple(F.n_per), tuple(F.n_far), tuple(F.n_near), tuple(F.n_zero),
                        ofar, rows.copy(), onear, ozero)


def precompute_0p(kind: Kernel, grid: GridSpec, R: float, engine: Optional[Engine] = None) -> PrecomputedKernel0P:
    """precompute_0p (fourier.h:74, fourier.cpp:722-803), built with cuFFT."""
    c = _stage_params(grid)
    n = (C.c_int32 * 3)()
    eng = engine or default_engine()
    with eng._lock:
        eng.check(eng._lib.sewald_gpu_precompute_0p(eng.ctx, C.byref(c), int(kind), float(R), n, None))
        tab = np.zeros(int(n[0]) * n[1] * n[2], np.complex128)
        eng.check(eng._lib.sewald_gpu_precompute_0p(eng.ctx, C.byref(c), int(kind), float(R), n, _cdp(tab)))
    return PrecomputedKernel0P(Kernel(kind), tuple(n), float(R), tab)


class Session:
    """Device-resident session (sewald_gpu_session_*): inputs and outputs are
    torch CUDA tensors; torch is used only for memory and streams. Every call
    runs on torch's current CUDA stream, so it is ordered with the caller's
    torch work (allocation, collectives) without extra synchronisation."""

    def __init__(self, params: EwaldParams, cell: Optional[Cell] = None, engine: Optional[Engine] = None):
        self.engine = engine or default_engine()
        self._lib = self.engine._lib
        self._sync_stream()
        c = params.to_c()
        if cell is not None:
            for i in range(3):
                c.L[i] = float(cell.L[i])
        h = C.c_void_p()
        self.engine.check(self._lib.sewald_gpu_session_create(self.engine.ctx, C.byref(c), C.byref(h)))
        self.s = h
        self._keep = []
        self._C = strength_components(Kernel(int(c.kind)))
        self._N = 0
        self._Nt = 0
        self._same = True

    def close(self):
        if getattr(self, "s", None):
            self._lib.sewald_gpu_session_destroy(self.s)
            self.s = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _sync_stream(self):
        import torch
        self.engine.set_stream(torch.cuda.current_stream().cuda_stream)

    def _ptr(self, t, name: str, doubles: Optional[int] = None, optional: bool = False):
        """Device pointer of a float64 (or complex128) CUDA tensor on this
        session's device holding exactly `doubles` doubles. The C-ABI reads
        and writes these buffers as double, so any other dtype, device, layout
        or size is refused here (InvalidArgument) instead of being
        reinterpreted or overrun on the device."""
        import torch
        if t is None:
            if optional:
                return None
            raise _abi.InvalidArgument(f"{name}: a tensor is required")
        if not isinstance(t, torch.Tensor):
            raise _abi.InvalidArgument(f"{name}: expected a torch CUDA tensor, got {type(t).__name__}")
        if t.dtype not in (torch.float64, torch.complex128):
            raise _abi.InvalidArgument(f"{name}: dtype must be torch.float64 (got {t.dtype})")
        if not t.is_cuda or (t.device.index if t.device.index is not None else 0) != self.engine.device:
            raise _abi.InvalidArgument(f"{name}: must live on cuda:{self.engine.device} (got {t.device})")
        if not t.is_contiguous():
            raise _abi.InvalidArgument(f"{name}: must be contiguous")
        n = t.numel() * (2 if t.dtype == torch.complex128 else 1)
        if doubles is not None and n != doubles:
            raise _abi.InvalidArgument(f"{name}: expected {doubles} doubles, got {n}")
        return C.c_void_p(t.data_ptr())

    @staticmethod
    def _rows(t, name: str) -> int:
        if t is None or t.dim() != 2 or t.shape[1] != 3:
            raise _abi.InvalidArgument(f"{name}: expected an (n, 3) tensor")
        return int(t.shape[0])

    def set_sources(self, x, f, nu=None):
        self._sync_stream()
        n = self._rows(x, "x")
        px = self._ptr(x, "x", 3 * n)
        pf = self._ptr(f, "f", 3 * n)
        pn = self._ptr(nu, "nu", 3 * n, optional=True)
        self._keep = [x, f, nu]
        self.engine.check(self._lib.sewald_gpu_session_set_sources(self.s, px, pf, pn, n))
        self._N = n
        if self._same:
            self._Nt = n

    def set_targets(self, xt=None, same_as_sources: bool = True):
        self._sync_stream()
        n = 0 if xt is None else self._rows(xt, "xt")
        p = None if xt is None else self._ptr(xt, "xt", 3 * n)
        self.engine.check(self._lib.sewald_gpu_session_set_targets(self.s, p, n, int(same_as_sources)))
        self._same = bool(same_as_sources)
        self._Nt = self._N if same_as_sources else n

    def grid_size(self) -> int:
        return int(self._lib.sewald_gpu_session_grid_size(self.s))

    def _flow_size(self) -> int:
        return 3 * self.grid_size() // self._C

    def spread(self, i0: int, i1: int, grid=None):
        self._sync_stream()
        g = self._ptr(grid, "grid", self.grid_size(), optional=True)
        self.engine.check(self._lib.sewald_gpu_session_spread(self.s, int(i0), int(i1), g))

    def solve(self, grid=None, precompute_0p: bool = True):
        self._sync_stream()
        g = self._ptr(grid, "grid", self.grid_size(), optional=True)
        self.engine.check(self._lib.sewald_gpu_session_solve(self.s, g, int(precompute_0p)))

    def evaluate(self, u, part: int = 0, nparts: int = 1, parts: int = 7):
        self._sync_stream()
        pu = self._ptr(u, "u", 3 * self._Nt)
        self.engine.check(self._lib.sewald_gpu_session_evaluate(self.s, int(part), int(nparts), int(parts), pu))

    # ---- slab-distributed D = 0 solve (parallel.d0_sharded_solve) ----------
    def d0_geometry(self, precompute_0p: bool = True) -> dict:
        """Padded-box geometry of the D = 0 real-transform solve: m (M_ext),
        n (transform box), h2 = n[2]//2 + 1, C (grid components)."""
        self._sync_stream()
        m, n = (C.c_int * 3)(), (C.c_int * 3)()
        h2, c = C.c_int(), C.c_int()
        self.engine.check(self._lib.sewald_gpu_session_d0_geometry(self.s, int(precompute_0p), m, n,
                                                                   C.byref(h2), C.byref(c)))
        return {"m": tuple(m), "n": tuple(n), "h2": h2.value, "C": c.value}

    @staticmethod
    def _bounds(b):
        arr = (C.c_int * len(b))(*[int(v) for v in b])
        return len(b) - 1, arr

    def d0_forward(self, grid_slab, xa: int, xb: int, kz_bounds, send, precompute_0p: bool = True):
        self._sync_stream()
        g = self.d0_geometry(precompute_0p)
        m, cc, h2 = g["m"], g["C"], g["h2"]
        w, arr = self._bounds(kz_bounds)
        pg = self._ptr(grid_slab, "grid_slab", cc * (xb - xa) * m[1] * m[2])
        ps = self._ptr(send, "send", 2 * cc * (xb - xa) * m[1] * h2)
        self.engine.check(self._lib.sewald_gpu_session_d0_forward(self.s, int(precompute_0p), pg, int(xa), int(xb),
                                                                  w, arr, ps))

    def d0_middle(self, recv, x_bounds, ka: int, kb: int, send, precompute_0p: bool = True):
        self._sync_stream()
        g = self.d0_geometry(precompute_0p)
        m, cc = g["m"], g["C"]
        w, arr = self._bounds(x_bounds)
        pr = self._ptr(recv, "recv", 2 * cc * m[0] * m[1] * (kb - ka))
        ps = self._ptr(send, "send", 2 * 3 * (kb - ka) * m[0] * m[1])
        self.engine.check(self._lib.sewald_gpu_session_d0_middle(self.s, int(precompute_0p), pr, w, arr, int(ka),
                                                                 int(kb), ps))

    def d0_inverse(self, recv, xa: int, xb: int, kz_bounds, flow_slab, precompute_0p: bool = True):
        self._sync_stream()
        g = self.d0_geometry(precompute_0p)
        m, h2 = g["m"], g["h2"]
        w, arr = self._bounds(kz_bounds)
        pr = self._ptr(recv, "recv", 2 * 3 * h2 * (xb - xa) * m[1])
        pf = self._ptr(flow_slab, "flow_slab", 3 * (xb - xa) * m[1] * m[2])
        self.engine.check(self._lib.sewald_gpu_session_d0_inverse(self.s, int(precompute_0p), pr, int(xa), int(xb),
                                                                  w, arr, pf))

    def set_flow(self, flow):
        self._sync_stream()
        self.engine.check(self._lib.sewald_gpu_session_set_flow(self.s, self._ptr(flow, "flow", self._flow_size())))

    def pair_count(self, reset: bool = False) -> int:
        return int(self._lib.sewald_gpu_session_pair_count(self.s, int(reset)))

    def run(self, u, precompute_0p: bool = True):
        self._sync_stream()
        pu = self._ptr(u, "u", 3 * self._Nt)
        self.engine.check(self._lib.sewald_gpu_session_run(self.s, int(precompute_0p), pu))
