"""ORACLE TEST INFRASTRUCTURE — not product code.

ctypes loader for oracle/_ref/libsewald_ref.so: the UNMODIFIED reference C++
library (/root/reference/proj/src/*.cpp) compiled by oracle/Makefile with the
committed FFTW/GSL shims, plus the extern "C" wrapper oracle/ref_capi.cpp.

Only tests/, __graft_entry__.smoke() and bench.py (reference arm and
cpu_baseline) may use this module, and only as the checker / CPU baseline.
The parameter struct layout mirrors include/sewald_gpu.h (declared again
here so the oracle does not import the product).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libsewald_ref.so")


class RefParams(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("d", C.c_int32),
        ("xi", C.c_double), ("rc", C.c_double), ("R", C.c_double),
        ("h", C.c_double), ("M", C.c_int32 * 3), ("M_ext", C.c_int32 * 3),
        ("L", C.c_double * 3), ("L_ext", C.c_double * 3), ("pad", C.c_double * 3),
        ("f_m", C.c_int32),
        ("win_kind", C.c_int32), ("P", C.c_int32), ("win_h", C.c_double),
        ("beta", C.c_double), ("nu", C.c_int32), ("alpha", C.c_double),
        ("s0", C.c_double), ("s_star", C.c_double), ("k_star", C.c_int32 * 3),
        ("s0_raw", C.c_double), ("s_star_raw", C.c_double),
    ]


class RefReport(C.Structure):
    _fields_ = [
        ("tau_abs", C.c_double), ("U", C.c_double), ("kinf", C.c_double),
        ("fourier_trunc", C.c_double), ("realspace_trunc", C.c_double),
        ("window_err", C.c_double), ("h_estimate", C.c_double),
        ("P_estimate", C.c_int32), ("h_target", C.c_double), ("P_target", C.c_int32),
        ("rc_clamped", C.c_int32), ("kinf_clamped", C.c_int32),
        ("window_saturated", C.c_int32), ("tg_support_from_pkb", C.c_int32),
    ]


DP = C.POINTER(C.c_double)
I64 = C.c_int64
PP = C.POINTER(RefParams)


class RefGeom(C.Structure):
    """sewald_fourier_geom_c (include/sewald_gpu.h) for the stage wrappers."""
    _fields_ = [("d", C.c_int32), ("comps", C.c_int32),
                ("n_per", C.c_int32 * 3), ("n_far", C.c_int32 * 3), ("n_near", C.c_int32 * 3),
                ("n_zero", C.c_int32 * 3), ("n_near_rows", C.c_int32),
                ("far_len", C.c_int64), ("near_len", C.c_int64), ("zero_len", C.c_int64)]


class RefModSpec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("d", C.c_int32), ("R", C.c_double), ("a_B", C.c_double),
                ("b_B", C.c_double), ("ell_H", C.c_double), ("ell_B", C.c_double), ("c_B", C.c_double)]


GP = C.POINTER(RefGeom)
IP32 = C.POINTER(C.c_int32)

_SIGS = {
    "ref_last_error": (C.c_char_p, []),
    "ref_last_seconds": (None, [DP]),
    "ref_select_parameters": (C.c_int, [C.c_int, C.c_int, DP, C.c_double, C.c_double, C.c_double, C.c_int,
                                        C.c_int, C.c_int, C.c_int, PP, C.POINTER(RefReport)]),
    "ref_pkb_coefficients": (C.c_int, [PP, DP]),
    "ref_window_eval": (C.c_int, [PP, DP, I64, DP]),
    "ref_window_hat": (C.c_int, [PP, DP, I64, DP]),
    "ref_build_grid": (C.c_int, [DP, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, PP]),
    "ref_spread": (C.c_int, [PP, DP, DP, DP, I64, DP]),
    "ref_gather": (C.c_int, [PP, DP, DP, I64, DP]),
    "ref_flow_field": (C.c_int, [PP, DP, DP, DP, I64, C.c_int, DP]),
    "ref_solve_grid": (C.c_int, [PP, DP, C.c_int, DP]),
    "ref_fourier_potential": (C.c_int, [PP, DP, DP, DP, I64, DP, I64, C.c_int, C.c_int, DP]),
    "ref_realspace_potential": (C.c_int, [C.c_int, C.c_int, DP, DP, DP, DP, I64, DP, I64, C.c_int,
                                          C.c_double, C.c_double, C.c_int, C.c_int, DP]),
    "ref_full_potential": (C.c_int, [PP, DP, DP, DP, I64, DP, I64, C.c_int, C.c_int, DP]),
    "ref_full_split": (C.c_int, [PP, DP, DP, DP, I64, DP, I64, C.c_int, C.c_int, C.c_int, DP]),
    "ref_full_parts": (C.c_int, [PP, DP, DP, DP, I64, DP, I64, C.c_int, C.c_int, C.c_int, DP, DP, DP]),
    "ref_precompute_0p": (C.c_int, [PP, DP, C.POINTER(C.c_int32)]),
    "ref_aft_forward": (C.c_int, [PP, DP, C.c_int, GP]),
    "ref_field_get": (C.c_int, [GP, IP32, DP, DP, DP]),
    "ref_field_set": (C.c_int, [GP, IP32, DP, DP, DP]),
    "ref_scale": (C.c_int, [PP, C.POINTER(RefModSpec), C.c_double, GP]),
    "ref_scale_table": (C.c_int, [PP, C.c_int, C.c_double, C.c_double, GP]),
    "ref_aft_inverse": (C.c_int, [PP, DP]),
    "ref_realspace_kernel": (C.c_int, [C.c_int, DP, C.c_double, DP]),
    "ref_modified_kernel_hat": (C.c_int, [C.c_int, C.c_int, C.c_double, DP, DP]),
}

_lib = None


class RefError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def available() -> bool:
    return os.path.exists(LIB_PATH)


def build(quiet: bool = True) -> bool:
    """Compile the reference (needs /root/reference; only in the builder container)."""
    if not os.path.isdir("/root/reference/proj"):
        return available()
    r = subprocess.run(["make", "-C", HERE, "-j8", "all"], capture_output=quiet, text=True)
    if r.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + (r.stdout or "") + (r.stderr or ""))
    return available()


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _chk(code):
    if code != 0:
        raise RefError(code, lib().ref_last_error().decode())


def _dp(a):
    return None if a is None else a.ctypes.data_as(DP)


def _v3(a):
    return None if a is None else np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1, 3))


def params_from(p) -> RefParams:
    """Copy any ctypes struct with the same field names into RefParams."""
    r = RefParams()
    for name, _ in RefParams._fields_:
        v = getattr(p, name)
        if hasattr(v, "__len__"):
            arr = getattr(r, name)
            for i in range(3):
                arr[i] = v[i]
        else:
            setattr(r, name, v)
    return r


def select_parameters(kind, d, L, Q, xi, tol=1e-8, relative=False, f_m=4, window=1, pollution_fix=True):
    p, rep = RefParams(), RefReport()
    Lc = (C.c_double * 3)(*[float(v) for v in L])
    _chk(lib().ref_select_parameters(int(kind), int(d), Lc, float(Q), float(xi), float(tol), int(relative),
                                     int(f_m), int(window), int(pollution_fix), C.byref(p), C.byref(rep)))
    return p, rep


def pkb_coefficients(p: RefParams) -> np.ndarray:
    out = np.zeros((p.P, p.nu + 1))
    _chk(lib().ref_pkb_coefficients(C.byref(p), _dp(out)))
    return out


def window_eval(p: RefParams, r) -> np.ndarray:
    r = np.ascontiguousarray(np.asarray(r, dtype=np.float64).ravel())
    out = np.zeros_like(r)
    _chk(lib().ref_window_eval(C.byref(p), _dp(r), r.size, _dp(out)))
    return out


def window_hat(p: RefParams, k) -> np.ndarray:
    k = np.ascontiguousarray(np.asarray(k, dtype=np.float64).ravel())
    out = np.zeros_like(k)
    _chk(lib().ref_window_hat(C.byref(p), _dp(k), k.size, _dp(out)))
    return out


def build_grid(L, d, h_target, P, kind, f_m) -> RefParams:
    p = RefParams()
    Lc = (C.c_double * 3)(*[float(v) for v in L])
    _chk(lib().ref_build_grid(Lc, int(d), float(h_target), int(P), int(kind), int(f_m), C.byref(p)))
    return p


def spread(p: RefParams, x, f, nu=None) -> np.ndarray:
    x, f, nu = _v3(x), _v3(f), _v3(nu)
    Cc = 9 if p.kind == 1 else 3
    out = np.zeros((Cc, p.M_ext[0], p.M_ext[1], p.M_ext[2]))
    _chk(lib().ref_spread(C.byref(p), _dp(x), _dp(f), _dp(nu), x.shape[0], _dp(out)))
    return out


def gather(p: RefParams, grid, xt) -> np.ndarray:
    grid = np.ascontiguousarray(grid, dtype=np.float64)
    xt = _v3(xt)
    out = np.zeros((xt.shape[0], 3))
    _chk(lib().ref_gather(C.byref(p), _dp(grid), _dp(xt), xt.shape[0], _dp(out)))
    return out


def flow_field(p: RefParams, x, f, nu=None, use_table=True) -> np.ndarray:
    x, f, nu = _v3(x), _v3(f), _v3(nu)
    out = np.zeros((3, p.M_ext[0], p.M_ext[1], p.M_ext[2]))
    _chk(lib().ref_flow_field(C.byref(p), _dp(x), _dp(f), _dp(nu), x.shape[0], int(use_table), _dp(out)))
    return out


def solve_grid(p: RefParams, grid, use_table=True) -> np.ndarray:
    grid = np.ascontiguousarray(grid, dtype=np.float64)
    out = np.zeros((3, p.M_ext[0], p.M_ext[1], p.M_ext[2]))
    _chk(lib().ref_solve_grid(C.byref(p), _dp(grid), int(use_table), _dp(out)))
    return out


def _targets(x, xt, same):
    if same:
        return None, x.shape[0]
    xt = _v3(xt)
    return xt, xt.shape[0]


def fourier_potential(p: RefParams, x, f, nu=None, xt=None, same=True, precompute_0p=True):
    x, f, nu = _v3(x), _v3(f), _v3(nu)
    xt, nt = _targets(x, xt, same)
    out = np.zeros((nt, 3))
    _chk(lib().ref_fourier_potential(C.byref(p), _dp(x), _dp(f), _dp(nu), x.shape[0], _dp(xt), nt,
                                      int(same), int(precompute_0p), _dp(out)))
    return out


def realspace_potential(kind, d, L, x, f, nu, xt, same, xi, rc, starred, n_threads=1):
    x, f, nu = _v3(x), _v3(f), _v3(nu)
    xt, nt = _targets(x, xt, same)
    out = np.zeros((nt, 3))
    Lc = (C.c_double * 3)(*[float(v) for v in L])
    _chk(lib().ref_realspace_potential(int(kind), int(d), Lc, _dp(x), _dp(f), _dp(nu), x.shape[0], _dp(xt),
                                       nt, int(same), float(xi), float(rc), int(starred), int(n_threads),
                                       _dp(out)))
    return out


def full_potential(p: RefParams, x, f, nu=None, xt=None, same=True, precompute_0p=True):
    x, f, nu = _v3(x), _v3(f), _v3(nu)
    xt, nt = _targets(x, xt, same)
    out = np.zeros((nt, 3))
    _chk(lib().ref_full_potential(C.byref(p), _dp(x), _dp(f), _dp(nu), x.shape[0], _dp(xt), nt, int(same),
                                  int(precompute_0p), _dp(out)))
    return out


def full_split(p: RefParams, x, f, nu=None, xt=None, same=True, precompute_0p=True, n_threads=1):
    """full_potential assembled as realspace.cpp:205-219 with n_threads on the
    real-space sum. Returns (u, seconds dict)."""
    x, f, nu = _v3(x), _v3(f), _v3(nu)
    xt, nt = _targets(x, xt, same)
    out = np.zeros((nt, 3))
    _chk(lib().ref_full_split(C.byref(p), _dp(x), _dp(f), _dp(nu), x.shape[0], _dp(xt), nt, int(same),
                              int(precompute_0p), int(n_threads), _dp(out)))
    secs = np.zeros(4)
    lib().ref_last_seconds(_dp(secs))
    return out, dict(fourier=secs[0], realspace=secs[1], terms=secs[2], total=secs[3])


def full_parts(p: RefParams, x, f, nu=None, xt=None, same=True, precompute_0p=True, n_threads=1):
    """As full_split, also returning the two sums it adds: (u, u_F, u_R, seconds)
    with u_F = se_fourier_potential (fourier.cpp:805-852) and u_R =
    realspace_potential (realspace.cpp:166-203), starred when same."""
    x, f, nu = _v3(x), _v3(f), _v3(nu)
    xt, nt = _targets(x, xt, same)
    out = np.zeros((nt, 3))
    uf = np.zeros((nt, 3))
    ur = np.zeros((nt, 3))
    _chk(lib().ref_full_parts(C.byref(p), _dp(x), _dp(f), _dp(nu), x.shape[0], _dp(xt), nt, int(same),
                              int(precompute_0p), int(n_threads), _dp(out), _dp(uf), _dp(ur)))
    secs = np.zeros(4)
    lib().ref_last_seconds(_dp(secs))
    return out, uf, ur, dict(fourier=secs[0], realspace=secs[1], terms=secs[2], total=secs[3])


def precompute_0p(p: RefParams) -> np.ndarray:
    n = (C.c_int32 * 3)()
    _chk(lib().ref_precompute_0p(C.byref(p), None, n))
    tab = np.zeros((n[0], n[1], n[2], 2))
    _chk(lib().ref_precompute_0p(C.byref(p), _dp(tab), n))
    return tab[..., 0] + 1j * tab[..., 1]


def realspace_kernel(kind, r, xi) -> np.ndarray:
    out = np.zeros(27)
    r = np.ascontiguousarray(np.asarray(r, dtype=np.float64))
    _chk(lib().ref_realspace_kernel(int(kind), _dp(r), float(xi), _dp(out)))
    return out[:9].reshape(3, 3) if kind != 1 else out.reshape(3, 3, 3)


def modified_kernel_hat(kind, d, R, k) -> np.ndarray:
    out = np.zeros(54)
    k = np.ascontiguousarray(np.asarray(k, dtype=np.float64))
    _chk(lib().ref_modified_kernel_hat(int(kind), int(d), float(R), _dp(k), _dp(out)))
    z = out[0::2] + 1j * out[1::2]
    return z[:9].reshape(3, 3) if kind != 1 else z.reshape(3, 3, 3)


# ---- stage functions (fourier.h:61-74), FourierField as a dict ----------------
# {"d", "comps", "n_per", "n_far", "n_near", "n_zero", "near_rows" (int32),
#  "far", "near", "zero" (complex128, flat as the reference's vectors)}

def _field_from_lib() -> dict:
    g = RefGeom()
    _chk(lib().ref_field_get(C.byref(g), None, None, None, None))
    rows = np.zeros(max(g.n_near_rows, 1), dtype=np.int32)
    arr = {k: np.zeros(2 * max(getattr(g, k + "_len"), 1)) for k in ("far", "near", "zero")}
    _chk(lib().ref_field_get(C.byref(g), rows.ctypes.data_as(IP32), _dp(arr["far"]), _dp(arr["near"]),
                             _dp(arr["zero"])))
    out = {"d": g.d, "comps": g.comps, "n_per": tuple(g.n_per), "n_far": tuple(g.n_far),
           "n_near": tuple(g.n_near), "n_zero": tuple(g.n_zero), "near_rows": rows[:g.n_near_rows].copy()}
    for k in ("far", "near", "zero"):
        n = getattr(g, k + "_len")
        out[k] = arr[k][0:2 * n:2] + 1j * arr[k][1:2 * n:2]
    return out


def _field_to_lib(F: dict):
    g = RefGeom()
    g.d, g.comps = F["d"], F["comps"]
    for i in range(3):
        g.n_per[i], g.n_far[i], g.n_near[i], g.n_zero[i] = F["n_per"][i], F["n_far"][i], F["n_near"][i], F["n_zero"][i]
    rows = np.ascontiguousarray(F["near_rows"], dtype=np.int32)
    g.n_near_rows = rows.size
    arrs = {}
    for k in ("far", "near", "zero"):
        a = np.ascontiguousarray(F[k], dtype=np.complex128)
        setattr(g, k + "_len", a.size)
        arrs[k] = a.view(np.float64) if a.size else np.zeros(1)
    _chk(lib().ref_field_set(C.byref(g), rows.ctypes.data_as(IP32) if rows.size else None, _dp(arrs["far"]),
                             _dp(arrs["near"]), _dp(arrs["zero"])))


def aft_forward(p: RefParams, field) -> dict:
    field = np.ascontiguousarray(field, dtype=np.float64)
    g = RefGeom()
    _chk(lib().ref_aft_forward(C.byref(p), _dp(field), int(field.shape[0]), C.byref(g)))
    return _field_from_lib()


def scale(p: RefParams, F: dict, spec: tuple, xi: float) -> dict:
    """spec = (kind, d, R, a_B, b_B, ell_H, ell_B, c_B)."""
    _field_to_lib(F)
    m = RefModSpec(*spec)
    g = RefGeom()
    _chk(lib().ref_scale(C.byref(p), C.byref(m), float(xi), C.byref(g)))
    return _field_from_lib()


def scale_table(p: RefParams, F: dict, kind: int, R: float, xi: float) -> dict:
    _field_to_lib(F)
    g = RefGeom()
    _chk(lib().ref_scale_table(C.byref(p), int(kind), float(R), float(xi), C.byref(g)))
    return _field_from_lib()


def aft_inverse(p: RefParams, F: dict) -> np.ndarray:
    _field_to_lib(F)
    out = np.zeros((F["comps"], p.M_ext[0], p.M_ext[1], p.M_ext[2]))
    _chk(lib().ref_aft_inverse(C.byref(p), _dp(out)))
    return out
