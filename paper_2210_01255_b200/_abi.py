"""ctypes binding of the C-ABI declared in include/sewald_gpu.h.

Loads paper_2210_01255_b200/lib/libsewald_gpu.so (built in-tree by
``__graft_entry__.build()``). There is no fallback: if the library is missing
the import fails with instructions, so no computation can silently run on a
CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SEWALD_LIB") or os.path.join(_HERE, "lib", "libsewald_gpu.so")

OK, EINVAL, EDOMAIN, ERUNTIME, ECUDA, ECUFFT, ENOMEM = range(7)
STOKESLET, STRESSLET, ROTLET = 0, 1, 2
WIN_KB, WIN_PKB, WIN_TG = 0, 1, 2


class sewald_params_c(C.Structure):
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


class sewald_report_c(C.Structure):
    _fields_ = [
        ("tau_abs", C.c_double), ("U", C.c_double), ("kinf", C.c_double),
        ("fourier_trunc", C.c_double), ("realspace_trunc", C.c_double),
        ("window_err", C.c_double), ("h_estimate", C.c_double),
        ("P_estimate", C.c_int32), ("h_target", C.c_double), ("P_target", C.c_int32),
        ("rc_clamped", C.c_int32), ("kinf_clamped", C.c_int32),
        ("window_saturated", C.c_int32), ("tg_support_from_pkb", C.c_int32),
    ]


class sewald_timings_c(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "h2d_ms", "sort_ms", "spread_ms", "fft_fwd_ms", "scale_ms", "fft_inv_ms", "gather_ms",
        "realspace_ms", "assemble_ms", "d2h_ms", "total_ms")] + [
        ("kernel_launches", C.c_int64), ("realspace_pairs", C.c_int64)]


class sewald_fourier_geom_c(C.Structure):
    _fields_ = [("d", C.c_int32), ("comps", C.c_int32),
                ("n_per", C.c_int32 * 3), ("n_far", C.c_int32 * 3), ("n_near", C.c_int32 * 3),
                ("n_zero", C.c_int32 * 3), ("n_near_rows", C.c_int32),
                ("far_len", C.c_int64), ("near_len", C.c_int64), ("zero_len", C.c_int64)]


class sewald_modspec_c(C.Structure):
    _fields_ = [("kind", C.c_int32), ("d", C.c_int32), ("R", C.c_double), ("a_B", C.c_double),
                ("b_B", C.c_double), ("ell_H", C.c_double), ("ell_B", C.c_double), ("c_B", C.c_double)]


DP = C.POINTER(C.c_double)
VP = C.c_void_p
I64 = C.c_int64
IP = C.POINTER(C.c_int)

# (name, restype, argtypes)
_SIGS = [
    ("sewald_select_parameters", C.c_int, [C.c_int, C.c_int, DP, C.c_double, C.c_double, C.c_double,
                                           C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.POINTER(sewald_params_c), C.POINTER(sewald_report_c)]),
    ("sewald_window_make", C.c_int, [C.c_int, C.c_int, C.c_double, C.POINTER(sewald_params_c)]),
    ("sewald_build_grid", C.c_int, [DP, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                    C.POINTER(sewald_params_c)]),
    ("sewald_pkb_coefficients", C.c_int, [C.POINTER(sewald_params_c), DP]),
    ("sewald_window_eval", C.c_int, [C.POINTER(sewald_params_c), DP, I64, DP]),
    ("sewald_window_hat", C.c_int, [C.POINTER(sewald_params_c), DP, I64, DP]),
    ("sewald_source_quantity", C.c_double, [C.c_int, DP, DP, I64]),
    ("sewald_last_error", C.c_char_p, []),
    ("sewald_gpu_create", C.c_int, [C.c_int, C.POINTER(VP)]),
    ("sewald_gpu_destroy", None, [VP]),
    ("sewald_gpu_last_error", C.c_char_p, [VP]),
    ("sewald_gpu_set_stream", C.c_int, [VP, VP]),
    ("sewald_gpu_get_timings", C.c_int, [VP, C.POINTER(sewald_timings_c)]),
    ("sewald_gpu_set_profiling", C.c_int, [VP, C.c_int]),
    ("sewald_gpu_host_buffer", C.c_int, [VP, C.c_size_t, C.POINTER(VP)]),
    ("sewald_gpu_fp64_peak", C.c_int, [VP, DP]),
    ("sewald_gpu_launch_count", I64, [VP]),
    ("sewald_gpu_set_option", C.c_int, [C.c_int, C.c_int]),
    ("sewald_gpu_multi_create", C.c_int, [C.c_int, IP, C.POINTER(VP)]),
    ("sewald_gpu_multi_destroy", None, [VP]),
    ("sewald_gpu_multi_last_error", C.c_char_p, [VP]),
    ("sewald_gpu_multi_size", C.c_int, [VP]),
    ("sewald_gpu_multi_context", VP, [VP, C.c_int]),
    ("sewald_gpu_multi_full_potential", C.c_int, [VP, C.POINTER(sewald_params_c), DP, DP, DP, I64, DP, I64,
                                                  C.c_int, C.c_int, DP]),
    ("sewald_gpu_multi_fourier_potential", C.c_int, [VP, C.POINTER(sewald_params_c), DP, DP, DP, I64, DP, I64,
                                                     C.c_int, C.c_int, DP]),
    ("sewald_gpu_get_option", C.c_int, [C.c_int, IP]),
    ("sewald_gpu_session_pair_count", I64, [VP, C.c_int]),
    ("sewald_gpu_full_potential", C.c_int, [VP, C.POINTER(sewald_params_c), DP, DP, DP, I64, DP, I64,
                                            C.c_int, C.c_int, DP]),
    ("sewald_gpu_fourier_potential", C.c_int, [VP, C.POINTER(sewald_params_c), DP, DP, DP, I64, DP,
                                               I64, C.c_int, C.c_int, DP]),
    ("sewald_gpu_realspace_potential", C.c_int, [VP, C.c_int, C.c_int, DP, DP, DP, DP, I64, DP, I64,
                                                 C.c_int, C.c_double, C.c_double, C.c_int, DP]),
    ("sewald_gpu_spread", C.c_int, [VP, C.POINTER(sewald_params_c), DP, DP, DP, I64, DP]),
    ("sewald_gpu_gather", C.c_int, [VP, C.POINTER(sewald_params_c), DP, DP, I64, DP]),
    ("sewald_modspec_optimal", C.c_int, [C.c_int, C.c_int, C.c_double, C.POINTER(sewald_modspec_c)]),
    ("sewald_aft_geometry", C.c_int, [C.POINTER(sewald_params_c), C.c_int, C.POINTER(sewald_fourier_geom_c),
                                      C.POINTER(C.c_int32)]),
    ("sewald_gpu_aft_forward", C.c_int, [VP, C.POINTER(sewald_params_c), DP, C.POINTER(sewald_fourier_geom_c),
                                         DP, DP, DP]),
    ("sewald_gpu_aft_inverse", C.c_int, [VP, C.POINTER(sewald_params_c), C.POINTER(sewald_fourier_geom_c),
                                         C.POINTER(C.c_int32), DP, DP, DP, DP]),
    ("sewald_gpu_scale", C.c_int, [VP, C.POINTER(sewald_params_c), C.POINTER(sewald_modspec_c), C.c_double,
                                   C.POINTER(sewald_fourier_geom_c), C.POINTER(C.c_int32), DP, DP, DP, DP, DP, DP]),
    ("sewald_gpu_scale_table", C.c_int, [VP, C.POINTER(sewald_params_c), C.c_int, C.POINTER(C.c_int32), DP,
                                         C.c_double, C.POINTER(sewald_fourier_geom_c), DP, DP]),
    ("sewald_gpu_precompute_0p", C.c_int, [VP, C.POINTER(sewald_params_c), C.c_int, C.c_double,
                                           C.POINTER(C.c_int32), DP]),
    ("sewald_gpu_set_table0p", C.c_int, [VP, C.POINTER(sewald_params_c), C.POINTER(C.c_int32), DP]),
    ("sewald_gpu_session_set_table0p", C.c_int, [VP, C.POINTER(C.c_int32), DP]),
    ("sewald_gpu_session_create", C.c_int, [VP, C.POINTER(sewald_params_c), C.POINTER(VP)]),
    ("sewald_gpu_session_destroy", None, [VP]),
    ("sewald_gpu_session_set_sources", C.c_int, [VP, VP, VP, VP, I64]),
    ("sewald_gpu_session_set_targets", C.c_int, [VP, VP, I64, C.c_int]),
    ("sewald_gpu_session_grid_size", I64, [VP]),
    ("sewald_gpu_session_spread", C.c_int, [VP, I64, I64, VP]),
    ("sewald_gpu_session_solve", C.c_int, [VP, VP, C.c_int]),
    ("sewald_gpu_session_evaluate", C.c_int, [VP, C.c_int, C.c_int, C.c_int, VP]),
    ("sewald_gpu_session_run", C.c_int, [VP, C.c_int, VP]),
    ("sewald_gpu_session_d0_geometry", C.c_int, [VP, C.c_int, IP, IP, IP, IP]),
    ("sewald_gpu_session_d0_forward", C.c_int, [VP, C.c_int, VP, C.c_int, C.c_int, C.c_int, IP, VP]),
    ("sewald_gpu_session_d0_middle", C.c_int, [VP, C.c_int, VP, C.c_int, IP, C.c_int, C.c_int, VP]),
    ("sewald_gpu_session_d0_inverse", C.c_int, [VP, C.c_int, VP, C.c_int, C.c_int, C.c_int, IP, VP]),
    ("sewald_gpu_session_set_flow", C.c_int, [VP, VP]),
    ("sewald_gpu_direct_sum_0p", C.c_int, [VP, C.c_int, DP, DP, DP, I64, DP, I64, C.c_int, DP]),
    ("sewald_gpu_ewald_fourier_3p", C.c_int, [VP, C.c_int, DP, C.c_double, IP, DP, DP, DP, I64, DP, I64, DP]),
    ("sewald_gpu_fourier_reference_potential", C.c_int, [VP, C.c_int, C.c_int, DP, C.c_double, IP, DP, DP, DP,
                                                         I64, DP, I64, DP]),
    ("sewald_gpu_qtensor", C.c_int, [VP, C.c_int, C.c_int, C.c_int, I64, DP, C.c_double, DP]),
    ("sewald_gpu_incomplete_bessel_k4", C.c_int, [VP, I64, DP, DP, DP]),
    ("sewald_rms_error", C.c_int, [DP, DP, I64, DP, DP]),
]

EXPORTED = [s[0] for s in _SIGS]

_lib = None
_lock = threading.Lock()


def load():
    """Load the engine library once; raise if it has not been built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA engine first "
                "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
        lib = C.CDLL(LIB_PATH)
        for name, res, args in _SIGS:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class SewaldError(Exception):
    """Base class; subclasses mirror the reference's std exception types."""


class InvalidArgument(SewaldError, ValueError):
    """std::invalid_argument in the reference."""


class DomainError(SewaldError, ArithmeticError):
    """std::domain_error in the reference."""


class SewaldRuntimeError(SewaldError, RuntimeError):
    """std::runtime_error in the reference."""


class DeviceError(SewaldError, RuntimeError):
    """CUDA / cuFFT / allocation failure."""


def raise_for(code: int, message: str):
    if code == OK:
        return
    cls = {EINVAL: InvalidArgument, EDOMAIN: DomainError, ERUNTIME: SewaldRuntimeError}.get(code, DeviceError)
    raise cls(message or f"sewald error code {code}")
