"""CPU tests: the host parameter layer, the C-ABI surface and the oracle pins.

select_parameters / build_grid / WindowSpec::make / pkb_build are restated
in the product's host layer and must be BIT-identical to the reference
(estimates.cpp:211-268, grid.cpp:35-77, window.cpp:76-138)."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden


def test_cabi_exports_every_declared_symbol(S):
    import ctypes
    from paper_2210_01255_b200 import _abi
    hdr = open(os.path.join(ROOT, "include", "sewald_gpu.h")).read()
    declared = set(re.findall(r"\b(sewald_[a-z0-9_]+)\s*\(", hdr))
    lib = ctypes.CDLL(_abi.LIB_PATH)
    missing = [n for n in sorted(declared) if not hasattr(lib, n)]
    assert not missing, missing
    assert declared <= set(_abi.EXPORTED), declared - set(_abi.EXPORTED)


@pytest.mark.parametrize("name", ["c1_stokeslet_d3", "stresslet_d3", "rotlet_d3", "stresslet_d2",
                                  "stokeslet_d2", "rotlet_d1_tg", "stokeslet_d1", "stokeslet_d0"])
def test_params_bit_identical_to_golden(S, name):
    g = load_golden(name)
    for key in [k for k in g if k.startswith("params")]:
        ref = S.api.sewald_params_c.from_buffer_copy(bytes(g[key]))
        sel = S.select_parameters(S.Kernel(int(g["kind"])), int(g["d"]), S.Cell(tuple(g["L"])), float(g["Q"]),
                                  ref.xi, S.ToleranceSpec(float(g["tol"])),
                                  S.SelectionOptions(4, S.WindowKind(int(g["window"])), True))
        assert bytes(sel.params.to_c()) == bytes(ref), key


def test_frozen_selection_values(S):
    """tests/test_estimates.cpp:300-353 frozen chain (stokeslet D=3 and D=0)."""
    sel = S.select_parameters(S.Kernel.stokeslet, 3, S.Cell((1, 1, 1)), 1.0, 10.0, S.ToleranceSpec(1e-8),
                              S.SelectionOptions(f_m=2))
    p, r = sel.params, sel.report
    assert abs(r.U - 1.97696) < 1e-5 and abs(r.kinf - 85.1186) < 1e-4
    assert tuple(p.grid.M) == (30, 30, 30) and p.window.P == 14
    assert p.window.beta == 35.0 and p.window.nu == 9
    assert abs(p.rc - 0.432372) < 1e-6


def test_params_sweep_vs_reference(S, ref):
    rng = np.random.default_rng(3)
    n = 0
    for kind in range(3):
        for d in range(4):
            for win in range(3):
                for _ in range(8):
                    L = rng.uniform(0.3, 3, 3)
                    if d >= 2:
                        L[1] = L[0] * rng.integers(1, 3)
                    if d == 3:
                        L[2] = L[0] * rng.integers(1, 3)
                    Q, xi, tol = 10 ** rng.uniform(-1, 6), 10 ** rng.uniform(0, 1.8), 10 ** rng.uniform(-12, -4)
                    try:
                        rp, rr = ref.select_parameters(kind, d, L, Q, xi, tol, False, 4, win, True)
                    except ref.RefError:
                        with pytest.raises(S.SewaldError):
                            S.select_parameters(S.Kernel(kind), d, S.Cell(L), Q, xi, S.ToleranceSpec(tol),
                                                S.SelectionOptions(4, S.WindowKind(win), True))
                        continue
                    sel = S.select_parameters(S.Kernel(kind), d, S.Cell(L), Q, xi, S.ToleranceSpec(tol),
                                              S.SelectionOptions(4, S.WindowKind(win), True))
                    assert bytes(sel.params.to_c()) == bytes(rp)
                    assert sel.report.U == rr.U and sel.report.kinf == rr.kinf
                    n += 1
    assert n > 200


@pytest.mark.parametrize("P", [4, 8, 12, 16, 18, 24])
def test_pkb_coefficients_bit_identical(S, ref, P):
    w = S.WindowSpec.make(S.WindowKind.pkb, P, 1.0 / 64)
    c = S.EwaldParams(window=w).to_c()
    assert np.array_equal(S.pkb_coefficients(w), ref.pkb_coefficients(ref.params_from(c)))


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_window_eval_and_hat(S, ref, kind):
    w = S.WindowSpec.make(S.WindowKind(kind), 12, 0.05)
    c = ref.params_from(S.EwaldParams(window=w).to_c())
    r = np.linspace(-0.35, 0.35, 301)
    k = np.linspace(-200, 200, 301)
    assert np.array_equal(S.window_eval(w, r), ref.window_eval(c, r))
    assert np.array_equal(S.window_hat(w, k), ref.window_hat(c, k))


def test_build_grid_matches(S, ref):
    for d in range(4):
        for kind in range(3):
            g = S.build_grid(S.Cell((1.0, 1.0, 1.0)), d, 1 / 37.3, 12, S.Kernel(kind), 4)
            r = ref.build_grid((1.0, 1.0, 1.0), d, 1 / 37.3, 12, kind, 4)
            assert tuple(g.M_ext) == tuple(r.M_ext) and g.h == r.h and tuple(g.pad) == tuple(r.pad)


def test_host_errors(S):
    with pytest.raises(S.InvalidArgument):
        S.select_parameters(S.Kernel.stokeslet, 4, S.Cell(), 1.0, 1.0)
    with pytest.raises(S.InvalidArgument):
        S.select_parameters(S.Kernel.stokeslet, 3, S.Cell(), 1.0, -1.0)
    with pytest.raises(S.InvalidArgument):
        S.WindowSpec.make(S.WindowKind.pkb, 5, 0.1)
    with pytest.raises(S.InvalidArgument):
        S.build_grid(S.Cell((1.0, 1.3, 1.0)), 2, 0.1, 8, S.Kernel.stokeslet, 4)


def test_oracle_reproduces_golden(ref):
    """Pin the oracle build against the committed fixtures it produced."""
    g = load_golden("c1_stokeslet_d3")
    p = ref.RefParams.from_buffer_copy(bytes(g["params"]))
    u = ref.full_potential(p, g["x"], g["f"])
    assert np.array_equal(u, g["u"])


def test_dropin_headers_self_contained(tmp_path):
    """Every drop-in header (include/sewald/*.h, include/sewald_gpu.h) compiles
    on its own, as the reference's headers do for its users."""
    import glob
    import os
    import shutil
    import subprocess
    from conftest import ROOT
    cxx = shutil.which("g++")
    if not cxx:
        pytest.skip("no g++")
    hdrs = sorted(glob.glob(os.path.join(ROOT, "include", "sewald", "*.h*")))
    assert hdrs
    for h in hdrs + [os.path.join(ROOT, "include", "sewald_gpu.h")]:
        rel = os.path.relpath(h, os.path.join(ROOT, "include"))
        src = tmp_path / "tu.cpp"
        src.write_text(f'#include "{rel}"\nint main() {{ return 0; }}\n')
        r = subprocess.run([cxx, "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror",
                            "-I", os.path.join(ROOT, "include"), str(src)], capture_output=True, text=True)
        assert r.returncode == 0, (rel, r.stderr[-2000:])


def test_kernel_options_roundtrip(S):
    """Kernel-choice switches (sewald_gpu_set_option): host-only, no GPU call."""
    old = S.get_kernel_option(S.KernelOption.RS_SYM)
    with S.kernel_options(RS_SYM=2, GATHER=1, GATHER_L=15):
        assert S.get_kernel_option(S.KernelOption.RS_SYM) == 2
        assert S.get_kernel_option(S.KernelOption.GATHER) == 1
        assert S.get_kernel_option(S.KernelOption.GATHER_L) == 15
    assert S.get_kernel_option(S.KernelOption.RS_SYM) == old
    with pytest.raises(S.InvalidArgument):
        S.set_kernel_option(S.KernelOption.GATHER_L, 17)
    with pytest.raises(S.InvalidArgument):
        S.set_kernel_option(S.KernelOption.RS_SYM, 5)
