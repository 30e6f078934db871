"""The C-ABI library loads and exports every symbol include/svh.h declares (CPU only)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "svh.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(svh_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_boundary():
    syms = declared_symbols()
    for s in ("svh_setup", "svh_matvec", "svh_solve", "svh_apply_system", "svh_destroy"):
        assert s in syms


def test_library_exports_all_declared_symbols():
    from paper_2105_08627_b200 import build, svh
    if not os.path.exists(svh.LIB_PATH):
        build.build(verbose=False)
    L = ctypes.CDLL(svh.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert set(declared_symbols()) == set(svh.EXPORTED)


def test_host_only_calls():
    """Calls that need no GPU: defaults, error string, launch counter, argument validation."""
    from paper_2105_08627_b200 import svh
    L = svh.lib()
    o = svh.Opts()
    L.svh_default_opts(ctypes.byref(o))
    assert o.restart == 50 and o.tucker_tol == 0.0
    assert isinstance(L.svh_last_error(), bytes)
    assert L.svh_launch_count() >= 0
    # invalid grid is rejected before any device work
    g = svh.Grid(0, 1, 1, 1e-6)
    h = ctypes.c_void_p()
    mats = (svh.Material * 1)(svh.Material(1e7, 1e-7))
    mat = (ctypes.c_uint8 * 1)(1)
    code = L.svh_setup(ctypes.byref(g), mat, mats, 1, 1e9, None, 0, ctypes.byref(h))
    assert code == -1
    assert b"bad grid" in L.svh_last_error()


def test_opts_validation_host_only():
    """svh_opts is validated before any device work: restart range (the FGMRES Hessenberg
    scratch), plan (0 auto, 3 P3s, 5 P5), precision (0 / 1; the complex128 build needs dense
    spectra) and the Schur solver."""
    from paper_2105_08627_b200 import svh
    L = svh.lib()
    g = svh.Grid(2, 1, 1, 1e-6)
    mats = (svh.Material * 1)(svh.Material(1e7, 1e-7))
    mat = (ctypes.c_uint8 * 2)(1, 1)
    for field, bad, msg in (("restart", 5000, b"restart"), ("restart", 0, b"restart"), ("plan", 4, b"plan"),
                            ("precision", 2, b"precision"), ("tucker_tol", 1.5, b"tucker_tol"),
                            ("schur_solver", 2, b"schur_solver")):
        o = svh.Opts()
        L.svh_default_opts(ctypes.byref(o))
        setattr(o, field, bad)
        h = ctypes.c_void_p()
        code = L.svh_setup(ctypes.byref(g), mat, mats, 1, 1e9, ctypes.byref(o), 0, ctypes.byref(h))
        assert code == -1, field
        assert msg in L.svh_last_error(), (field, L.svh_last_error())
    o = svh.Opts()
    L.svh_default_opts(ctypes.byref(o))
    o.precision, o.tucker_tol = 1, 1e-6
    h = ctypes.c_void_p()
    assert L.svh_setup(ctypes.byref(g), mat, mats, 1, 1e9, ctypes.byref(o), 0, ctypes.byref(h)) == -1
    assert b"complex128" in L.svh_last_error()
