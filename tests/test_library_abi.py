"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/psi.h
declares (no compute calls: this runs without a GPU)."""

import ctypes
import os
import re
import subprocess

import pytest

import paper_2206_09960_b200 as psi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "psi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(psi_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    assert declared_symbols() == sorted(psi.EXPORTED)


def test_library_builds_and_exports_every_symbol():
    path = psi._build.build()
    lib = ctypes.CDLL(path)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.check_output(["nm", "-D", "--defined-only", path], text=True)
    exported = set(re.findall(r" T (psi_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_library_is_sm100a_code():
    path = psi._build.build()
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], text=True)
    assert "sm_100a" in out


def test_error_paths_without_device():
    """Argument validation happens before any CUDA call."""
    lib = psi.load_library()
    ctx = ctypes.c_void_p()
    st = lib.psi_build_graph(0, 0, None, None, None, None, 0, None, ctypes.byref(ctx))
    assert st == psi.PSI_E_INVALID_ARG and b"n = 0" in lib.psi_last_error()
    st = lib.psi_iterate(None, 1e-9, 10, 0, None, None)
    assert st == psi.PSI_E_INVALID_ARG
    info = psi.psi_info()
    assert lib.psi_get_info(None, ctypes.byref(info)) == psi.PSI_E_INVALID_ARG
    st = lib.psi_build_graph_batch(10, 0, None, None, 0, None, None, 0, None, ctypes.byref(ctx))
    assert st == psi.PSI_E_INVALID_ARG and b"nprof" in lib.psi_last_error()
    assert lib.psi_get_profile_stats(None, None, None) == psi.PSI_E_INVALID_ARG
    assert lib.psi_time_sweep_batch(None, 1, None) == psi.PSI_E_INVALID_ARG
    lib.psi_destroy(None)   # no-op


def test_no_oracle_import_in_product_package():
    """The product path never touches oracle/ (parity would be void)."""
    pkg = os.path.join(ROOT, "paper_2206_09960_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f


def test_binding_rejects_bad_arrays():
    """the binding validates dtype / shape / contiguity before any C call (a numpy
    default-int64 followers array would otherwise be read as int32 pairs)."""
    import numpy as np
    import paper_2206_09960_b200 as psi
    rp = np.array([0, 1, 1], dtype=np.int64)
    f = np.array([1], dtype=np.int32)
    lam = np.array([0.5, 0.5])
    mu = np.array([0.5, 0.5])
    with pytest.raises(TypeError, match="followers"):
        psi.PsiGraph(rp, f.astype(np.int64), lam, mu)
    with pytest.raises(TypeError, match="lam"):
        psi.PsiGraph(rp, f, lam.astype(np.float32), mu)
    with pytest.raises(ValueError, match="mu"):
        psi.PsiGraph(rp, f, lam, mu[:1])
    with pytest.raises(ValueError, match="row_ptr"):
        psi.PsiGraph(rp[:2], f, lam, mu)
    with pytest.raises(ValueError, match="contiguous"):
        psi.PsiGraph(rp, f, np.array([0.5, 9, 0.5, 9])[::2], mu)
    # outputs: exact dtype and size, writable, contiguous -- never a silent temporary copy
    import torch
    with pytest.raises(ValueError, match="shape"):
        psi._check(torch.empty(3, dtype=torch.float64), "out", "float64", (2,), writable=True)
    with pytest.raises(TypeError):
        psi._check(torch.empty(2, dtype=torch.float32), "out", "float64", (2,), writable=True)
    with pytest.raises(ValueError, match="contiguous"):
        psi._check(torch.empty(4, dtype=torch.float64)[::2], "out", "float64", (2,), writable=True)
    ro = np.zeros(2)
    ro.flags.writeable = False
    with pytest.raises(ValueError, match="read-only"):
        psi._check(ro, "out", "float64", (2,), writable=True)
    ptr, kind, keep = psi._check([0, 1], "x", "int64", (2,))
    assert kind == psi.PSI_MEM_HOST and keep.dtype == np.int64
