"""Build libpsi.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib", "libpsi.so")
LIB_CHECKED = os.path.join(HERE, "lib", "libpsi_checked.so")   # -DPSI_CHECKS: device bounds checks
SOURCES = ["psi_api.cu", "psi_ingest.cu", "psi_sweep.cu", "psi_heavy.cu", "psi_pagerank.cu", "psi_powernf.cu",
           "psi_batch.cu"]
DEPS = SOURCES + ["psi_internal.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "-t", "0"]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(ROOT, "include", "psi.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """Build lib/libpsi.so, or with checked=True lib/libpsi_checked.so (-DPSI_CHECKS)."""
    lib = LIB_CHECKED if checked else LIB
    if not force and not _stale(lib):
        return lib
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    tmp = lib + f".tmp{os.getpid()}"
    extra = ["-DPSI_CHECKS"] if checked else []
    # experiment builds only (never set by build() / the tests): e.g. PSI_NVCC_EXTRA=-DPSI_EXP_...
    extra += os.environ.get("PSI_NVCC_EXTRA", "").split()
    cmd = [NVCC, *FLAGS, *extra, "-o", tmp] + [os.path.join(CSRC, f) for f in SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-4000:]}")
    if verbose:
        print(res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
