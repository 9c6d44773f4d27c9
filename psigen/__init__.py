"""Seeded synthetic inputs for Power-psi (INPUT GENERATOR ONLY).

Shared by both sides of the parity tests -- the fp64 oracle and the CUDA
library consume exactly the arrays produced here.  This module holds none of
the method's arithmetic (no W, c, d, A, B, s, psi): only graphs and activity
vectors, following SURVEY.md §8(d).1 and DESIGN.md "Input recipe".

Graph format (the C-ABI input, reading R8 of DESIGN.md): CSR of *followers per
leader* -- row_ptr int64[N+1], followers int32[M], row j = F(j) sorted
strictly increasing, no self loops.  Edge (n, j) means "n follows j".
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "psigen.cpp")
_LIB = os.path.join(_HERE, "lib", "libpsigen.so")
_lib = None

SEED = 0


def build(force: bool = False) -> str:
    """Compile libpsigen.so (g++ + OpenMP) if missing or stale."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    tmp = _LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["g++", "-O3", "-fopenmp", "-shared", "-fPIC", "-std=c++17",
                           "-o", tmp, _SRC])
    os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.POINTER(ctypes.c_void_p)
        i64, u64, dbl, ci = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int
        lib.psigen_er.argtypes = [i64, dbl, u64, ci, P]
        lib.psigen_chung_lu.argtypes = [i64, i64, dbl, dbl, u64, P]
        lib.psigen_rmat.argtypes = [ci, i64, dbl, dbl, dbl, u64, ci, ci, P]
        for f in (lib.psigen_er, lib.psigen_chung_lu, lib.psigen_rmat):
            f.restype = ci
        lib.psigen_n.argtypes = [ctypes.c_void_p]
        lib.psigen_n.restype = i64
        lib.psigen_m.argtypes = [ctypes.c_void_p]
        lib.psigen_m.restype = i64
        lib.psigen_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.psigen_free.argtypes = [ctypes.c_void_p]
        lib.psigen_uniform.argtypes = [i64, dbl, dbl, u64, u64, ctypes.c_void_p]
        lib.psigen_lognormal.argtypes = [i64, dbl, dbl, u64, u64, ctypes.c_void_p]
        lib.psigen_zero_subset.argtypes = [i64, i64, u64, ctypes.c_void_p]
        lib.psigen_num_threads.restype = ci
        _lib = lib
    return _lib


def _take(handle, alloc=None):
    """Copy a generated graph out of C++ into (row_ptr, followers) arrays.

    ``alloc(shape, dtype)`` may return pinned host memory (e.g. a numpy view
    of a pinned torch tensor); defaults to numpy.empty.
    """
    lib = _load()
    try:
        n = lib.psigen_n(handle)
        m = lib.psigen_m(handle)
        alloc = alloc or (lambda shape, dt: np.empty(shape, dtype=dt))
        row_ptr = alloc((n + 1,), np.int64)
        followers = alloc((m,), np.int32)
        lib.psigen_copy(handle, row_ptr.ctypes.data, followers.ctypes.data)
    finally:
        lib.psigen_free(handle)
    return row_ptr, followers


def er_graph(n, mean, seed=SEED, fix_leaderless=True, alloc=None):
    """Directed G(N, p = mean/(N-1)), no self loops; users without a leader get one."""
    h = ctypes.c_void_p()
    if _load().psigen_er(n, float(mean), seed, int(fix_leaderless), ctypes.byref(h)) != 0:
        raise ValueError("psigen_er: bad arguments")
    return _take(h, alloc)


def chung_lu_graph(n, m, gamma=2.1, max_w=1.4e5, seed=SEED, alloc=None):
    """Chung-Lu power law with exactly m unique edges (leaderless users kept)."""
    h = ctypes.c_void_p()
    if _load().psigen_chung_lu(n, m, float(gamma), float(max_w), seed, ctypes.byref(h)) != 0:
        raise ValueError("psigen_chung_lu: bad arguments")
    return _take(h, alloc)


def rmat_graph(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=SEED, scramble=True,
               fix_leaderless=True, alloc=None):
    """R-MAT (Graph500 quadrants), scrambled labels, dedup, leader fix."""
    h = ctypes.c_void_p()
    if _load().psigen_rmat(scale, edge_factor, a, b, c, seed, int(scramble),
                           int(fix_leaderless), ctypes.byref(h)) != 0:
        raise ValueError("psigen_rmat: bad arguments")
    return _take(h, alloc)


def uniform(n, lo, hi, seed=SEED, stream=0):
    out = np.empty(n, dtype=np.float64)
    _load().psigen_uniform(n, lo, hi, seed, stream, out.ctypes.data)
    return out


def lognormal(n, m, s, seed=SEED, stream=0):
    """exp(m + s Z): m, s are the mean / std of the underlying normal."""
    out = np.empty(n, dtype=np.float64)
    _load().psigen_lognormal(n, m, s, seed, stream, out.ctypes.data)
    return out


def zero_subset(arr, k, seed=SEED):
    """Set exactly k seeded-random entries of arr (float64, contiguous) to 0."""
    assert arr.dtype == np.float64 and arr.flags.c_contiguous
    _load().psigen_zero_subset(arr.shape[0], k, seed, arr.ctypes.data)
    return arr


def num_threads() -> int:
    return _load().psigen_num_threads()


def csr_from_edges(n, edges):
    """Follower-CSR from a list of (follower, leader) pairs (tiny graphs, tests).

    Duplicates are kept out; self loops are rejected.
    """
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if e.size and np.any(e[:, 0] == e[:, 1]):
        raise ValueError("self loop")
    key = np.unique(e[:, 1] * n + e[:, 0]) if e.size else np.zeros(0, np.int64)
    leader, follower = key // n, key % n
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr, leader + 1, 1)
    return np.cumsum(row_ptr), follower.astype(np.int32)


# --------------------------------------------------------------------------
# BASELINE.json configs (SURVEY.md §8(d).1 readings)
# --------------------------------------------------------------------------

@dataclass
class Workload:
    name: str
    row_ptr: np.ndarray
    followers: np.ndarray
    lam: np.ndarray
    mu: np.ndarray
    eps: float

    @property
    def n(self) -> int:
        return int(self.lam.shape[0])

    @property
    def m(self) -> int:
        return int(self.followers.shape[0])


CONFIG_NAMES = {
    0: "C1-tiny: ER N=64 p=10/63, lam,mu~U(0.05,1)",
    1: "C1: ER N=10,000 mean 10 leaders, lam,mu~U(0.05,1), eps=1e-12",
    2: "C2: ER N=1,000,000 mean 15, lam=mu=1 (PageRank alpha=0.5), eps=1e-12",
    3: "C3: Chung-Lu N=5,000,000 M=1e8 gamma=2.1, LogNormal activity, eps=1e-9",
    4: "C4: R-MAT scale 24 ef 16 (0.57,0.19,0.19,0.05), LogNormal, eps=1e-9",
    5: "C5: R-MAT scale 26 ef 16, LogNormal, 5% mu=0, eps=1e-9",
}


def _lognormal_activity(n, seed):
    lam = lognormal(n, -1.0, 1.5, seed, stream=1)
    mu = lognormal(n, -0.5, 1.0, seed, stream=2)
    return lam, mu


def activity_profiles(n: int, k: int, kind: str = "lognormal", seed: int = SEED,
                      pure_posters: bool = False):
    """k independent activity profiles (lam, mu), each of shape (k, n), for the multi-profile
    batch.  Profile j draws from streams 100 + 2j / 101 + 2j of the
    configs' generator: "lognormal" = configs 3-5 (LogNormal(-1, 1.5), LogNormal(-0.5, 1.0)),
    "uniform" = config 1 (U(0.05, 1)); pure_posters zeroes floor(0.05 n) mu per profile
    (config 5)."""
    lam = np.empty((k, n), dtype=np.float64)
    mu = np.empty((k, n), dtype=np.float64)
    for j in range(k):
        if kind == "lognormal":
            lam[j] = lognormal(n, -1.0, 1.5, seed, 100 + 2 * j)
            mu[j] = lognormal(n, -0.5, 1.0, seed, 101 + 2 * j)
        elif kind == "uniform":
            lam[j] = uniform(n, 0.05, 1.0, seed, 100 + 2 * j)
            mu[j] = uniform(n, 0.05, 1.0, seed, 101 + 2 * j)
        else:
            raise ValueError(kind)
        if pure_posters:
            row = np.ascontiguousarray(mu[j])
            zero_subset(row, n // 20, seed + 1 + j)
            mu[j] = row
    return lam, mu


def make_config(k: int, seed: int = SEED, alloc=None, scale: int | None = None) -> Workload:
    """Config k of BASELINE.json (k = 1..5; 0 = the N=64 ER companion of config 1).

    ``scale`` overrides the R-MAT scale of configs 4/5 (tests use small ones).
    """
    if k == 0:
        rp, f = er_graph(64, 10.0, seed, True, alloc)
        return Workload(CONFIG_NAMES[0], rp, f, uniform(64, 0.05, 1.0, seed, 1),
                        uniform(64, 0.05, 1.0, seed, 2), 1e-12)
    if k == 1:
        n = 10_000
        rp, f = er_graph(n, 10.0, seed, True, alloc)
        return Workload(CONFIG_NAMES[1], rp, f, uniform(n, 0.05, 1.0, seed, 1),
                        uniform(n, 0.05, 1.0, seed, 2), 1e-12)
    if k == 2:
        n = 1_000_000
        rp, f = er_graph(n, 15.0, seed, True, alloc)
        return Workload(CONFIG_NAMES[2], rp, f, np.ones(n), np.ones(n), 1e-12)
    if k == 3:
        n = 5_000_000 if scale is None else (1 << scale)
        m = 100_000_000 if scale is None else 20 * n
        rp, f = chung_lu_graph(n, m, 2.1, 1.4e5 if scale is None else max(100.0, n / 50), seed,
                               alloc)
        lam, mu = _lognormal_activity(n, seed)
        return Workload(CONFIG_NAMES[3], rp, f, lam, mu, 1e-9)
    if k in (4, 5):
        sc = (24 if k == 4 else 26) if scale is None else scale
        rp, f = rmat_graph(sc, 16, 0.57, 0.19, 0.19, seed, True, True, alloc)
        n = 1 << sc
        lam, mu = _lognormal_activity(n, seed)
        if k == 5:
            zero_subset(mu, n // 20, seed)          # exactly floor(0.05 N) pure posters
        return Workload(CONFIG_NAMES[k], rp, f, lam, mu, 1e-9)
    raise ValueError(f"unknown config {k}")
