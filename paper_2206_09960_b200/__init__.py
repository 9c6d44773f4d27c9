"""Power-psi on one B200: thin Python binding over the C-ABI library libpsi.so.

The binding only marshals arguments (pointers, sizes, the CUDA stream) to the C
entry points declared in ``include/psi.h``; every step of the hot path runs in
the library's sm_100a kernels.  PyTorch is used for device memory and streams.
There is no CPU fallback: if libpsi.so cannot be built or loaded, every call
raises.

    import torch, paper_2206_09960_b200 as psi
    g = psi.PsiGraph(row_ptr, followers, lam, mu)      # torch CUDA tensors or host arrays
    status, T, gap = g.iterate(eps=1e-9)
    scores = g.get_psi()                                # torch.float64 on the device
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

PSI_OK = 0
PSI_NOT_CONVERGED = 1
PSI_E_INVALID_ARG = -1
PSI_E_GRAPH = -2
PSI_E_ACTIVITY = -3
PSI_E_OOM = -4
PSI_E_CUDA = -5
PSI_E_STATE = -6
PSI_E_NUMERIC = -7
PSI_MEM_HOST = 0
PSI_MEM_DEVICE = 1
NORMS = {"row": 0, "col": 1, "one": 2}

_STATUS_NAMES = {0: "PSI_OK", 1: "PSI_NOT_CONVERGED", -1: "PSI_E_INVALID_ARG", -2: "PSI_E_GRAPH",
                 -3: "PSI_E_ACTIVITY", -4: "PSI_E_OOM", -5: "PSI_E_CUDA", -6: "PSI_E_STATE",
                 -7: "PSI_E_NUMERIC"}

EXPORTED = ["psi_build_graph", "psi_iterate", "psi_get_psi", "psi_get_series",
            "psi_get_residual_history", "psi_time_sweep", "psi_get_info", "psi_pagerank",
            "psi_get_pagerank", "psi_power_nf", "psi_nsystems", "psi_build_graph_batch",
            "psi_get_profile_stats", "psi_get_profile_history", "psi_time_sweep_batch",
            "psi_empty_cache", "psi_destroy", "psi_last_error"]


class PsiError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class psi_info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m", ctypes.c_int64), ("n_f", ctypes.c_int64),
                ("n_g", ctypes.c_int64), ("n_leaderless", ctypes.c_int64),
                ("kappa_row", ctypes.c_double), ("kappa_col", ctypes.c_double),
                ("rho_A", ctypes.c_double), ("ingest_ms", ctypes.c_double),
                ("iterate_ms", ctypes.c_double), ("last_iters", ctypes.c_int64),
                ("last_gap", ctypes.c_double), ("num_tiles", ctypes.c_int64),
                ("num_long_rows", ctypes.c_int64), ("grid", ctypes.c_int64),
                ("device_bytes", ctypes.c_int64), ("relabeled", ctypes.c_int64),
                ("block", ctypes.c_int64), ("hot_smem", ctypes.c_int64),
                ("n_heavy", ctypes.c_int64), ("heavy_entries", ctypes.c_int64),
                ("heavy_panels", ctypes.c_int64), ("heavy_labels", ctypes.c_int64),
                ("last_solver", ctypes.c_int64), ("n_profiles", ctypes.c_int64),
                ("tile_edges", ctypes.c_int64), ("overlapped", ctypes.c_int64),
                ("sliced_ell", ctypes.c_int64), ("sell_long_rows", ctypes.c_int64),
                ("sell_pieces", ctypes.c_int64), ("sell_words", ctypes.c_int64),
                ("stream_edges", ctypes.c_int64)]


_lib = None


def library_path() -> str:
    return _build.LIB


def load_library(build_if_stale: bool = True):
    """Load libpsi.so (building it in-tree with nvcc if missing/stale). Raises on failure."""
    global _lib
    if _lib is not None:
        return _lib
    checked = os.environ.get("PSI_LIB", "") == "checked"   # device bounds-checked build
    path = _build.LIB_CHECKED if checked else _build.LIB
    if build_if_stale and _build._stale(path):
        _build.build(checked=checked)
    if not os.path.exists(path):
        raise RuntimeError(f"libpsi.so not found at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    vp, i64, dbl, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    lib.psi_build_graph.argtypes = [i64, i64, vp, vp, vp, vp, ci, vp, ctypes.POINTER(vp)]
    lib.psi_iterate.argtypes = [vp, dbl, i64, ci, ctypes.POINTER(i64), ctypes.POINTER(dbl)]
    lib.psi_get_psi.argtypes = [vp, vp, ci]
    lib.psi_get_series.argtypes = [vp, vp, ci]
    lib.psi_pagerank.argtypes = [vp, dbl, dbl, i64, ctypes.POINTER(i64), ctypes.POINTER(dbl)]
    lib.psi_get_pagerank.argtypes = [vp, vp, ci]
    lib.psi_power_nf.argtypes = [vp, vp, i64, dbl, i64, vp, vp, ci, vp]
    lib.psi_nsystems.argtypes = [vp, dbl, i64, vp, ci, ctypes.POINTER(i64)]
    lib.psi_get_residual_history.argtypes = [vp, vp, i64, ctypes.POINTER(i64)]
    lib.psi_get_info.argtypes = [vp, ctypes.POINTER(psi_info)]
    lib.psi_time_sweep.argtypes = [vp, i64, ctypes.POINTER(dbl), ctypes.POINTER(dbl),
                                   ctypes.POINTER(dbl)]
    lib.psi_build_graph_batch.argtypes = [i64, i64, vp, vp, i64, vp, vp, ci, vp, ctypes.POINTER(vp)]
    lib.psi_get_profile_stats.argtypes = [vp, vp, vp]
    lib.psi_get_profile_history.argtypes = [vp, i64, vp, i64, ctypes.POINTER(i64)]
    lib.psi_time_sweep_batch.argtypes = [vp, i64, ctypes.POINTER(dbl)]
    lib.psi_empty_cache.argtypes = []
    lib.psi_empty_cache.restype = ci
    lib.psi_destroy.argtypes = [vp]
    lib.psi_destroy.restype = None
    lib.psi_last_error.restype = ctypes.c_char_p
    for f in ("psi_build_graph", "psi_iterate", "psi_get_psi", "psi_get_series",
              "psi_get_residual_history", "psi_get_info", "psi_time_sweep", "psi_pagerank",
              "psi_get_pagerank", "psi_power_nf", "psi_nsystems", "psi_build_graph_batch",
              "psi_get_profile_stats", "psi_get_profile_history", "psi_time_sweep_batch"):
        getattr(lib, f).restype = ci
    _lib = lib
    return lib


def _err(lib) -> str:
    return (lib.psi_last_error() or b"").decode()


_DT = {"int64": (np.int64, "torch.int64"), "int32": (np.int32, "torch.int32"),
       "float64": (np.float64, "torch.float64")}


def _check(a, name: str, dtype: str, shape: tuple, writable: bool = False):
    """Validate one array argument against the C-ABI contract (include/psi.h) and return
    (pointer, mem_kind, keepalive).  Raises TypeError / ValueError instead of casting or
    copying: the library reads and writes exactly the bytes this pointer addresses."""
    try:
        import torch
        is_t = isinstance(a, torch.Tensor)
    except ImportError:
        is_t = False
    if is_t:
        if str(a.dtype) != _DT[dtype][1]:
            raise TypeError(f"{name}: dtype {a.dtype}, expected {_DT[dtype][1]}")
        if tuple(a.shape) != tuple(shape):
            raise ValueError(f"{name}: shape {tuple(a.shape)}, expected {tuple(shape)}")
        if not a.is_contiguous():
            raise ValueError(f"{name}: tensor must be contiguous")
        if a.is_cuda and a.device.index != torch.cuda.current_device():
            raise ValueError(f"{name}: on {a.device}, the current device is "
                             f"cuda:{torch.cuda.current_device()}")
        if not a.is_cuda and a.device.type != "cpu":
            raise ValueError(f"{name}: unsupported device {a.device}")
        return a.data_ptr(), (PSI_MEM_DEVICE if a.is_cuda else PSI_MEM_HOST), a
    if not isinstance(a, np.ndarray):
        if writable:
            raise TypeError(f"{name}: output must be a numpy array or torch tensor")
        a = np.asarray(a)
        if a.dtype != _DT[dtype][0] and a.size == 0:
            a = a.astype(_DT[dtype][0])           # an empty list has no dtype of its own
    if a.dtype != _DT[dtype][0]:
        raise TypeError(f"{name}: dtype {a.dtype}, expected {np.dtype(_DT[dtype][0])}")
    if a.shape != tuple(shape):
        raise ValueError(f"{name}: shape {a.shape}, expected {tuple(shape)}")
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError(f"{name}: array must be C-contiguous")
    if writable and not a.flags["WRITEABLE"]:
        raise ValueError(f"{name}: array is read-only")
    return a.ctypes.data, PSI_MEM_HOST, a


def _current_stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class PsiGraph:
    """One ingested follower graph + activity (a psi_ctx).

    row_ptr int64[N+1], followers int32[M] (CSR of followers per leader), lam/mu float64[N];
    all four on the device (torch CUDA tensors) or all on the host (pinned torch tensors or
    numpy arrays).  Work runs on torch's current CUDA stream at construction.

    lam/mu of shape (k, N), k >= 2, build a multi-profile batch context
    (psi_build_graph_batch): iterate() then runs Alg. 2 for every profile and get_psi()
    returns (k, N); profile_stats() gives each profile's T and gap.
    """

    def __init__(self, row_ptr, followers, lam, mu, stream=None):
        self._lib = load_library()
        self._ctx = ctypes.c_void_p()
        shape = tuple(lam.shape) if hasattr(lam, "shape") else (len(lam),)
        if len(shape) not in (1, 2):
            raise ValueError(f"lam: shape {shape}, expected (N,) or (k, N)")
        self.k = int(shape[0]) if len(shape) == 2 else 1
        self.batch = len(shape) == 2
        self.n = int(shape[-1])
        self.m = int(len(followers))
        parts = [_check(row_ptr, "row_ptr", "int64", (self.n + 1,)),
                 _check(followers, "followers", "int32", (self.m,)),
                 _check(lam, "lam", "float64", shape), _check(mu, "mu", "float64", shape)]
        kinds = {k for _, k, _ in parts}
        if len(kinds) != 1:
            raise ValueError("row_ptr, followers, lam, mu must all be host or all device")
        self.stream = stream if stream is not None else _current_stream()
        if len(shape) == 2:
            st = self._lib.psi_build_graph_batch(self.n, self.m, parts[0][0], parts[1][0], self.k,
                                                 parts[2][0], parts[3][0], kinds.pop(),
                                                 self.stream, ctypes.byref(self._ctx))
        else:
            st = self._lib.psi_build_graph(self.n, self.m, parts[0][0], parts[1][0], parts[2][0],
                                           parts[3][0], kinds.pop(), self.stream,
                                           ctypes.byref(self._ctx))
        if st != PSI_OK:
            raise PsiError(st, _err(self._lib))

    # -- Alg. 2
    def iterate(self, eps: float = 1e-9, max_iters: int = 100_000, norm: str = "row"):
        """Returns (status, T, gap_T); status is PSI_OK or PSI_NOT_CONVERGED."""
        T = ctypes.c_int64()
        gap = ctypes.c_double()
        st = self._lib.psi_iterate(self._ctx, float(eps), int(max_iters), NORMS[norm],
                                   ctypes.byref(T), ctypes.byref(gap))
        if st < 0:
            raise PsiError(st, _err(self._lib))
        return st, T.value, gap.value

    def _get(self, fn, out, device, shape=None):
        import torch
        shape = (self.n,) if shape is None else shape
        if out is None:
            out = torch.empty(shape, dtype=torch.float64,
                              device="cuda" if device else "cpu")
        ptr, kind, keep = _check(out, "out", "float64", shape, writable=True)
        st = fn(self._ctx, ptr, kind)
        if st != PSI_OK:
            raise PsiError(st, _err(self._lib))
        return out

    def get_psi(self, out=None, device: bool = True):
        """psi[n] in the caller's original labels (torch.float64); (k, n) on a batch context."""
        return self._get(self._lib.psi_get_psi, out, device,
                         (self.k, self.n) if self.batch else None)

    def profile_stats(self):
        """Batch context: (T[k], gap[k]) numpy arrays of the last iterate()."""
        T = np.zeros(self.k, dtype=np.int64)
        gap = np.zeros(self.k, dtype=np.float64)
        st = self._lib.psi_get_profile_stats(self._ctx, T.ctypes.data, gap.ctypes.data)
        if st != PSI_OK:
            raise PsiError(st, _err(self._lib))
        return T, gap

    def profile_history(self, p: int) -> np.ndarray:
        """Batch context: raw eps_t of profile p, t = 1..T_p."""
        n = ctypes.c_int64()
        st = self._lib.psi_get_profile_history(self._ctx, int(p), None, 0, ctypes.byref(n))
        if st != PSI_OK:
            raise PsiError(st, _err(self._lib))
        out = np.empty(max(n.value, 0), dtype=np.float64)
        if n.value:
            st = self._lib.psi_get_profile_history(self._ctx, int(p), out.ctypes.data, n.value,
                                                   ctypes.byref(n))
            if st != PSI_OK:
                raise PsiError(st, _err(self._lib))
        return out

    def time_sweep_batch(self, sweeps: int = 20) -> float:
        """Batch context: device ms of one four-profile sweep (k_tiles_b + k_fix_b)."""
        ms = ctypes.c_double()
        st = self._lib.psi_time_sweep_batch(self._ctx, int(sweeps), ctypes.byref(ms))
        if st != PSI_OK:
            raise PsiError(st, _err(self._lib))
        return ms.value

    def get_series(self, out=None, device: bool = True):
        """s_T[n] (Eq. (13)-(14)) in original labels."""
        return self._get(self._lib.psi_get_series, out, device)

    def pagerank(self, alpha: float = 0.85, eps: float = 1e-9, max_iters: int = 100_000):
        """PageRank power method, Eq. (22), on this graph: returns (status, T, gap_T)."""
        T = ctypes.c_int64()
        gap = ctypes.c_double()
        st = self._lib.psi_pagerank(self._ctx, float(alpha), float(eps), int(max_iters),
                                    ctypes.byref(T), ctypes.byref(gap))
        if st < 0:
            raise PsiError(st, _err(self._lib))
        return st, T.value, gap.value

    def get_pagerank(self, out=None, device: bool = True):
        """pi[n] of the last pagerank() in the caller's original labels (torch.float64)."""
        return self._get(self._lib.psi_get_pagerank, out, device)

    def power_nf(self, origins, eps: float = 1e-9, max_iters: int = 100_000):
        """Alg. 1 for the given origins: returns (status, p, q, iters) with p, q torch.float64
        (k, n) on the device (origin-major) and iters a numpy int64 array."""
        import torch
        org = np.ascontiguousarray(np.asarray(origins, dtype=np.int32).ravel())
        k = org.size
        p = torch.empty((k, self.n), dtype=torch.float64, device="cuda")
        q = torch.empty((k, self.n), dtype=torch.float64, device="cuda")
        iters = np.zeros(k, dtype=np.int64)
        st = self._lib.psi_power_nf(self._ctx, org.ctypes.data, k, float(eps), int(max_iters),
                                    p.data_ptr(), q.data_ptr(), PSI_MEM_DEVICE, iters.ctypes.data)
        if st < 0:
            raise PsiError(st, _err(self._lib))
        return st, p, q, iters

    def nsystems(self, eps: float = 1e-9, max_iters: int = 100_000):
        """psi by Alg. 1 for every origin + Eq. (1): returns (status, psi on device, matvecs)."""
        import torch
        out = torch.empty(self.n, dtype=torch.float64, device="cuda")
        mv = ctypes.c_int64()
        st = self._lib.psi_nsystems(self._ctx, float(eps), int(max_iters), out.data_ptr(),
                                    PSI_MEM_DEVICE, ctypes.byref(mv))
        if st < 0:
            raise PsiError(st, _err(self._lib))
        return st, out, mv.value

    def get_residual_history(self) -> np.ndarray:
        n = ctypes.c_int64()
        st = self._lib.psi_get_residual_history(self._ctx, None, 0, ctypes.byref(n))
        if st != PSI_OK:
            raise PsiError(st, _err(self._lib))
        out = np.empty(max(n.value, 0), dtype=np.float64)
        if n.value:
            st = self._lib.psi_get_residual_history(self._ctx, out.ctypes.data, n.value,
                                                    ctypes.byref(n))
            if st != PSI_OK:
                raise PsiError(st, _err(self._lib))
        return out

    def time_sweep(self, sweeps: int = 20):
        """(k_heavy ms, k_tiles ms, k_fix ms): average per-launch device time over `sweeps`
        sweeps (CUDA events on the context's stream around each launch)."""
        h, a, b = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        st = self._lib.psi_time_sweep(self._ctx, int(sweeps), ctypes.byref(h), ctypes.byref(a),
                                      ctypes.byref(b))
        if st != PSI_OK:
            raise PsiError(st, _err(self._lib))
        return h.value, a.value, b.value

    def info(self) -> dict:
        inf = psi_info()
        st = self._lib.psi_get_info(self._ctx, ctypes.byref(inf))
        if st != PSI_OK:
            raise PsiError(st, _err(self._lib))
        return {name: getattr(inf, name) for name, _ in psi_info._fields_}

    def close(self):
        if self._ctx:
            self._lib.psi_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def empty_cache() -> None:
    """Return the device memory the library's pool (current device) caches but no context uses
    (psi_empty_cache; the analogue of torch.cuda.empty_cache())."""
    lib = load_library()
    st = lib.psi_empty_cache()
    if st != PSI_OK:
        raise PsiError(st, _err(lib))


def psi_scores(row_ptr, followers, lam, mu, eps=1e-9, max_iters=100_000, norm="row"):
    """One-shot convenience: ingest, Alg. 2 to eps, return (psi, T, status)."""
    with PsiGraph(row_ptr, followers, lam, mu) as g:
        st, T, _ = g.iterate(eps, max_iters, norm)
        return g.get_psi(), T, st
