"""Error and ranking metrics used by the parity protocol.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

from __future__ import annotations

import numpy as np


def relative_error(psi_true, psi_eps) -> float:
    """Eq. (23): ||psi_true - psi_eps||_2 / ||psi_true||_2."""
    psi_true = np.asarray(psi_true, dtype=np.float64)
    return float(np.linalg.norm(psi_true - psi_eps) / np.linalg.norm(psi_true))


def max_rel_error(ref, got) -> float:
    """max_j |got_j - ref_j| / |ref_j|, with 0/0 := 0 (reading R6: lambda_j = 0 => psi_j = 0)."""
    ref = np.asarray(ref, dtype=np.float64)
    got = np.asarray(got, dtype=np.float64)
    diff = np.abs(got - ref)
    den = np.abs(ref)
    out = np.zeros_like(diff)
    nz = den > 0
    out[nz] = diff[nz] / den[nz]
    out[~nz & (diff > 0)] = np.inf
    return float(out.max()) if out.size else 0.0


def top_k(psi, k: int) -> np.ndarray:
    """Labels of the k largest psi, descending; ties by ascending label (reading R10)."""
    psi = np.asarray(psi)
    order = np.lexsort((np.arange(psi.size), -psi))
    return order[:k]
