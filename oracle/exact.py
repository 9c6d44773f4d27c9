"""The exact limit of Power-psi: Eq. (12) with the Neumann series summed.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

    psi^T = (1/N) [ c^T (I - A)^{-1} B + d^T ]                (Eq. (12) with (10)-(11))

i.e. solve (I - A)^T s = c densely (LAPACK, partial pivoting) and read out
psi = (B^T s + d) / N.  A and B are materialised densely from their entry
definitions, independently of ``operator.build_operator``'s sparse
per-edge construction.  Dense, so N up to ~1.2e4 (config 1).
"""

from __future__ import annotations

import numpy as np


def dense_A_B(row_ptr, followers, lam, mu):
    """Dense A, B, c, d from P:171-175 (rows j, columns i; i in L(j) <=> j in F(i))."""
    lam = np.asarray(lam, dtype=np.float64)
    mu = np.asarray(mu, dtype=np.float64)
    n = lam.shape[0]
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    followers = np.asarray(followers, dtype=np.int64)
    leader = np.repeat(np.arange(n), np.diff(row_ptr))     # edge (follower j -> leader i)
    Lind = np.zeros((n, n))                                # Lind[j, i] = 1{i in L(j)}
    Lind[followers, leader] = 1.0
    W = Lind @ (lam + mu)                                  # sum_{l in L(j)} (lam_l + mu_l)
    Wsafe = np.where(W > 0, W, 1.0)                        # leaderless rows stay 0 (R5)
    A = Lind * mu[None, :] / Wsafe[:, None]
    B = Lind * lam[None, :] / Wsafe[:, None]
    c = mu / (lam + mu)
    d = lam / (lam + mu)
    return A, B, c, d


def psi_exact(row_ptr, followers, lam, mu) -> np.ndarray:
    A, B, c, d = dense_A_B(row_ptr, followers, lam, mu)
    n = c.shape[0]
    s = np.linalg.solve((np.eye(n) - A).T, c)             # s^T = c^T (I - A)^{-1}
    return (B.T @ s + d) / n
