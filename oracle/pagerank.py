"""PageRank power method, Eq. (22).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

    W = D_out^{-1} L            (L[j, i] = 1{j follows i}, D_out = out-degree |L(j)|)
    pi_t^T = alpha pi_{t-1}^T W + (1 - alpha)/N 1^T      (Eq. (22))
    stop when ||pi_t - pi_{t-1}||_1 <= eps               ("pi-tolerance")

The walk steps follower -> leader, so (pi^T W)_i = sum_{j in F(i)} pi_j / |L(j)|.
Rows of leaderless users are zero (no dangling redistribution, SPEC S:311,
reading R5): this is exactly the homogeneous A = alpha W of P:341, so that
psi = pi holds with the same W.

``pi0`` defaults to (1/N) 1; passing psi_0 = (c^T B + d^T)/N makes the iterates
equal Alg. 2's psi_t at every t (Eq. (21)).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def pagerank_power(row_ptr, followers, alpha: float, *, eps: float = 1e-12,
                   max_iters: int = 100_000, pi0=None, keep_iterates: bool = False):
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    followers = np.asarray(followers, dtype=np.int64)
    n = row_ptr.shape[0] - 1
    outdeg = np.bincount(followers, minlength=n).astype(np.float64)   # |L(j)|
    # W^T[i, j] = W[j, i] = 1/|L(j)| for j in F(i): same pattern as the input CSR.
    vals = 1.0 / outdeg[followers] if followers.size else np.zeros(0)
    WT = sp.csr_matrix((vals, followers, row_ptr), shape=(n, n))
    pi = np.full(n, 1.0 / n) if pi0 is None else np.array(pi0, dtype=np.float64)
    its = [pi.copy()] if keep_iterates else []
    t = 0
    gap = np.inf
    while gap > eps and t < max_iters:
        new = alpha * (WT @ pi) + (1.0 - alpha) / n
        gap = float(np.abs(new - pi).sum())
        pi = new
        t += 1
        if keep_iterates:
            its.append(pi.copy())
    return pi, t, its
