"""Alg. 1 "Power-NF" and the N-systems psi it yields, literally, in fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Per origin i:

    p_i <- b_i ; t <- 0 ; gap <- 1                                (Alg. 1 lines 1-3)
    while gap > eps:                                              (line 4)
        p_old <- p_i ; p_i <- A p_old + b_i                       (lines 5-6; Eq. (8))
        gap <- ||p_i - p_old||_1 ; t <- t + 1                      (lines 7-8; L1 as in SPEC S:286)
    q_i = C p_i + d_i                                             (Eq. (7))
    psi_i = (1/N) sum_n q_i^(n)                                   (Eq. (1))

with A[j, l] = mu_l / W_j 1{l in L(j)}, b_i[j] = lambda_i / W_j 1{i in L(j)}, C = diag(c),
d_i = d_i e_i.  A is the *column* (right) product here -- the transpose of the
row-vector products of Alg. 2 -- so this module builds A itself from the leader sets (via
operator.build_operator's explicit A^T, transposed), with a max_iters cap (reading R3).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .operator import build_operator


@dataclass
class PowerNFResult:
    p: np.ndarray
    q: np.ndarray
    iterations: int
    history: list = field(default_factory=list)
    converged: bool = True


def _A_and_b(op: dict, i: int):
    """A (CSR, rows j) = (A^T)^T and the column b_i of B."""
    A = op["AT"].T.tocsr()                      # A[j, l] = mu_l / W_j for l in L(j)
    b = np.asarray(op["BT"][i].todense()).ravel()   # row i of B^T = column i of B
    return A, b


def power_nf(row_ptr=None, followers=None, lam=None, mu=None, origin: int = 0, *,
             op: dict | None = None, eps: float = 1e-9, max_iters: int = 100_000,
             keep_history: bool = True) -> PowerNFResult:
    if op is None:
        op = build_operator(row_ptr, followers, lam, mu, with_B=True)
    A, b = _A_and_b(op, origin)
    c, d = op["c"], op["d"]
    p = b.copy()                                # p_i <- b_i
    t, gap, hist = 0, 1.0, []
    while gap > eps and t < max_iters:
        p_old = p
        p = A @ p_old + b                       # p_i <- A p_old + b_i
        gap = float(np.abs(p - p_old).sum())
        hist.append(gap)
        t += 1
    q = c * p                                   # q_i = C p_i + d_i
    q[origin] += d[origin]
    return PowerNFResult(p=p, q=q, iterations=t, history=hist if keep_history else [],
                         converged=bool(gap <= eps))


def psi_power_nf(row_ptr, followers, lam, mu, *, eps: float = 1e-9, max_iters: int = 100_000):
    """psi by N runs of Alg. 1 (the paper's N-systems baseline); returns (psi, T_i)."""
    op = build_operator(row_ptr, followers, lam, mu, with_B=True)
    n = op["n"]
    psi = np.empty(n)
    Ts = np.empty(n, dtype=np.int64)
    for i in range(n):
        r = power_nf(op=op, origin=i, eps=eps, max_iters=max_iters, keep_history=False)
        psi[i] = r.q.sum() / n
        Ts[i] = r.iterations
    return psi, Ts
