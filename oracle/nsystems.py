"""The psi-score from its original definition: N linear systems (§II).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

For every origin i ("posts of origin i") this builds the newsfeed
balance equations straight from Eqs. (4)-(5), using the leader
sets L(j) and the activities -- *not* the matrices A, B of P:171-173 -- solves
them densely (LAPACK), maps p_i to the wall shares q_i with Eqs. (2)-(3)
 and averages by Eq. (1):

  (4)  j != i:  sum_{k in L(j)} (lam_k + mu_k) p^(j) = lam_i 1{i in L(j)} + sum_{k in L(j)} mu_k p^(k)
  (5)  j == i:  sum_{k in L(i)} (lam_k + mu_k) p^(i) = sum_{k in L(i)} mu_k p^(k)
  (2)  n != i:  (lam_n + mu_n) q^(n) = mu_n p^(n)
  (3)  n == i:  (lam_i + mu_i) q^(i) = lam_i + mu_i p^(i)
  (1)  psi_i = (1/N) sum_n q_i^(n)

Reading R5 (leaderless users, L(j) empty): Eq. (4) degenerates to 0 = 0; the
newsfeed of j stays empty, p^(j) = 0.

Cost O(N^4): brute force for N <= ~64, which is its purpose (the paper's
"N linear systems of size N").
"""

from __future__ import annotations

import numpy as np

from .operator import leader_sets


def newsfeed_wall(row_ptr, followers, lam, mu, i: int):
    """(p_i, q_i) for origin i from Eqs. (4)-(5) then (2)-(3)."""
    lam = np.asarray(lam, dtype=np.float64)
    mu = np.asarray(mu, dtype=np.float64)
    n = lam.shape[0]
    L = leader_sets(row_ptr, followers, n)
    M = np.zeros((n, n))
    rhs = np.zeros(n)
    for j in range(n):
        if not L[j]:                       # R5: empty newsfeed
            M[j, j] = 1.0
            continue
        M[j, j] += sum(lam[k] + mu[k] for k in L[j])
        for k in L[j]:
            M[j, k] -= mu[k]
        if j != i and i in L[j]:           # Eq. (4) source term; Eq. (5) has none
            rhs[j] = lam[i]
    p = np.linalg.solve(M, rhs)
    q = mu * p / (lam + mu)                # Eq. (2)
    q[i] = (lam[i] + mu[i] * p[i]) / (lam[i] + mu[i])   # Eq. (3)
    return p, q


def psi_nsystems(row_ptr, followers, lam, mu) -> np.ndarray:
    """psi by Eq. (1) over all N origins (each one a dense solve)."""
    n = len(lam)
    psi = np.empty(n)
    for i in range(n):
        _, q = newsfeed_wall(row_ptr, followers, lam, mu, i)
        psi[i] = q.sum() / n
    return psi
