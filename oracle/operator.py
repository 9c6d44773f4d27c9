"""The model matrices A, B and vectors c, d of PAPER.md §II.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Input convention (reading R8, "(i,j) in E encodes that user i follows
user j"): a CSR whose row ``j`` lists F(j), the *followers* of leader ``j``::

    row_ptr  int64[N+1]   row_ptr[0] = 0, row_ptr[N] = M
    followers int32[M]    followers[row_ptr[j]:row_ptr[j+1]] = F(j)

so edge (n, j) in E  <=>  n in F(j)  <=>  j in L(n).

The paper's matrices, written out entry by entry:

    A[j, i] = mu_i     / W_j * 1{i in L(j)}
    B[j, i] = lambda_i / W_j * 1{i in L(j)}       (column i of B is b_i)
    W_j     = sum_{l in L(j)} (lambda_l + mu_l)   (the newsfeed normaliser)
    c_j     = mu_j / (lambda_j + mu_j)            (diag of C)
    d_j     = lambda_j / (lambda_j + mu_j)        (diag of D)

Leaderless users (W_j = 0, reading R5): rows j of A and B are zero.

The oracle stores A and B *transposed* with an explicit value per edge
(``AT[i, j] = A[j, i]``), because Alg. 2 only ever multiplies row vectors from
the left (s^T A, s^T B), and ``AT @ s`` is then a plain SciPy CSR mat-vec over
exactly the input's sparsity pattern (row i = leader i, columns F(i)).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

_CHUNK = 1 << 26  # edges per chunk when streaming over huge edge arrays


def _edge_blocks(row_ptr: np.ndarray):
    """Yield (lo, hi, rows): edge range [lo, hi) of whole rows and the leader
    (row) index of every edge in it, ~_CHUNK edges at a time."""
    n = row_ptr.shape[0] - 1
    r0 = 0
    while r0 < n:
        target = row_ptr[r0] + _CHUNK
        r1 = int(np.searchsorted(row_ptr, target, side="right")) - 1
        r1 = min(max(r1, r0 + 1), n)
        lo, hi = int(row_ptr[r0]), int(row_ptr[r1])
        rows = np.repeat(np.arange(r0, r1, dtype=np.int64), np.diff(row_ptr[r0:r1 + 1]))
        yield lo, hi, rows
        r0 = r1


def newsfeed_normaliser(row_ptr, followers, lam, mu) -> np.ndarray:
    """W_j = sum_{l in L(j)} (lambda_l + mu_l)  (denominators of A, B).

    Each edge (leader l -> follower j) adds w_l to W_j; np.bincount sums the
    edges of each follower in increasing edge (= leader) order.
    """
    n = lam.shape[0]
    m = followers.shape[0]
    w = lam + mu
    W = np.zeros(n, dtype=np.float64)
    for lo, hi, rows in _edge_blocks(row_ptr):
        W += np.bincount(followers[lo:hi], weights=w[rows], minlength=n)
    return W


def build_operator(row_ptr, followers, lam, mu, with_B: bool = True) -> dict:
    """Explicit A^T, B^T (SciPy CSR, fp64 per-edge values), c, d, W.

    ``with_B=False`` skips B^T (the large-graph path builds it after the loop
    by reusing A^T's index arrays, see ``power_psi``).
    """
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    followers = np.asarray(followers, dtype=np.int32)
    lam = np.asarray(lam, dtype=np.float64)
    mu = np.asarray(mu, dtype=np.float64)
    n = lam.shape[0]
    m = followers.shape[0]
    W = newsfeed_normaliser(row_ptr, followers, lam, mu)
    w = lam + mu
    c = mu / w
    d = lam / w
    # int32 index arrays when they fit, so SciPy does not copy 4M bytes.
    idx_t = np.int32 if m < 2**31 - 1 else np.int64
    indptr = row_ptr.astype(idx_t)
    indices = followers.astype(idx_t, copy=False)
    a_val = np.empty(m, dtype=np.float64)
    for lo, hi, rows in _edge_blocks(row_ptr):
        a_val[lo:hi] = mu[rows] / W[followers[lo:hi]]     # A[j,i] = mu_i / W_j
    AT = sp.csr_matrix((a_val, indices, indptr), shape=(n, n), copy=False)
    op = {"n": n, "m": m, "W": W, "c": c, "d": d, "lam": lam, "mu": mu,
          "AT": AT, "row_ptr": row_ptr, "followers": followers}
    if with_B:
        op["BT"] = B_transpose(op)
    return op


def B_transpose(op: dict, out: np.ndarray | None = None):
    """B^T with B[j, i] = lambda_i / W_j * 1{i in L(j)}.

    ``out`` may be A^T's value array, reused in place to save memory.
    """
    row_ptr, followers = op["row_ptr"], op["followers"]
    lam, W = op["lam"], op["W"]
    m = followers.shape[0]
    b_val = np.empty(m, dtype=np.float64) if out is None else out
    for lo, hi, rows in _edge_blocks(row_ptr):
        b_val[lo:hi] = lam[rows] / W[followers[lo:hi]]
    AT = op["AT"]
    return sp.csr_matrix((b_val, AT.indices, AT.indptr), shape=AT.shape, copy=False)


def norm_of_B(BT, which: str = "row") -> float:
    """The B_norm of Alg. 2 line 2; the paper leaves the norm open.

    * ``"row"`` (default, reading R1): max row sum of B,
      max_j sum_{i in L(j)} lambda_i / W_j -- the operator norm induced by the
      L1 norm on *row* vectors, which is what (18)-(19) multiply.
    * ``"col"``: max column sum of B (SPEC's induced 1-norm reading).
    * ``"one"``: 1 (ignore the factor).
    B >= 0 entrywise, so the absolute sums are plain sums.
    """
    if which == "one":
        return 1.0
    if BT.nnz == 0:
        return 0.0
    if which == "row":        # rows of B  = columns of B^T
        return float(np.asarray(BT.sum(axis=0)).max())
    if which == "col":        # columns of B = rows of B^T
        return float(np.asarray(BT.sum(axis=1)).max())
    raise ValueError(f"unknown norm {which!r}")


def graph_scalars(op: dict) -> dict:
    """The per-graph scalars that the ingest reports (``psi_get_info``), from the explicit
    operator:

    * ``kappa_row`` = ||B|| read as the max row sum of B (Alg. 2 line 2; reading R1),
      ``kappa_col`` = the max column sum of B (SPEC's reading) -- both via ``norm_of_B``;
    * ``rho_A`` = the max row sum of A, max_j sum_{i in L(j)} mu_i / W_j: the
      contraction factor of Eq. (14)'s residual recursion, < 1 under the convergence
      condition (reading R14);
    * ``n_f`` = users with >= 1 follower (a non-empty row of the input CSR),
      ``n_g`` = users with >= 1 leader (j in F(l) for some l), ``n_leaderless`` = N - n_g
      (W_j = 0, reading R5).
    """
    row_ptr, followers, n = op["row_ptr"], op["followers"], op["n"]
    BT = op.get("BT")
    if BT is None:
        BT = B_transpose(op)
    n_g = int(np.count_nonzero(np.bincount(followers, minlength=n)))
    return {"kappa_row": norm_of_B(BT, "row"), "kappa_col": norm_of_B(BT, "col"),
            "rho_A": norm_of_B(op["AT"], "row"),
            "n_f": int(np.count_nonzero(np.diff(row_ptr))), "n_g": n_g, "n_leaderless": n - n_g}


def leader_sets(row_ptr, followers, n) -> list[list[int]]:
    """L(j) for every user j (small graphs only): j in F(l)  <=>  l in L(j)."""
    L: list[list[int]] = [[] for _ in range(n)]
    for l in range(n):
        for j in followers[row_ptr[l]:row_ptr[l + 1]]:
            L[int(j)].append(l)
    return L
