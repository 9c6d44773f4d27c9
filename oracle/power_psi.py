"""Alg. 2 "Power-psi", literally, in fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

    Input: N, A, B, c, d, s-tolerance eps
    s <- c                                                        (s_0 = c, Eq. (14))
    B_norm <- ||B||                                               (reading R1)
    t <- 0 ; gap <- 1
    while gap > eps:
        s_old <- s
        s^T <- s_old^T A + c^T                                    (Eq. (14); reading R2)
        gap <- B_norm * ||s_old - s||_1                           (L1 per P:282)
        t <- t + 1
    psi^T <- (1/N) (s^T B + d^T)                                  (Eq. (12))

Additions that the paper leaves to the implementation (DESIGN.md readings):

* ``max_iters`` safety cap (R3/SPEC S:278): the loop also stops at t = max_iters
  and the result says ``converged=False``. ``eps = 0`` therefore runs exactly
  ``max_iters`` sweeps unless the fp iteration reaches an exact fixed point
  first (gap == 0 is not > 0, so Alg. 2 stops), which is the fixed-count parity
  mode.
* ``history[t-1] = ||s_t - s_{t-1}||_1`` (Eq. (15), the raw epsilon_t, not
  multiplied by B_norm).
* ``keep_iterates=True`` also returns every s_t and psi_t (psi_t is Eq. (12)
  with s replaced by s_t, the "psi_t" of P:288), for the bound (19) and the
  homogeneous per-iteration pins.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .operator import build_operator, norm_of_B, B_transpose


@dataclass
class PowerPsiResult:
    psi: np.ndarray
    iterations: int                 # T: number of s-updates (A products), reading R4
    history: list                   # epsilon_t, t = 1..T (Eq. (15))
    converged: bool
    b_norm: float
    s: np.ndarray                   # s_T
    s_iterates: list = field(default_factory=list)
    psi_iterates: list = field(default_factory=list)


def power_psi(row_ptr=None, followers=None, lam=None, mu=None, *, op: dict | None = None,
              eps: float = 1e-9, max_iters: int = 100_000, norm: str = "row",
              keep_iterates: bool = False) -> PowerPsiResult:
    """Run Alg. 2 on the follower graph (CSR of followers per leader) + activity."""
    if op is None:
        op = build_operator(row_ptr, followers, lam, mu, with_B=True)
    AT = op["AT"]
    BT = op.get("BT")
    if BT is None:
        BT = B_transpose(op)
        op["BT"] = BT
    c, d, n = op["c"], op["d"], op["n"]

    s = c.copy()                                        # s <- c
    b_norm = norm_of_B(BT, norm)                        # B_norm <- ||B||
    t = 0
    gap = 1.0
    history: list[float] = []
    s_its = [s.copy()] if keep_iterates else []
    psi_its = [(BT @ s + d) / n] if keep_iterates else []
    while gap > eps and t < max_iters:
        s_old = s
        s = AT @ s_old + c                              # s^T <- s_old^T A + c^T
        eps_t = float(np.abs(s_old - s).sum())          # ||s_old - s||_1
        history.append(eps_t)
        gap = b_norm * eps_t
        t += 1
        if keep_iterates:
            s_its.append(s.copy())
            psi_its.append((BT @ s + d) / n)
    psi = (BT @ s + d) / n                              # psi^T <- (s^T B + d^T)/N
    return PowerPsiResult(psi=psi, iterations=t, history=history,
                          converged=bool(gap <= eps), b_norm=b_norm, s=s,
                          s_iterates=s_its, psi_iterates=psi_its)
