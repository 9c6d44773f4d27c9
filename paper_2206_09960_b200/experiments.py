"""Experiments 1-2 of the paper (§V) on the GPU path: SURVEY §8(f) row 3.

For each method and each tolerance eps of a decade grid ("from 10^-9 to 10^-1") the
sweep records the number of matrix-vector multiplications, the iterations, the device time and
the relative error of Eq. (23) against a reference psi:

* ``power_psi``  -- Alg. 2, s-tolerance eps; matvecs = T + 1 (T products with A, one with B);
* ``power_nf``   -- Alg. 1 for every origin + Eq. (1) (psi_nsystems), p-tolerance eps;
  matvecs = sum_i T_i;
* ``pagerank``   -- Eq. (22) with alpha = mu/(lambda + mu), pi-tolerance eps; matvecs = T;
  only meaningful for homogeneous activity, where psi = pi.

Fig. 4-5 plot matvecs against the achieved error, not against eps: Power-psi's s-tolerance is
an N-scaled quantity (bound (19): delta_t <= eps_t ||B|| / N) while PageRank's
pi-tolerance is not, so equal eps is not equal precision.  ``error_curve`` therefore runs
each method for a fixed number of sweeps t (eps = 0, max_iters = t) and records
(matvecs, error) -- the curve of Fig. 4-5 -- and ``matvecs_to_reach`` reads it at a target
error.

The reference is Power-psi at eps = 1e-14 on the same context ("tightest run" when
the exact solve is infeasible); tests/test_gpu_experiments.py pins it to the oracle's dense
exact solve of Eq. (12).  Every number comes from the C-ABI library (no CPU path).
"""

from __future__ import annotations

import numpy as np

DEFAULT_TOLS = [10.0 ** -k for k in range(1, 10)]


def relative_error(ref: np.ndarray, approx: np.ndarray) -> float:
    """Eq. (23): ||psi_true - psi_eps||_2 / ||psi_true||_2."""
    return float(np.linalg.norm(ref - approx) / np.linalg.norm(ref))


def tolerance_sweep(graph, methods=("power_psi", "power_nf"), tols=DEFAULT_TOLS, alpha=None,
                    reference_eps: float = 1e-14, max_iters: int = 100_000):
    """Rows (method, eps, matvecs, iterations, ms, error, converged) on an open PsiGraph."""
    import torch
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn):
        torch.cuda.synchronize()
        ev0.record()
        r = fn()
        ev1.record()
        torch.cuda.synchronize()
        return r, ev0.elapsed_time(ev1)

    graph.iterate(reference_eps, max_iters)
    ref = graph.get_psi().cpu().numpy()
    rows = []
    for m in methods:
        for eps in tols:
            if m == "power_psi":
                (st, T, _), ms = timed(lambda: graph.iterate(eps, max_iters))
                approx = graph.get_psi().cpu().numpy()
                mv, it = T + 1, T
            elif m == "power_nf":
                (st, approx_t, mv), ms = timed(lambda: graph.nsystems(eps, max_iters))
                approx = approx_t.cpu().numpy()
                it = mv
            elif m == "pagerank":
                if alpha is None:
                    raise ValueError("pagerank needs alpha = mu/(lambda+mu) (homogeneous activity)")
                (st, T, _), ms = timed(lambda: graph.pagerank(alpha, eps, max_iters))
                approx = graph.get_pagerank().cpu().numpy()
                mv, it = T, T
            else:
                raise ValueError(f"unknown method {m!r}")
            rows.append({"method": m, "eps": eps, "matvecs": int(mv), "iterations": int(it),
                         "ms": round(float(ms), 4), "error": relative_error(ref, approx),
                         "converged": st == 0})
    return rows, ref


def error_curve(graph, method: str, ts, alpha=None, reference=None, reference_eps: float = 1e-14):
    """[(t, matvecs, error)] for fixed-count runs of `method` with t = each entry of `ts`."""
    if reference is None:
        graph.iterate(reference_eps)
        reference = graph.get_psi().cpu().numpy()
    out = []
    for t in ts:
        if method == "power_psi":
            graph.iterate(0.0, t)
            approx, mv = graph.get_psi().cpu().numpy(), t + 1
        elif method == "pagerank":
            graph.pagerank(alpha, 0.0, t)
            approx, mv = graph.get_pagerank().cpu().numpy(), t
        elif method == "power_nf":
            _, approx_t, mv = graph.nsystems(0.0, t)
            approx = approx_t.cpu().numpy()
        else:
            raise ValueError(f"unknown method {method!r}")
        out.append((int(t), int(mv), relative_error(reference, approx)))
    return out


def matvecs_to_reach(curve, target: float):
    """Fewest matvecs on an error curve with error <= target (None if never reached)."""
    hits = [mv for (_, mv, err) in curve if err <= target]
    return min(hits) if hits else None


def to_csv(rows, header: str = "") -> str:
    lines = [f"# {h}" for h in header.splitlines() if h]
    lines.append("method,tolerance,matvecs,iterations,ms,error,converged")
    for r in rows:
        lines.append(f"{r['method']},{r['eps']:.0e},{r['matvecs']},{r['iterations']},{r['ms']},"
                     f"{r['error']:.6e},{int(r['converged'])}")
    return "\n".join(lines) + "\n"
