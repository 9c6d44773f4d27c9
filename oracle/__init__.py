"""fp64 CPU oracle for Power-psi (arXiv 2206.09960) -- TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct statement of what the
B200 hot path computes. It exists to prove the CUDA path right; it is never
part of that path.

Rules ("Oracle"):

* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import anything in here.
  The product package ``paper_2206_09960_b200`` never does, and it fails
  loudly when its CUDA library is missing (there is no CPU fallback).
* It shares no code with the CUDA path: no kernels, headers, helpers,
  tables or constant generators.  Both sides only consume the same seeded
  input arrays, produced by the separate ``psigen`` module (which holds none
  of the method's arithmetic).
* Every function cites the passage of ``PAPER.md`` (P:line) it follows.
  Readings where the paper is silent or ambiguous are listed in DESIGN.md
  ("Readings of the paper") and referenced here as R1..R14.
* Floating point is fp64 throughout; library primitives used as single steps
  are SciPy's CSR mat-vec, NumPy's bincount and LAPACK's dense solve.

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``) tie every function here to
something other than itself: the SPEC/paper worked examples
(tests/golden/), closed forms (cycle, star, chain, mu == 0, edgeless), the
brute-force N-systems solve of Eqs. (2)-(5), networkx's PageRank, and the
paper's invariants (sum rule, monotonicity, contraction, bound (19)).
No function in this package is "parity unpinned".
"""

from .operator import build_operator, graph_scalars, leader_sets, norm_of_B
from .power_psi import power_psi, PowerPsiResult
from .nsystems import psi_nsystems
from .exact import psi_exact, dense_A_B
from .pagerank import pagerank_power
from .power_nf import power_nf, psi_power_nf, PowerNFResult
from .metrics import relative_error, max_rel_error, top_k

__all__ = [
    "build_operator", "graph_scalars", "leader_sets", "norm_of_B", "power_psi", "PowerPsiResult",
    "psi_nsystems", "psi_exact", "dense_A_B", "pagerank_power", "power_nf", "psi_power_nf",
    "PowerNFResult",
    "relative_error", "max_rel_error", "top_k",
]
