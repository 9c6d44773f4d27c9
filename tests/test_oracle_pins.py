"""Pins for the fp64 oracle (-m "not gpu").

Every check ties oracle/ to something other than itself: the SPEC's worked
examples (tests/golden/), analytic closed forms derived from the paper's
equations, the brute-force N-systems definition (Eqs. (1)-(5)), a dense LAPACK
solve of Eq. (12), networkx's PageRank, and the paper's invariants.  A
plausible slip in the oracle (dropped c^T term, A vs A^T, W over followers
instead of leaders, wrong norm, off-by-one in the iteration count, missing
1/N) fails at least one of them.
"""

import json
import os

import numpy as np
import pytest

import oracle
from oracle.operator import build_operator, norm_of_B
from oracle.nsystems import newsfeed_wall
from psigen import csr_from_edges

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _graph(case):
    rp, f = csr_from_edges(case["n"], case["edges"])
    return rp, f, np.array(case["lam"], float), np.array(case["mu"], float)


def random_graph(rng, n, p, leaderless_frac=0.1, mu0_frac=0.1, lam0_frac=0.0):
    """Random directed graph + activity with leaderless users, mu=0 and lam=0 users."""
    edges = [(i, j) for i in range(n) for j in range(n) if i != j and rng.random() < p]
    drop = set(rng.choice(n, size=int(leaderless_frac * n), replace=False).tolist())
    edges = [(i, j) for (i, j) in edges if i not in drop]          # users in drop lead only
    lam = rng.uniform(0.05, 1.0, n)
    mu = rng.uniform(0.05, 1.0, n)
    pick = rng.permutation(n)                      # disjoint mu=0 / lam=0 sets: lam+mu > 0
    n_mu0, n_lam0 = int(mu0_frac * n), int(lam0_frac * n)
    mu[pick[:n_mu0]] = 0.0
    lam[pick[n_mu0:n_mu0 + n_lam0]] = 0.0
    rp, f = csr_from_edges(n, edges)
    return rp, f, lam, mu


# ---------------------------------------------------------------- SPEC fixtures

@pytest.mark.parametrize("name", ["chain", "mutual", "cycle3_homogeneous", "edgeless"])
def test_spec_psi_fixtures(name):
    case = _gold("spec_examples.json")[name]
    rp, f, lam, mu = _graph(case)
    for norm in ("row", "col", "one"):
        r = oracle.power_psi(rp, f, lam, mu, eps=1e-14, norm=norm)
        np.testing.assert_allclose(r.psi, case["psi"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.psi_exact(rp, f, lam, mu), case["psi"], atol=1e-12)
    np.testing.assert_allclose(oracle.psi_nsystems(rp, f, lam, mu), case["psi"], atol=1e-12)
    if "psi_sum" in case:
        assert abs(r.psi.sum() - case["psi_sum"]) < 1e-12


@pytest.mark.parametrize("name", ["chain", "mutual"])
def test_spec_operator_fixtures(name):
    case = _gold("spec_examples.json")[name]
    rp, f, lam, mu = _graph(case)
    op = build_operator(rp, f, lam, mu)
    np.testing.assert_allclose(op["W"], case["W"], atol=1e-15)
    np.testing.assert_allclose(op["AT"] @ np.array(case["sTA_of"]), case["sTA"], atol=1e-15)
    np.testing.assert_allclose(op["BT"] @ np.array(case["sTB_of"]), case["sTB"], atol=1e-15)
    assert abs(norm_of_B(op["BT"], "col") - case["b_norm_col"]) < 1e-15
    if "c" in case:
        np.testing.assert_allclose(op["c"], case["c"])
        np.testing.assert_allclose(op["d"], case["d"])
    p, q = newsfeed_wall(rp, f, lam, mu, case["power_nf_origin"])
    np.testing.assert_allclose(p, case["p"], atol=1e-14)
    np.testing.assert_allclose(q, case["q"], atol=1e-14)


def test_spec_chain_converges_nilpotent():
    case = _gold("spec_examples.json")["chain"]
    rp, f, lam, mu = _graph(case)
    r = oracle.power_psi(rp, f, lam, mu, eps=1e-12)
    assert r.converged and r.iterations <= case["max_iters_to_converge"]
    # A^2 = 0: eps_2 = ||c^T A^2||_1 = 0 exactly, eps_1 = ||c^T A||_1 = 0.25
    assert r.history[0] == pytest.approx(0.25, abs=1e-15) and r.history[1] == 0.0


def test_spec_b_column_star():
    case = _gold("spec_examples.json")["star_homogeneous_b_column"]
    rp, f, lam, mu = _graph(case)
    A, B, c, d = oracle.dense_A_B(rp, f, lam, mu)
    np.testing.assert_allclose(B[:, 0], case["B_col0"], atol=1e-15)
    op = build_operator(rp, f, lam, mu)
    np.testing.assert_allclose(op["BT"].toarray(), B.T, atol=1e-15)   # sparse == dense build
    np.testing.assert_allclose(op["AT"].toarray(), A.T, atol=1e-15)


def test_edgeless_b_norm_zero():
    case = _gold("spec_examples.json")["edgeless"]
    rp, f, lam, mu = _graph(case)
    op = build_operator(rp, f, lam, mu)
    assert norm_of_B(op["BT"], "col") == 0.0 and norm_of_B(op["BT"], "row") == 0.0


# ------------------------------------------------------------- closed forms

def test_heterogeneous_cycle_closed_form():
    """j follows j+1 (mod N): u_j = sum_{k<N} prod_{m=1..k} c_{j-m} / (1 - prod c),
    psi = d * u / N (derived from Eq. (12) on the cycle)."""
    rng = np.random.default_rng(1)
    n = 7
    rp, f = csr_from_edges(n, [(j, (j + 1) % n) for j in range(n)])
    lam, mu = rng.uniform(0.05, 1, n), rng.uniform(0.05, 1, n)
    c, d = mu / (lam + mu), lam / (lam + mu)
    u = np.empty(n)
    for j in range(n):
        acc, prod = 0.0, 1.0
        for k in range(n):
            acc += prod
            prod *= c[(j - k - 1) % n]
        u[j] = acc / (1.0 - np.prod(c))
    want = d * u / n
    r = oracle.power_psi(rp, f, lam, mu, eps=0.0, max_iters=2000)
    np.testing.assert_allclose(r.psi, want, rtol=1e-13)
    np.testing.assert_allclose(oracle.psi_exact(rp, f, lam, mu), want, rtol=1e-13)


def test_star_closed_form_and_sum_rule():
    """Hub 0 leaderless, leaves follow only 0: psi_0 = d_0 (1 + sum c_i)/N, psi_i = d_i/N,
    sum psi = 1 - c_0 (1 + sum c_i)/N (Eq. (12) on the star)."""
    rng = np.random.default_rng(2)
    k = 9
    n = k + 1
    rp, f = csr_from_edges(n, [(i, 0) for i in range(1, n)])
    lam, mu = rng.uniform(0.05, 1, n), rng.uniform(0.05, 1, n)
    c, d = mu / (lam + mu), lam / (lam + mu)
    want = d / n
    want[0] = d[0] * (1 + c[1:].sum()) / n
    r = oracle.power_psi(rp, f, lam, mu, eps=1e-15)
    np.testing.assert_allclose(r.psi, want, rtol=1e-14)
    assert abs(r.psi.sum() - (1 - c[0] * (1 + c[1:].sum()) / n)) < 1e-14


def test_mu_zero_gives_uniform_and_edgeless_gives_d_over_n():
    rng = np.random.default_rng(3)
    rp, f, lam, _ = random_graph(rng, 20, 0.2)
    r = oracle.power_psi(rp, f, lam, np.zeros(20), eps=1e-15)
    np.testing.assert_allclose(r.psi, np.full(20, 1 / 20), rtol=1e-15)
    rp0, f0 = csr_from_edges(5, [])
    lam5, mu5 = rng.uniform(0.1, 1, 5), rng.uniform(0.1, 1, 5)
    r = oracle.power_psi(rp0, f0, lam5, mu5, eps=1e-15)
    np.testing.assert_allclose(r.psi, lam5 / (lam5 + mu5) / 5, rtol=1e-15)


# --------------------------------------------- the paper's main identity

@pytest.mark.parametrize("seed", range(50))
def test_nsystems_equals_single_system_equals_power_psi(seed):
    """Eqs. (1)-(5) solved N times (brute force) == Eq. (12) dense == Alg. 2 at convergence
    (P:209-259).  Graphs with leaderless users and mu = 0 users (R5, R6)."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(10, 65))
    p = float(rng.uniform(0.05, 0.3))
    rp, f, lam, mu = random_graph(rng, n, p, lam0_frac=0.05 if seed % 5 == 0 else 0.0)
    brute = oracle.psi_nsystems(rp, f, lam, mu)
    exact = oracle.psi_exact(rp, f, lam, mu)
    r = oracle.power_psi(rp, f, lam, mu, eps=0.0, max_iters=5000)
    np.testing.assert_allclose(exact, brute, rtol=1e-11, atol=1e-16)
    np.testing.assert_allclose(r.psi, brute, rtol=1e-11, atol=1e-16)


def test_config0_ER64_nsystems():
    """BASELINE.json config 1's 'N=64 subgraph' cross-check (reading R12)."""
    import psigen
    w = psigen.make_config(0)
    brute = oracle.psi_nsystems(w.row_ptr, w.followers, w.lam, w.mu)
    r = oracle.power_psi(w.row_ptr, w.followers, w.lam, w.mu, eps=w.eps)
    assert r.converged
    assert oracle.relative_error(brute, r.psi) < 1e-11
    assert abs(r.psi.sum() - 1.0) < 1e-11          # leader-complete => sum rule = 1


# ------------------------------------------------------------------ invariants

@pytest.mark.parametrize("seed", range(20))
def test_sum_rule_monotonicity_lower_bound(seed):
    """sum psi = 1 - (1/N) sum_{L(n) empty} s_n (derived from Eq. (12)); s_t, psi_t
    entrywise non-decreasing; psi >= d/N."""
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(10, 80))
    rp, f, lam, mu = random_graph(rng, n, float(rng.uniform(0.03, 0.3)), leaderless_frac=0.15)
    r = oracle.power_psi(rp, f, lam, mu, eps=0.0, max_iters=3000, keep_iterates=True)
    indeg = np.bincount(f, minlength=n)
    leaderless = indeg == 0
    assert abs(r.psi.sum() - (1 - r.s[leaderless].sum() / n)) < 1e-12
    for a, b in zip(r.s_iterates[:40], r.s_iterates[1:41]):
        assert np.all(b >= a - 1e-15 * np.abs(b))
    for a, b in zip(r.psi_iterates[:40], r.psi_iterates[1:41]):
        assert np.all(b >= a - 1e-15 * np.abs(b))
    d = lam / (lam + mu)
    assert np.all(r.psi >= d / n * (1 - 1e-15))


@pytest.mark.parametrize("seed", range(20))
def test_contraction_and_bound19(seed):
    """eps_{t+1} <= rho_A eps_t <= (max c) eps_t; delta_t <= eps_t kappa_row / N;
    truncation: 0 <= psi - psi_T, ||psi - psi_T||_1 <= kappa_row eps_T rho_A / (N (1 - rho_A))."""
    rng = np.random.default_rng(3000 + seed)
    n = int(rng.integers(10, 80))
    rp, f, lam, mu = random_graph(rng, n, float(rng.uniform(0.05, 0.3)))
    op = build_operator(rp, f, lam, mu)
    rho = float(np.asarray(op["AT"].sum(axis=0)).max()) if op["AT"].nnz else 0.0
    c = op["c"]
    assert rho <= c.max() + 1e-15
    r = oracle.power_psi(op=op, eps=1e-13, keep_iterates=True)
    h = r.history
    scale = max(np.abs(r.s).sum(), 1.0)
    for t in range(len(h) - 1):
        if h[t] > 1e-11 * scale:
            assert h[t + 1] <= rho * h[t] * (1 + 1e-9) + 1e-15
    kr = norm_of_B(op["BT"], "row")
    for t in range(1, len(r.psi_iterates)):
        delta = np.abs(r.psi_iterates[t] - r.psi_iterates[t - 1]).sum()
        assert delta <= h[t - 1] * kr / n * (1 + 1e-12) + 1e-17
    exact = oracle.psi_exact(rp, f, lam, mu)
    diff = exact - r.psi
    assert np.all(diff >= -1e-15)
    if rho < 1:
        assert diff.sum() <= kr * h[-1] * rho / (n * (1 - rho)) * (1 + 1e-6) + 1e-15


def test_kappa_col_counterexample():
    g = _gold("kappa_col_counterexample.json")
    rp, f, lam, mu = _graph(g)
    op = build_operator(rp, f, lam, mu)
    kc, kr = norm_of_B(op["BT"], "col"), norm_of_B(op["BT"], "row")
    tol = g["abs_tol"]
    assert abs(kc - g["kappa_col"]) < tol and abs(kr - g["kappa_row"]) < tol
    r = oracle.power_psi(op=op, eps=0.0, max_iters=1, keep_iterates=True)
    eps1 = r.history[0]
    delta1 = np.abs(r.psi_iterates[1] - r.psi_iterates[0]).sum()
    assert abs(eps1 - g["eps_1"]) < tol and abs(delta1 - g["delta_1"]) < tol
    n = g["n"]
    assert delta1 > eps1 * kc / n          # (19) with the column-sum norm fails
    assert delta1 <= eps1 * kr / n         # (19) with the row-sum norm holds


def test_scale_invariance_and_permutation_equivariance():
    rng = np.random.default_rng(7)
    n = 40
    rp, f, lam, mu = random_graph(rng, n, 0.15)
    base = oracle.power_psi(rp, f, lam, mu, eps=0.0, max_iters=500).psi
    scaled = oracle.power_psi(rp, f, 3.7 * lam, 3.7 * mu, eps=0.0, max_iters=500).psi
    np.testing.assert_allclose(scaled, base, rtol=1e-13)
    perm = rng.permutation(n)                           # new label of old user u = perm[u]
    edges = []
    for l in range(n):
        for j in f[rp[l]:rp[l + 1]]:
            edges.append((perm[j], perm[l]))
    rp2, f2 = csr_from_edges(n, edges)
    lam2, mu2 = np.empty(n), np.empty(n)
    lam2[perm], mu2[perm] = lam, mu
    out = oracle.power_psi(rp2, f2, lam2, mu2, eps=0.0, max_iters=500).psi
    np.testing.assert_allclose(out[perm], base, rtol=1e-13)


# ------------------------------------------------------- PageRank

@pytest.mark.parametrize("seed", range(10))
def test_homogeneous_psi_equals_pagerank_every_iteration(seed):
    """Eq. (21): with lam, mu constant, Alg. 2's psi_t are the PageRank iterates (22)
    started at pi_0 = psi_0, for every t."""
    rng = np.random.default_rng(4000 + seed)
    n = int(rng.integers(10, 60))
    rp, f, _, _ = random_graph(rng, n, float(rng.uniform(0.05, 0.3)))
    lam, mu = np.full(n, 0.15), np.full(n, 0.85)
    r = oracle.power_psi(rp, f, lam, mu, eps=0.0, max_iters=30, keep_iterates=True)
    _, _, its = oracle.pagerank_power(rp, f, 0.85, eps=0.0, max_iters=30,
                                      pi0=r.psi_iterates[0], keep_iterates=True)
    for t in range(31):
        np.testing.assert_allclose(r.psi_iterates[t], its[t], rtol=1e-13, atol=1e-17)


def test_homogeneous_psi_equals_networkx_pagerank():
    """psi = pi against networkx's PageRank on a leader-complete graph."""
    import networkx as nx
    import psigen
    rp, f = psigen.er_graph(300, 6.0, seed=5, fix_leaderless=True)
    n = 300
    lam, mu = np.full(n, 1.0), np.full(n, 1.0)
    r = oracle.power_psi(rp, f, lam, mu, eps=1e-15)
    G = nx.DiGraph()
    G.add_nodes_from(range(n))
    for l in range(n):
        for j in f[rp[l]:rp[l + 1]]:
            G.add_edge(int(j), l)                     # walk follower -> leader
    pr = nx.pagerank(G, alpha=0.5, tol=1e-15, max_iter=1000)
    np.testing.assert_allclose(r.psi, [pr[i] for i in range(n)], rtol=1e-10)
    pi, _, _ = oracle.pagerank_power(rp, f, 0.5, eps=1e-15)
    np.testing.assert_allclose(pi, r.psi, rtol=1e-12)


# ------------------------------------------------------------- config 1 at size

def test_config1_power_psi_vs_dense_exact():
    """C1 (N=10k) Alg. 2 at eps=1e-12 against the dense LAPACK solve of Eq. (12):
    within the truncation bound, and the exact fixed point is approached from below."""
    import psigen
    w = psigen.make_config(1)
    r = oracle.power_psi(w.row_ptr, w.followers, w.lam, w.mu, eps=w.eps)
    assert r.converged
    exact = oracle.psi_exact(w.row_ptr, w.followers, w.lam, w.mu)
    assert oracle.relative_error(exact, r.psi) < 1e-11
    assert oracle.max_rel_error(exact, r.psi) < 1e-10
    assert abs(r.psi.sum() - 1.0) < 1e-10


def test_metrics_pins():
    assert oracle.relative_error([3.0, 4.0], [3.0, 4.0]) == 0.0
    assert oracle.relative_error([3.0, 4.0], [0.0, 0.0]) == 1.0      # ||x||/||x||
    assert oracle.max_rel_error([0.0, 2.0], [0.0, 2.2]) == pytest.approx(0.1)
    assert list(oracle.top_k([0.1, 0.3, 0.3, 0.2], 3)) == [1, 2, 3]  # ties by label


# ------------------------------------------------------- Alg. 1 Power-NF

@pytest.mark.parametrize("name", ["chain", "mutual"])
def test_power_nf_spec_fixtures(name):
    """SPEC S:290-292 worked examples: per-origin p_i, q_i of Alg. 1 + Eq. (7)."""
    from oracle.power_nf import power_nf
    case = _gold("spec_examples.json")[name]
    rp, f, lam, mu = _graph(case)
    r = power_nf(rp, f, lam, mu, origin=case["power_nf_origin"], eps=1e-15)
    assert r.converged
    np.testing.assert_allclose(r.p, case["p"], atol=1e-14)
    np.testing.assert_allclose(r.q, case["q"], atol=1e-14)


def test_power_nf_edgeless_and_first_iterate():
    """b_i = 0 when nobody follows i: p = 0, q = d_i e_i; Alg. 1 line 1 (p <- b_i) with eps >= 1."""
    from oracle.power_nf import power_nf
    case = _gold("spec_examples.json")["edgeless"]
    rp, f, lam, mu = _graph(case)
    r = power_nf(rp, f, lam, mu, origin=2, eps=1e-12)
    assert np.all(r.p == 0)
    np.testing.assert_allclose(r.q, [0, 0, lam[2] / (lam[2] + mu[2])])
    rng = np.random.default_rng(9)
    rp, f, lam, mu = random_graph(rng, 20, 0.2)
    A, B, c, d = oracle.dense_A_B(rp, f, lam, mu)
    r = power_nf(rp, f, lam, mu, origin=3, eps=1.0)
    assert r.iterations == 0 and np.array_equal(r.p, B[:, 3])
    r = power_nf(rp, f, lam, mu, origin=3, eps=0.0, max_iters=2)   # p_2 = A(A b + b) + b
    np.testing.assert_allclose(r.p, A @ (A @ B[:, 3] + B[:, 3]) + B[:, 3], rtol=1e-14)


@pytest.mark.parametrize("seed", range(10))
def test_power_nf_converges_to_balance_equations(seed):
    """Alg. 1's fixed point is the solution of Eqs. (4)-(5) and (2)-(3) built from the leader
    sets (oracle.nsystems, independent of A, B); psi via N runs of Alg. 1 = Eq. (1) brute force
    = Alg. 2."""
    from oracle.power_nf import power_nf, psi_power_nf
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(8, 30))
    rp, f, lam, mu = random_graph(rng, n, float(rng.uniform(0.08, 0.3)))
    for i in (0, n // 2, n - 1):
        p_ex, q_ex = newsfeed_wall(rp, f, lam, mu, i)
        r = power_nf(rp, f, lam, mu, origin=i, eps=0.0, max_iters=3000)
        np.testing.assert_allclose(r.p, p_ex, rtol=1e-11, atol=1e-15)
        np.testing.assert_allclose(r.q, q_ex, rtol=1e-11, atol=1e-15)
        # p_t = sum_{tau<=t} A^tau b_i is non-decreasing (A, b >= 0)
        r2 = power_nf(rp, f, lam, mu, origin=i, eps=0.0, max_iters=5)
        r3 = power_nf(rp, f, lam, mu, origin=i, eps=0.0, max_iters=6)
        assert np.all(r3.p >= r2.p)
    psi, Ts = psi_power_nf(rp, f, lam, mu, eps=1e-14)
    np.testing.assert_allclose(psi, oracle.psi_nsystems(rp, f, lam, mu), rtol=1e-10, atol=1e-16)
    np.testing.assert_allclose(psi, oracle.power_psi(rp, f, lam, mu, eps=1e-15).psi, rtol=1e-10,
                               atol=1e-16)


# ------------------------------------------------ ingest scalars (psi_get_info)

@pytest.mark.parametrize("seed", range(12))
def test_graph_scalars_vs_dense_and_leader_sets(seed):
    """oracle.graph_scalars (kappa_row / kappa_col / rho_A / N_f / N_g / leaderless count, the
    values psi_get_info exports) against the dense entry-by-entry A, B of P:171-173
    (oracle.dense_A_B, an independent construction) and the brute-force leader sets; every row
    with a leader satisfies rowsum(A)_j + rowsum(B)_j = sum_{i in L(j)} w_i / W_j = 1."""
    rng = np.random.default_rng(4000 + seed)
    n = int(rng.integers(5, 60))
    rp, f, lam, mu = random_graph(rng, n, float(rng.uniform(0.02, 0.3)), leaderless_frac=0.2,
                                  lam0_frac=0.05 if seed % 3 == 0 else 0.0)
    op = build_operator(rp, f, lam, mu)
    sc = oracle.graph_scalars(op)
    A, B, c, d = oracle.dense_A_B(rp, f, lam, mu)
    assert sc["kappa_row"] == pytest.approx(B.sum(axis=1).max(), rel=1e-14, abs=0)
    assert sc["kappa_col"] == pytest.approx(B.sum(axis=0).max(), rel=1e-14, abs=0)
    assert sc["rho_A"] == pytest.approx(A.sum(axis=1).max(), rel=1e-14, abs=0)
    L = oracle.leader_sets(rp, f, n)
    has_lead = np.array([len(x) > 0 for x in L])
    assert sc["n_g"] == int(has_lead.sum()) and sc["n_leaderless"] == n - sc["n_g"]
    assert sc["n_f"] == sum(1 for l in range(n) if rp[l + 1] > rp[l])
    rs = A.sum(axis=1) + B.sum(axis=1)
    np.testing.assert_allclose(rs[has_lead], 1.0, rtol=1e-14)
    assert np.all(rs[~has_lead] == 0.0)
    assert sc["kappa_row"] <= 1.0 + 1e-15 and sc["rho_A"] <= c.max() + 1e-15


def test_graph_scalars_hand_values():
    """Chain 0 -> 1 (0 follows 1), lambda = (0.2, 0.6), mu = (0.3, 0.4): W_0 = 1.0, user 1
    leaderless; B[0,1] = 0.6, A[0,1] = 0.4 -- all norms read off by hand."""
    rp, f = csr_from_edges(2, [(0, 1)])
    op = build_operator(rp, f, np.array([0.2, 0.6]), np.array([0.3, 0.4]))
    sc = oracle.graph_scalars(op)
    assert sc == pytest.approx({"kappa_row": 0.6, "kappa_col": 0.6, "rho_A": 0.4, "n_f": 1,
                                "n_g": 1, "n_leaderless": 1}, abs=1e-16)


@pytest.mark.parametrize("chunk", [1, 3, 7, 61])
def test_edge_blocks_chunking_is_exact(monkeypatch, chunk):
    """oracle.operator streams huge edge arrays in blocks of ~_CHUNK edges of whole rows (the
    branch C4/C5 take with _CHUNK = 2^26).  Forcing tiny chunks -- rows longer than a chunk,
    many blocks -- must give the same W, A^T, B^T (vs their entry definitions) and psi as one
    block (up to the summation order of W), and psi must
    obey the sum rule sum psi = 1 - (1/N) sum_{L(n) empty} s_n (derived from Eq. (12))."""
    import oracle.operator as opmod
    rng = np.random.default_rng(77)
    n = 120
    rp, f, lam, mu = random_graph(rng, n, 0.12, leaderless_frac=0.1)
    hub = [(i, 0) for i in range(2, n) if i % 2 == 0]       # a row longer than any tiny chunk
    edges = [(int(j), int(l)) for l in range(n) for j in f[rp[l]:rp[l + 1]]]
    rp, f = csr_from_edges(n, sorted(set(edges) | set(hub)))
    base = build_operator(rp, f, lam, mu)
    r0 = oracle.power_psi(op=base, eps=0.0, max_iters=60)
    monkeypatch.setattr(opmod, "_CHUNK", chunk)
    blocks = list(opmod._edge_blocks(rp))
    assert len(blocks) > 1 and blocks[0][0] == 0 and blocks[-1][1] == len(f)
    assert all(b[1] == c[0] for b, c in zip(blocks, blocks[1:]))          # contiguous cover
    assert all(np.array_equal(b[2], np.repeat(np.arange(n), np.diff(rp))[b[0]:b[1]]) for b in blocks)
    op = build_operator(rp, f, lam, mu)
    # W_j = sum_{l in L(j)} (lambda_l + mu_l) written out with exactly rounded sums;
    # the blocked sums may associate differently, so equal up to rounding
    import math
    L = oracle.leader_sets(rp, f, n)
    W_def = np.array([math.fsum(lam[l] + mu[l] for l in L[j]) for j in range(n)])
    np.testing.assert_allclose(op["W"], W_def, rtol=4e-16 * n, atol=0)
    np.testing.assert_allclose(op["W"], base["W"], rtol=4e-16 * n, atol=0)
    rows = np.repeat(np.arange(n), np.diff(rp))
    Wd = np.where(W_def > 0, W_def, 1.0)
    np.testing.assert_allclose(op["AT"].data, mu[rows] / Wd[f], rtol=1e-14)     # A[j,i] = mu_i/W_j
    np.testing.assert_allclose(op["BT"].data, lam[rows] / Wd[f], rtol=1e-14)    # B[j,i] = lam_i/W_j
    assert np.array_equal(op["AT"].indices, base["AT"].indices)
    r1 = oracle.power_psi(op=op, eps=0.0, max_iters=60)
    np.testing.assert_allclose(r1.psi, r0.psi, rtol=1e-13)
    leaderless = np.bincount(f, minlength=n) == 0
    r2 = oracle.power_psi(op=op, eps=0.0, max_iters=4000)
    assert abs(r2.psi.sum() - (1 - r2.s[leaderless].sum() / n)) < 1e-12
