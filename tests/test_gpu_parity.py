"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle (-m gpu).

Parity protocol:
  1. the oracle runs Alg. 2 to eps and records T*, eps_t, psi;
  2. the GPU runs psi_iterate(eps=0, max_iters=T*) (fixed count) -> max relative
     error per psi entry <= 1e-10 (north_star), same top-k (ties R10);
  3. the GPU runs psi_iterate(eps) -> |T_gpu - T*| <= 1 and matching eps_t histories.
"""

import numpy as np
import pytest

import oracle
import psigen

pytestmark = pytest.mark.gpu

TOL = 1e-10          # north_star: max relative error per psi entry, fp64


def to_dev(*arrays):
    import torch
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrays]


def gpu_run(psi, rp, f, lam, mu, eps, max_iters=100_000, norm="row", host=False):
    import torch
    args = (rp, f, lam, mu) if host else to_dev(rp, f, lam, mu)
    with psi.PsiGraph(*args) as g:
        st, T, gap = g.iterate(eps, max_iters, norm)
        out = g.get_psi().cpu().numpy()
        s = g.get_series().cpu().numpy()
        hist = g.get_residual_history()
        info = g.info()
    torch.cuda.synchronize()
    return dict(psi=out, T=T, gap=gap, status=st, hist=hist, s=s, info=info)


def check_topk(ref, got, ks=(10, 100, 1000)):
    """Same top-k; pairs within 1e-10 relative may swap (reading R10)."""
    for k in ks:
        k = min(k, ref.size)
        a, b = oracle.top_k(ref, k), oracle.top_k(got, k)
        if np.array_equal(a, b):
            continue
        # allowed only for near-ties at the boundary / inside
        diff = set(a.tolist()) ^ set(b.tolist())
        kth = np.sort(ref)[::-1][k - 1]
        for j in diff:
            assert abs(ref[j] - kth) <= 1e-10 * kth, (k, j)
        for x, y in zip(a, b):
            if x != y:
                assert abs(ref[x] - ref[y]) <= 1e-10 * max(ref[x], ref[y]), (k, x, y)


def check_scalars(op, info):
    """The ingest's scalars (psi_get_info) against the oracle's (oracle.graph_scalars):
    ||B|| by rows / columns (Alg. 2 line 2; reading R1), rho_A (the convergence
    factor, R14) to 1e-12 relative; N_f, N_g and the leaderless count exactly."""
    sc = oracle.graph_scalars(op)
    for k in ("kappa_row", "kappa_col", "rho_A"):
        assert abs(info[k] - sc[k]) <= 1e-12 * abs(sc[k]), (k, info[k], sc[k])
    for k in ("n_f", "n_g", "n_leaderless"):
        assert info[k] == sc[k], (k, info[k], sc[k])


def parity(psi, w, norm="row", eps=None, full=True):
    eps = w.eps if eps is None else eps
    op = oracle.build_operator(w.row_ptr, w.followers, w.lam, w.mu)
    ref = oracle.power_psi(op=op, eps=eps, norm=norm)
    got = gpu_run(psi, w.row_ptr, w.followers, w.lam, w.mu, 0.0, ref.iterations, norm)
    check_scalars(op, got["info"])
    del op
    assert got["T"] == ref.iterations
    err = oracle.max_rel_error(ref.psi, got["psi"])
    assert err <= TOL, err
    assert oracle.relative_error(ref.psi, got["psi"]) <= TOL
    check_topk(ref.psi, got["psi"])
    assert oracle.max_rel_error(ref.s, got["s"]) <= TOL
    if full:
        g2 = gpu_run(psi, w.row_ptr, w.followers, w.lam, w.mu, eps, 10 * ref.iterations + 10, norm)
        assert abs(g2["T"] - ref.iterations) <= 1, (g2["T"], ref.iterations)
        h_ref = np.array(ref.history)
        k = min(len(h_ref), len(g2["hist"]))
        s1 = np.abs(ref.s).sum()
        np.testing.assert_allclose(g2["hist"][:k], h_ref[:k], rtol=1e-6, atol=1e-13 * s1)
    return ref, got


# ---------------------------------------------------------------- fixtures


@pytest.mark.parametrize("name", ["chain", "mutual", "cycle3_homogeneous", "edgeless"])
def test_spec_fixtures_on_gpu(gpu, name, driver):
    import json, os
    case = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                       "spec_examples.json")))[name]
    rp, f = psigen.csr_from_edges(case["n"], case["edges"])
    lam, mu = np.array(case["lam"]), np.array(case["mu"])
    got = gpu_run(gpu, rp, f, lam, mu, 1e-14)
    np.testing.assert_allclose(got["psi"], case["psi"], rtol=0, atol=1e-12)
    if "psi_sum" in case:
        assert abs(got["psi"].sum() - case["psi_sum"]) < 1e-12


def test_chain_iteration_count_and_history(gpu, driver):
    rp, f = psigen.csr_from_edges(2, [(0, 1)])
    got = gpu_run(gpu, rp, f, np.array([0.5, 0.5]), np.array([0.5, 0.5]), 1e-12)
    assert got["T"] == 2 and got["hist"][0] == pytest.approx(0.25, abs=1e-15) and got["hist"][1] == 0
    np.testing.assert_allclose(got["s"], [0.5, 0.75], atol=1e-15)


def test_heterogeneous_cycle_and_star_closed_forms(gpu, driver):
    rng = np.random.default_rng(11)
    n = 9
    rp, f = psigen.csr_from_edges(n, [(j, (j + 1) % n) for j in range(n)])
    lam, mu = rng.uniform(0.05, 1, n), rng.uniform(0.05, 1, n)
    c, d = mu / (lam + mu), lam / (lam + mu)
    u = np.array([sum(np.prod([c[(j - m) % n] for m in range(1, k + 1)]) for k in range(n))
                  for j in range(n)]) / (1 - np.prod(c))
    got = gpu_run(gpu, rp, f, lam, mu, 0.0, 3000)
    np.testing.assert_allclose(got["psi"], d * u / n, rtol=1e-13)
    k = 40
    rp, f = psigen.csr_from_edges(k + 1, [(i, 0) for i in range(1, k + 1)])
    lam, mu = rng.uniform(0.05, 1, k + 1), rng.uniform(0.05, 1, k + 1)
    c, d = mu / (lam + mu), lam / (lam + mu)
    got = gpu_run(gpu, rp, f, lam, mu, 1e-15)
    want = d / (k + 1)
    want[0] = d[0] * (1 + c[1:].sum()) / (k + 1)
    np.testing.assert_allclose(got["psi"], want, rtol=1e-14)


@pytest.mark.parametrize("seed", range(30))
def test_random_small_graphs_fixed_count(gpu, seed, driver):
    """Random graphs N in [10, 300] (leaderless, mu = 0 and lambda = 0 users): exact
    Alg. 2 parity at a fixed T, all three norms."""
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(10, 300))
    p = float(rng.uniform(0.01, 0.3))
    mask = rng.random((n, n)) < p
    np.fill_diagonal(mask, False)
    mask[rng.choice(n, n // 10, replace=False), :] = False            # leaderless users
    fol, lead = np.nonzero(mask)
    rp, f = psigen.csr_from_edges(n, np.stack([fol, lead], 1))
    lam, mu = rng.uniform(0.05, 1, n), rng.uniform(0.05, 1, n)
    pick = rng.permutation(n)
    mu[pick[: n // 10]] = 0.0
    lam[pick[n // 10: n // 10 + n // 20]] = 0.0
    norm = ("row", "col", "one")[seed % 3]
    T = int(rng.integers(0, 40))
    ref = oracle.power_psi(rp, f, lam, mu, eps=0.0, max_iters=T, norm=norm)
    got = gpu_run(gpu, rp, f, lam, mu, 0.0, T, norm)
    assert got["T"] == ref.iterations
    assert oracle.max_rel_error(ref.psi, got["psi"]) <= 1e-12
    # eps_t is a sum of differences of rounded iterates: |d eps_t| <= ~N u ||s_t||_1
    np.testing.assert_allclose(got["hist"], ref.history, rtol=1e-6,
                               atol=1e-13 * max(1.0, np.abs(ref.s).sum()))


@pytest.mark.parametrize("heavy", ["0", "1"])
def test_long_rows_span_many_tiles(gpu, heavy, monkeypatch):
    """A hub followed by everybody (row longer than several 2048-item tiles) + a chain; with
    the heavy-row kernel off the hub is a split row of the edge stream (k_fix), with it on
    its followers below H come from staged shared memory."""
    monkeypatch.setenv("PSI_HEAVY", heavy)
    n = 9000
    edges = [(i, 0) for i in range(1, n)] + [(0, 1)] + [(i, i + 1) for i in range(1, n - 1)]
    rp, f = psigen.csr_from_edges(n, edges)
    rng = np.random.default_rng(3)
    lam, mu = rng.uniform(0.05, 1, n), rng.uniform(0.05, 1, n)
    ref = oracle.power_psi(rp, f, lam, mu, eps=1e-13)
    got = gpu_run(gpu, rp, f, lam, mu, 0.0, ref.iterations)
    assert oracle.max_rel_error(ref.psi, got["psi"]) <= TOL
    if heavy == "0":
        assert got["info"]["num_long_rows"] >= 1 and got["info"]["n_heavy"] == 0
    else:
        assert got["info"]["n_heavy"] >= 1


# ---------------------------------------------------------------- configs

def test_config0_and_nsystems(gpu):
    w = psigen.make_config(0)
    parity(gpu, w)
    brute = oracle.psi_nsystems(w.row_ptr, w.followers, w.lam, w.mu)
    got = gpu_run(gpu, w.row_ptr, w.followers, w.lam, w.mu, w.eps)
    assert oracle.relative_error(brute, got["psi"]) < 1e-11


@pytest.mark.parametrize("norm", ["row", "col", "one"])
def test_config1_parity(gpu, norm, driver):
    w = psigen.make_config(1)
    parity(gpu, w, norm=norm)


def test_config1_vs_exact(gpu):
    w = psigen.make_config(1)
    exact = oracle.psi_exact(w.row_ptr, w.followers, w.lam, w.mu)
    got = gpu_run(gpu, w.row_ptr, w.followers, w.lam, w.mu, w.eps)
    assert oracle.max_rel_error(exact, got["psi"]) < 1e-10
    assert abs(got["psi"].sum() - 1) < 1e-10


def test_config2_parity_and_pagerank(gpu):
    w = psigen.make_config(2)
    ref, got = parity(gpu, w)
    # near-uniform ER rows: the sliced-ELL layout pads little, so the library picks it, and
    # with no long rows k_sell finishes each sweep itself (no k_fix launch)
    assert got["info"]["sliced_ell"] == 1 and got["info"]["sell_long_rows"] == 0
    pi, _, _ = oracle.pagerank_power(w.row_ptr, w.followers, 0.5, eps=1e-14)
    assert oracle.max_rel_error(pi, got["psi"]) < 1e-9     # psi = PageRank(0.5)


def test_config3_parity(gpu):
    """Config 3 (Chung-Lu, 5M users, 1e8 edges, leaderless users kept): fixed-count parity,
    the ingest scalars, and the eps-mode stop (T within one sweep, eps_t history)."""
    w = psigen.make_config(3)
    ref, got = parity(gpu, w, full=True)
    assert got["info"]["n_leaderless"] > 0
    assert got["info"]["sliced_ell"] == 0        # power-law rows pad the slices 2.4x: tiles


def test_kappa_col_counterexample_through_cabi(gpu, driver):
    """The 4-user graph on which bound (19) fails with the column-sum norm (reading R1,
    tests/golden/kappa_col_counterexample.json): through the C-ABI every norm gives
    last_gap = ||B||_norm * eps_T (Alg. 2), the oracle's T and eps_t, and
    psi_get_info's kappa_row / kappa_col equal the golden values."""
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                    "kappa_col_counterexample.json")))
    rp, f = psigen.csr_from_edges(g["n"], g["edges"])
    lam, mu = np.array(g["lam"]), np.array(g["mu"])
    op = oracle.build_operator(rp, f, lam, mu)
    for norm, kappa in (("row", g["kappa_row"]), ("col", g["kappa_col"]), ("one", 1.0)):
        ref = oracle.power_psi(op=op, eps=1e-9, norm=norm)
        got = gpu_run(gpu, rp, f, lam, mu, 1e-9, 10_000, norm)
        info = got["info"]
        check_scalars(op, info)
        assert abs(info["kappa_row"] - g["kappa_row"]) < g["abs_tol"]
        assert abs(info["kappa_col"] - g["kappa_col"]) < g["abs_tol"]
        k = {"row": info["kappa_row"], "col": info["kappa_col"], "one": 1.0}[norm]
        assert abs(k - kappa) < g["abs_tol"]
        assert got["T"] == ref.iterations
        assert got["gap"] == pytest.approx(k * got["hist"][-1], rel=1e-15, abs=0)
        # eps_t = sum |s_t - s_{t-1}| of rounded iterates (|s| ~ 1): equal up to ~N u
        np.testing.assert_allclose(got["hist"], ref.history, rtol=1e-12, atol=1e-14)
        assert abs(got["hist"][0] - g["eps_1"]) < g["abs_tol"]
        assert oracle.max_rel_error(ref.psi, got["psi"]) <= TOL


def test_config4_small_scale_parity(gpu):
    w = psigen.make_config(4, scale=18)
    parity(gpu, w)


def test_config5_small_scale_parity(gpu):
    w = psigen.make_config(5, scale=18)
    parity(gpu, w)


# ------------------------------------------------------------ determinism, host input

def test_deterministic_and_host_equals_device(gpu):
    w = psigen.make_config(4, scale=16)
    a = gpu_run(gpu, w.row_ptr, w.followers, w.lam, w.mu, w.eps)
    b = gpu_run(gpu, w.row_ptr, w.followers, w.lam, w.mu, w.eps)
    c = gpu_run(gpu, w.row_ptr, w.followers, w.lam, w.mu, w.eps, host=True)
    assert np.array_equal(a["psi"], b["psi"]) and np.array_equal(a["hist"], b["hist"])
    assert np.array_equal(a["psi"], c["psi"])


def test_repeated_iterate_on_one_context(gpu):
    import torch
    w = psigen.make_config(1)
    with gpu.PsiGraph(*to_dev(w.row_ptr, w.followers, w.lam, w.mu)) as g:
        _, T1, _ = g.iterate(1e-9)
        p1 = g.get_psi().cpu().numpy()
        _, T2, _ = g.iterate(1e-12)
        _, T3, _ = g.iterate(1e-9)
        p3 = g.get_psi().cpu().numpy()
    assert T2 > T1 == T3 and np.array_equal(p1, p3)


# ------------------------------------------------ staged-segment heavy-row path (k_heavy)

@pytest.mark.parametrize("env", [
    {"PSI_HEAVY": "0"},                                     # edge-stream sweep only
    {"PSI_HEAVY": "1", "PSI_HEAVY_MIN": "2", "PSI_HEAVY_LABELS": "24576"},   # nearly every row heavy
    {"PSI_HEAVY": "1", "PSI_HEAVY_MIN": "16"},              # default H, more heavy rows
    {"PSI_HEAVY": "1"},                                     # library defaults, forced on
    {"PSI_HEAVY": "1", "PSI_OVERLAP": "1"},                 # k_heavy || k_tiles (overlapped plan)
    {"PSI_HEAVY": "1", "PSI_OVERLAP": "1", "PSI_HEAVY_MIN": "2", "PSI_HEAVY_LABELS": "24576"},
    {"PSI_HEAVY": "1", "PSI_OVERLAP": "0"},                 # serial plan
    {"PSI_HEAVY": "1", "PSI_HEAVY_SEARCH": "0"},            # fixed panel shape (no claim-order search)
    {"PSI_HEAVY": "1", "PSI_HEAVY_MIN": "2", "PSI_HEAVY_LABELS": "24576", "PSI_HEAVY_SLOTS": "2048"},  # many small panels
    {"PSI_HEAVY": "1", "PSI_HEAVY_SEG_SHIFT": "12", "PSI_HEAVY_SLOTS": "16384"},   # 32 KB segments, 16384 slots
])
def test_heavy_rows_parity(gpu, env, monkeypatch):
    """psi_build_graph reads the heavy-row knobs; every split of the work between k_heavy
    (followers < H from TMA-staged shared memory) and k_tiles must give the oracle's psi."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    w = psigen.make_config(5, scale=17)
    ref, got = parity(gpu, w)
    info = got["info"]
    if env.get("PSI_HEAVY") == "0":
        assert info["n_heavy"] == 0 and info["tile_edges"] == 512
    else:
        assert info["n_heavy"] > 0 and info["heavy_entries"] > 0 and info["heavy_panels"] > 0
        assert info["tile_edges"] == 1024
        if "PSI_OVERLAP" in env:
            assert info["overlapped"] == int(env["PSI_OVERLAP"])


def test_heavy_hub_many_slots(gpu, monkeypatch):
    """A hub followed by nearly everyone is spread over many slots (virtual rows) and
    warps; its psi must still match the oracle (and the readout path too)."""
    monkeypatch.setenv("PSI_HEAVY", "1")
    monkeypatch.setenv("PSI_HEAVY_MIN", "8")
    rng = np.random.default_rng(7)
    n = 40_000
    src = rng.integers(0, n, 400_000)
    dst = rng.integers(0, n, 400_000)
    keep = src != dst
    edges = np.stack([src[keep], dst[keep]], 1)
    hub = np.stack([np.arange(1, n), np.zeros(n - 1, dtype=np.int64)], 1)   # all follow user 0
    rp, f = psigen.csr_from_edges(n, np.concatenate([edges, hub]))
    lam = rng.uniform(0.05, 1.0, n)
    mu = rng.uniform(0.05, 1.0, n)
    ref = oracle.power_psi(rp, f, lam, mu, eps=1e-11)
    got = gpu_run(gpu, rp, f, lam, mu, 0.0, ref.iterations)
    assert got["info"]["n_heavy"] > 0
    assert oracle.max_rel_error(ref.psi, got["psi"]) <= TOL
    check_topk(ref.psi, got["psi"])


def test_heavy_rows_deterministic(gpu, monkeypatch):
    """k_heavy claims panels dynamically; each panel's sums have a fixed order, so psi and
    the eps history must be bitwise identical run to run."""
    monkeypatch.setenv("PSI_HEAVY", "1")
    monkeypatch.setenv("PSI_HEAVY_MIN", "8")
    w = psigen.make_config(4, scale=17)
    a = gpu_run(gpu, w.row_ptr, w.followers, w.lam, w.mu, w.eps)
    b = gpu_run(gpu, w.row_ptr, w.followers, w.lam, w.mu, w.eps)
    assert a["info"]["n_heavy"] > 0
    assert np.array_equal(a["psi"], b["psi"]) and np.array_equal(a["hist"], b["hist"])


# ------------------------------------------------ BASELINE.json full sizes (bench launch config)

@pytest.mark.slow
@pytest.mark.parametrize("cfg", [4, 5])
def test_full_size_parity(gpu, cfg):
    """Configs 4 (R-MAT s24, 273M edges) and 5 (R-MAT s26, 1.1e9 edges) at full size with the
    library defaults bench.py times: every psi entry against the fp64 oracle at the oracle's
    T*, the same top-k, and the eps-mode stop within one sweep of T*."""
    w = psigen.make_config(cfg)
    parity(gpu, w, full=True)


# ------------------------------------------------ exact and ragged tile boundaries, tiny graphs

@pytest.mark.parametrize("F", [511, 512, 513, 1023, 1024, 1025, 1536])
def test_tile_boundary_sizes(gpu, F, driver):
    """Leader 0 followed by users 1..F, each of them followed by 0: 2F active edge slots, so the
    edge stream ends exactly on, just before or just after a 1024-edge tile boundary, and row 0
    spans one or two tiles (a split row)."""
    n = F + 1
    edges = [(i, 0) for i in range(1, n)] + [(0, i) for i in range(1, n)]
    rp, f = psigen.csr_from_edges(n, edges)
    rng = np.random.default_rng(F)
    lam, mu = rng.uniform(0.05, 1.0, n), rng.uniform(0.05, 1.0, n)
    ref = oracle.power_psi(rp, f, lam, mu, eps=1e-13)
    got = gpu_run(gpu, rp, f, lam, mu, 0.0, ref.iterations)
    assert got["T"] == ref.iterations
    assert oracle.max_rel_error(ref.psi, got["psi"]) <= TOL


def test_single_user_and_no_edges(gpu, driver):
    """N = 1 (no edges possible): psi = d / N after T = 1 (epsilon_1 = 0)."""
    rp, f = np.zeros(2, np.int64), np.zeros(0, np.int32)
    lam, mu = np.array([0.3]), np.array([0.6])
    ref = oracle.power_psi(rp, f, lam, mu, eps=1e-12)
    got = gpu_run(gpu, rp, f, lam, mu, 1e-12)
    assert got["T"] == ref.iterations
    np.testing.assert_allclose(got["psi"], ref.psi, rtol=1e-15)
