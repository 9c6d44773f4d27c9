"""GPU parity of the sliced-ELL sweep (k_sell) against the fp64 oracle (-m gpu).

The sliced-ELL layout changes only how the sums S_j = sum_{n in F(j)} x_n of Alg. 2
 are scheduled -- windows of rows sorted by length, 32 rows per slice summed one per
lane, long rows in pieces summed by whole warps and joined in piece order -- so every case
must give the oracle's psi per entry at the oracle's T* (north_star 1e-10), its eps_t history
and T within one sweep when run to eps.  Tiny windows, long-row limits and pieces
(PSI_SELL_SHIFT / _LMAX / _PIECE) put many long rows and multi-piece rows into small graphs.
"""

import numpy as np
import pytest

import oracle
import psigen
from test_gpu_parity import TOL, check_topk, gpu_run, parity

pytestmark = pytest.mark.gpu


def sell_env(monkeypatch, **kw):
    monkeypatch.setenv("PSI_SELL", "1")
    for k, v in kw.items():
        monkeypatch.setenv("PSI_SELL_" + k.upper(), str(v))


def random_graph(seed, nmin=10, nmax=400):
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(nmin, nmax))
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
    return rng, rp, f, lam, mu


@pytest.mark.parametrize("seed", range(24))
def test_sell_random_small_graphs(gpu, seed, monkeypatch):
    """Windows of 32-256 rows (or cut after 1-4 x 32 edges), rows longer than 2-40 followers
    summed by warps in pieces of 32-96 followers: fixed-count parity, all three norms, eps_t
    history."""
    rng, rp, f, lam, mu = random_graph(seed)
    sell_env(monkeypatch, shift=5 + seed % 4, lmax=(2, 7, 40)[seed % 3], piece=(32, 33, 96)[seed % 3],
             kcap=(1, 4, 1000)[seed % 3])
    norm = ("row", "col", "one")[seed % 3]
    T = int(rng.integers(0, 40))
    ref = oracle.power_psi(rp, f, lam, mu, eps=0.0, max_iters=T, norm=norm)
    got = gpu_run(gpu, rp, f, lam, mu, 0.0, T, norm)
    assert got["info"]["sliced_ell"] == 1
    assert got["T"] == ref.iterations
    assert oracle.max_rel_error(ref.psi, got["psi"]) <= 1e-12
    np.testing.assert_allclose(got["hist"], ref.history, rtol=1e-6,
                               atol=1e-13 * max(1.0, np.abs(ref.s).sum()))


@pytest.mark.parametrize("piece", [32, 4096])
def test_sell_hub_in_pieces(gpu, piece, monkeypatch):
    """A hub followed by everybody (9000 followers: 282 or 3 pieces) + a chain."""
    sell_env(monkeypatch, piece=piece)
    n = 9000
    edges = [(i, 0) for i in range(1, n)] + [(0, 1)] + [(i, i + 1) for i in range(1, n - 1)]
    rp, f = psigen.csr_from_edges(n, edges)
    rng = np.random.default_rng(3)
    lam, mu = rng.uniform(0.05, 1, n), rng.uniform(0.05, 1, n)
    ref = oracle.power_psi(rp, f, lam, mu, eps=1e-13)
    got = gpu_run(gpu, rp, f, lam, mu, 0.0, ref.iterations)
    info = got["info"]
    assert info["sliced_ell"] == 1 and info["sell_long_rows"] == 1
    assert info["sell_pieces"] == -(-(n - 1) // piece)
    assert oracle.max_rel_error(ref.psi, got["psi"]) <= TOL
    check_topk(ref.psi, got["psi"])


@pytest.mark.parametrize("env", [
    {},                                                     # library window / lmax / piece
    {"lmax": 16, "piece": 64},                              # many long rows, many pieces
    {"shift": 5},                                           # one slice per window
    {"shift": 10, "kcap": 100000},                         # 32 slices per window
    {"kcap": 1},                                            # one 32-row block per window
])
def test_sell_config1_all_norms(gpu, env, monkeypatch):
    sell_env(monkeypatch, **env)
    w = psigen.make_config(1)
    for norm in ("row", "col", "one"):
        ref, got = parity(gpu, w, norm=norm)
        assert got["info"]["sliced_ell"] == 1


@pytest.mark.parametrize("env", [
    {"PSI_HEAVY": "1"},
    {"PSI_HEAVY": "1", "PSI_HEAVY_MIN": "2", "PSI_HEAVY_LABELS": "24576"},
    {"PSI_HEAVY": "1", "PSI_SELL_LMAX": "8", "PSI_SELL_PIECE": "64"},
    {"PSI_HEAVY": "0", "PSI_SELL_LMAX": "8", "PSI_SELL_PIECE": "64"},
])
def test_sell_with_heavy_rows(gpu, env, monkeypatch):
    """k_heavy (followers < H from staged shared memory) + k_sell (the rest): R-MAT with
    pure posters at scale 17, every split of the work."""
    sell_env(monkeypatch)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    w = psigen.make_config(5, scale=17)
    ref, got = parity(gpu, w)
    info = got["info"]
    assert info["sliced_ell"] == 1
    assert (info["n_heavy"] > 0) == (env["PSI_HEAVY"] == "1")
    if "PSI_SELL_LMAX" in env:
        assert info["sell_long_rows"] > 0 and info["sell_pieces"] >= info["sell_long_rows"]


def test_sell_deterministic_and_repeated(gpu, monkeypatch):
    """Work items are claimed dynamically but every sum has a fixed order: psi and eps_t are
    bitwise identical run to run; a context iterated again (new solve, older piece epochs in
    memory) gives the same result; eps >= 1 gives T = 0 and psi from x_0."""
    import torch
    sell_env(monkeypatch, lmax=8, piece=64, kcap=16)
    monkeypatch.setenv("PSI_HEAVY", "0")
    w = psigen.make_config(4, scale=16)
    a = gpu_run(gpu, w.row_ptr, w.followers, w.lam, w.mu, w.eps)
    b = gpu_run(gpu, w.row_ptr, w.followers, w.lam, w.mu, w.eps)
    assert a["info"]["sell_pieces"] > 0
    assert np.array_equal(a["psi"], b["psi"]) and np.array_equal(a["hist"], b["hist"])
    dev = [torch.from_numpy(np.ascontiguousarray(x)).cuda()
           for x in (w.row_ptr, w.followers, w.lam, w.mu)]
    with gpu.PsiGraph(*dev) as g:
        _, T1, _ = g.iterate(w.eps)
        p1 = g.get_psi().cpu().numpy()
        _, T0, _ = g.iterate(2.0)
        p0 = g.get_psi().cpu().numpy()
        _, T2, _ = g.iterate(1e-12)
        _, T3, _ = g.iterate(w.eps)
        p3 = g.get_psi().cpu().numpy()
    assert T0 == 0 and T2 > T1 == T3 and np.array_equal(p1, p3)
    assert np.array_equal(p1, a["psi"])
    ref0 = oracle.power_psi(w.row_ptr, w.followers, w.lam, w.mu, eps=2.0)
    assert ref0.iterations == 0 and oracle.max_rel_error(ref0.psi, p0) <= TOL


@pytest.mark.parametrize("alpha", [0.85, 0.5])
def test_sell_pagerank(gpu, alpha, monkeypatch):
    from test_gpu_pagerank import pr_parity
    sell_env(monkeypatch, lmax=16, piece=64)
    pr_parity(gpu, psigen.make_config(1), alpha)
    monkeypatch.setenv("PSI_HEAVY", "1")
    pr_parity(gpu, psigen.make_config(5, scale=16), alpha, eps=1e-12)


def test_sell_config3_parity(gpu, monkeypatch):
    """Config 3 at full size (Chung-Lu, 5M users, 1e8 edges, leaderless users): fixed-count
    parity, the ingest scalars, the eps-mode stop and history."""
    sell_env(monkeypatch)
    w = psigen.make_config(3)
    ref, got = parity(gpu, w, full=True)
    assert got["info"]["sliced_ell"] == 1


@pytest.mark.parametrize("seed", range(8))
def test_sell_fused_finish(gpu, seed, monkeypatch):
    """No long rows and no heavy rows: k_sell's last CTA reduces eps_t and runs the stop rule
    itself (no k_fix launch).  Fixed-count parity, the eps_t history, the eps-mode stop (T
    within one sweep) and the readout, through the graph loop and the direct launches."""
    rng, rp, f, lam, mu = random_graph(100 + seed)
    sell_env(monkeypatch, shift=5 + seed % 4, lmax=2047, kcap=(1, 4, 1000)[seed % 3])
    if seed % 2:
        monkeypatch.setenv("PSI_GRAPH", "0")
    norm = ("row", "col", "one")[seed % 3]
    T = int(rng.integers(0, 40))
    ref = oracle.power_psi(rp, f, lam, mu, eps=0.0, max_iters=T, norm=norm)
    got = gpu_run(gpu, rp, f, lam, mu, 0.0, T, norm)
    assert got["info"]["sliced_ell"] == 1 and got["info"]["sell_long_rows"] == 0
    assert got["info"]["n_heavy"] == 0
    assert got["T"] == ref.iterations
    assert oracle.max_rel_error(ref.psi, got["psi"]) <= 1e-12
    np.testing.assert_allclose(got["hist"], ref.history, rtol=1e-6,
                               atol=1e-13 * max(1.0, np.abs(ref.s).sum()))
    ref2 = oracle.power_psi(rp, f, lam, mu, eps=1e-10, norm=norm)
    got2 = gpu_run(gpu, rp, f, lam, mu, 1e-10, 10_000, norm)
    assert abs(got2["T"] - ref2.iterations) <= 1
    assert oracle.max_rel_error(ref2.psi, got2["psi"]) <= 1e-9
