"""GPU parity of the PageRank power method (psi_pagerank, Eq. (22))
against the oracle's pagerank_power (pinned in test_oracle_pins.py against networkx and the
homogeneous psi = PageRank identity).  Fixed-count protocol as for psi: the oracle
runs to eps and records T*; the GPU runs exactly T* sweeps (eps = 0) and must agree to 1e-10
per entry with the same top-k; run to eps it must stop within one sweep of T*."""

import numpy as np
import pytest

import oracle
import psigen

pytestmark = pytest.mark.gpu

TOL = 1e-10


def to_dev(*arrays):
    import torch
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrays]


def gpu_pagerank(psi, rp, f, lam, mu, alpha, eps, max_iters=100_000):
    with psi.PsiGraph(*to_dev(rp, f, lam, mu)) as g:
        st, T, gap = g.pagerank(alpha, eps, max_iters)
        pi = g.get_pagerank().cpu().numpy()
        hist = g.get_residual_history()
        info = g.info()
    return dict(pi=pi, T=T, gap=gap, status=st, hist=hist, info=info)


def pr_parity(psi, w, alpha, eps=1e-12):
    ref, T, its = oracle.pagerank_power(w.row_ptr, w.followers, alpha, eps=eps, keep_iterates=True)
    got = gpu_pagerank(psi, w.row_ptr, w.followers, w.lam, w.mu, alpha, 0.0, T)
    assert got["T"] == T
    err = oracle.max_rel_error(ref, got["pi"])
    assert err <= TOL, err
    for k in (10, 100, 1000):
        k = min(k, ref.size)
        a, b = oracle.top_k(ref, k), oracle.top_k(got["pi"], k)
        if not np.array_equal(a, b):          # only near-ties may swap (reading R10)
            for x, y in zip(a, b):
                if x != y:
                    assert abs(ref[x] - ref[y]) <= 1e-10 * max(ref[x], ref[y])
    # residual history = ||pi_t - pi_{t-1}||_1 of the oracle's iterates
    h_ref = np.array([np.abs(its[t + 1] - its[t]).sum() for t in range(T)])
    np.testing.assert_allclose(got["hist"], h_ref, rtol=1e-6, atol=1e-14)
    g2 = gpu_pagerank(psi, w.row_ptr, w.followers, w.lam, w.mu, alpha, eps)
    assert abs(g2["T"] - T) <= 1
    return ref, got


@pytest.mark.parametrize("alpha", [0.85, 0.5])
def test_pagerank_config1(gpu, alpha, driver):
    pr_parity(gpu, psigen.make_config(1), alpha)


def test_pagerank_config2_equals_homogeneous_psi(gpu):
    """Config 2 (lambda = mu = 1): psi = PageRank(alpha = mu/(lambda+mu) = 1/2)."""
    w = psigen.make_config(2)
    ref, got = pr_parity(gpu, w, 0.5)
    with gpu.PsiGraph(*to_dev(w.row_ptr, w.followers, w.lam, w.mu)) as g:
        g.iterate(1e-14)
        psi_v = g.get_psi().cpu().numpy()
    assert oracle.max_rel_error(got["pi"], psi_v) < 1e-9


def test_pagerank_config3_leaderless(gpu):
    w = psigen.make_config(3, scale=18)
    ref, got = pr_parity(gpu, w, 0.85, eps=1e-9)
    assert got["info"]["n_leaderless"] > 0


@pytest.mark.parametrize("heavy", ["0", "1"])
def test_pagerank_rmat_heavy_rows(gpu, heavy, monkeypatch):
    monkeypatch.setenv("PSI_HEAVY", heavy)
    monkeypatch.setenv("PSI_HEAVY_MIN", "16")
    w = psigen.make_config(5, scale=17)
    ref, got = pr_parity(gpu, w, 0.85, eps=1e-9)
    assert (got["info"]["n_heavy"] > 0) == (heavy == "1")


def test_pagerank_edgeless_and_chain(gpu, driver):
    # edgeless: every user is follower-less -> pi = (1 - alpha)/N after one sweep, and the
    # second sweep changes nothing (exact fixed point: the loop stops at T = 2 < max_iters)
    n = 5
    rp = np.zeros(n + 1, dtype=np.int64)
    f = np.zeros(0, dtype=np.int32)
    lam = np.ones(n)
    got = gpu_pagerank(gpu, rp, f, lam, lam, 0.85, 0.0, 3)
    ref, T, _ = oracle.pagerank_power(rp, f, 0.85, eps=0.0, max_iters=3)
    assert got["T"] == T == 2
    np.testing.assert_allclose(got["pi"], ref, rtol=1e-15)
    # chain 0 -> 1 (0 follows 1): user 1 is leaderless
    rp, f = psigen.csr_from_edges(2, [(0, 1)])
    for iters in (0, 1, 2, 5):
        ref, T, _ = oracle.pagerank_power(rp, f, 0.85, eps=0.0, max_iters=iters)
        got = gpu_pagerank(gpu, rp, f, np.ones(2), np.ones(2), 0.85, 0.0, iters)
        assert got["T"] == T
        np.testing.assert_allclose(got["pi"], ref, rtol=1e-14)


def test_pagerank_state_and_args(gpu):
    w = psigen.make_config(1)
    with gpu.PsiGraph(*to_dev(w.row_ptr, w.followers, w.lam, w.mu)) as g:
        with pytest.raises(gpu.PsiError):
            g.get_pagerank()                               # PSI_E_STATE before any run
        for bad in ((1.0, 1e-9), (-0.1, 1e-9), (0.85, -1.0), (float("nan"), 1e-9)):
            with pytest.raises(gpu.PsiError):
                g.pagerank(*bad)
        g.iterate(1e-9)
        psi_before = g.get_psi().cpu().numpy()
        g.pagerank(0.85, 1e-9)
        assert np.array_equal(g.get_psi().cpu().numpy(), psi_before)   # psi untouched
        with pytest.raises(gpu.PsiError):
            g.get_series()                                 # iterate buffers now hold pi / Dt
        g.iterate(1e-9)
        g.get_series()
        st, T, gap = g.pagerank(0.85, 0.0, 2)              # max_iters reached, gap > 0
        assert st == gpu.PSI_NOT_CONVERGED and T == 2
