"""Multi-profile batch (psi_build_graph_batch) against the fp64 oracle (-m gpu).

k activity profiles share one graph; the library sweeps four at a time with interleaved x.
Each profile p must behave exactly as Alg. 2 run alone on (lambda_p, mu_p):
  * eps mode: its own stop, T_p within one sweep of the oracle's T*_p (c.5 step 3);
  * psi_p equal to the oracle's psi after T_p sweeps to 1e-10 per entry (north_star), same top-k;
  * its eps_t history equal to the oracle's;
  * and equal to a single-profile context of the same profile (same T, psi to rounding).
"""

import numpy as np
import pytest

import oracle
import psigen

pytestmark = pytest.mark.gpu

TOL = 1e-10


def to_dev(*arrays):
    import torch
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrays]


def batch_run(psi, rp, f, lam, mu, eps, max_iters=100_000, norm="row"):
    with psi.PsiGraph(*to_dev(rp, f, lam, mu)) as g:
        st, T, gap = g.iterate(eps, max_iters, norm)
        out = g.get_psi().cpu().numpy()
        info = g.info()
        if lam.ndim == 2 and lam.shape[0] > 1:
            Tp, gp = g.profile_stats()
            hist = [g.profile_history(p) for p in range(lam.shape[0])]
        else:
            Tp, gp, hist = np.array([T]), np.array([gap]), [g.get_residual_history()]
    return dict(psi=out, T=T, gap=gap, status=st, Tp=Tp, gp=gp, hist=hist, info=info)


def check_profile(rp, f, lam, mu, eps, got_psi, got_T, got_hist, norm="row"):
    ref = oracle.power_psi(rp, f, lam, mu, eps=eps, norm=norm)
    assert abs(got_T - ref.iterations) <= 1, (got_T, ref.iterations)
    at = ref if got_T == ref.iterations else oracle.power_psi(rp, f, lam, mu, eps=0.0,
                                                               max_iters=got_T, norm=norm)
    err = oracle.max_rel_error(at.psi, got_psi)
    assert err <= TOL, err
    for k in (10, 100):
        k = min(k, at.psi.size)
        a, b = oracle.top_k(at.psi, k), oracle.top_k(got_psi, k)
        if not np.array_equal(a, b):
            for x, y in zip(a, b):
                if x != y:
                    assert abs(at.psi[x] - at.psi[y]) <= 1e-10 * max(at.psi[x], at.psi[y])
    h_ref = np.array(at.history)
    k = min(len(h_ref), len(got_hist))
    np.testing.assert_allclose(got_hist[:k], h_ref[:k], rtol=1e-6,
                               atol=1e-13 * np.abs(at.s).sum())


@pytest.mark.parametrize("k", [2, 4, 5, 9])
def test_batch_config1_profiles(gpu, k):
    """Config 1's graph with k U(0.05, 1) profiles (k = 5, 9: ragged last group of four)."""
    w = psigen.make_config(1)
    lam, mu = psigen.activity_profiles(w.row_ptr.size - 1, k, "uniform")
    r = batch_run(gpu, w.row_ptr, w.followers, lam, mu, 1e-12)
    assert r["psi"].shape == (k, lam.shape[1]) and r["info"]["n_profiles"] == k
    assert r["T"] == r["Tp"].max() and r["status"] == 0
    # the context's scalars are profile 0's (||B|| by rows / columns, rho_A: P:316)
    sc = oracle.graph_scalars(oracle.build_operator(w.row_ptr, w.followers, lam[0], mu[0]))
    for key in ("kappa_row", "kappa_col", "rho_A"):
        assert abs(r["info"][key] - sc[key]) <= 1e-12 * abs(sc[key]), key
    for p in range(k):
        check_profile(w.row_ptr, w.followers, lam[p], mu[p], 1e-12, r["psi"][p], r["Tp"][p],
                      r["hist"][p])


def test_batch_fixed_count(gpu):
    """eps = 0: every profile runs exactly max_iters sweeps (the parity protocol's mode)."""
    w = psigen.make_config(1)
    lam, mu = psigen.activity_profiles(w.row_ptr.size - 1, 4, "uniform", seed=3)
    r = batch_run(gpu, w.row_ptr, w.followers, lam, mu, 0.0, 37)
    assert list(r["Tp"]) == [37] * 4 and r["status"] > 0          # PSI_NOT_CONVERGED
    for p in range(4):
        ref = oracle.power_psi(w.row_ptr, w.followers, lam[p], mu[p], eps=0.0, max_iters=37)
        assert oracle.max_rel_error(ref.psi, r["psi"][p]) <= TOL


def test_batch_heavy_tailed_graph_mixed_profiles(gpu):
    """R-MAT (config 5 shape, scale 15) with profiles of different convergence speed:
    LogNormal with pure posters, homogeneous (0.15, 0.85) (psi = PageRank(0.85), slow), and
    mu = 0 (c = 0: psi = 1/N after one sweep).  Each stops on its own rule."""
    w = psigen.make_config(5, scale=15)
    n = w.row_ptr.size - 1
    lam, mu = psigen.activity_profiles(n, 5, "lognormal", pure_posters=True)
    lam[1], mu[1] = 0.15, 0.85
    lam[2], mu[2] = 0.7, 0.0
    r = batch_run(gpu, w.row_ptr, w.followers, lam, mu, 1e-9)
    assert r["info"]["n_heavy"] == 0
    assert r["Tp"][2] == 1 and np.allclose(r["psi"][2], 1.0 / n, rtol=1e-15)
    assert len(set(r["Tp"].tolist())) > 2          # profiles stopped at different sweeps
    for p in range(5):
        check_profile(w.row_ptr, w.followers, lam[p], mu[p], 1e-9, r["psi"][p], r["Tp"][p],
                      r["hist"][p])


def test_batch_equals_single_contexts(gpu):
    """Profile p of a batch = a single-profile context built on (lambda_p, mu_p)."""
    w = psigen.make_config(3, scale=14)
    n = w.row_ptr.size - 1
    lam, mu = psigen.activity_profiles(n, 4, "lognormal")
    r = batch_run(gpu, w.row_ptr, w.followers, lam, mu, 1e-9)
    for p in range(4):
        s = batch_run(gpu, w.row_ptr, w.followers, lam[p], mu[p], 1e-9)
        assert s["T"] == r["Tp"][p]
        assert oracle.max_rel_error(s["psi"], r["psi"][p]) <= 1e-13
        np.testing.assert_allclose(r["hist"][p], s["hist"][0], rtol=1e-6,
                                   atol=1e-12 * s["hist"][0][0])


def test_batch_norm_one_and_col_rejected(gpu):
    w = psigen.make_config(0)
    lam, mu = psigen.activity_profiles(64, 2, "uniform")
    r = batch_run(gpu, w.row_ptr, w.followers, lam, mu, 1e-12, norm="one")
    for p in range(2):
        check_profile(w.row_ptr, w.followers, lam[p], mu[p], 1e-12, r["psi"][p], r["Tp"][p],
                      r["hist"][p], norm="one")
    with gpu.PsiGraph(*to_dev(w.row_ptr, w.followers, lam, mu)) as g:
        with pytest.raises(gpu.PsiError):
            g.iterate(1e-9, 100, "col")


def test_batch_degenerate(gpu):
    """max_iters = 0 and eps >= 1 (T = 0, psi from x_0 = a); an edgeless graph (psi = d/N);
    deterministic re-runs; a bad profile is rejected at the boundary."""
    w = psigen.make_config(0)
    lam, mu = psigen.activity_profiles(64, 3, "uniform", seed=9)
    for eps, mi in ((0.0, 0), (2.0, 50)):
        r = batch_run(gpu, w.row_ptr, w.followers, lam, mu, eps, mi)
        assert list(r["Tp"]) == [0, 0, 0]
        for p in range(3):
            ref = oracle.power_psi(w.row_ptr, w.followers, lam[p], mu[p], eps=eps, max_iters=mi)
            assert oracle.max_rel_error(ref.psi, r["psi"][p]) <= TOL
    a = batch_run(gpu, w.row_ptr, w.followers, lam, mu, 1e-12)
    b = batch_run(gpu, w.row_ptr, w.followers, lam, mu, 1e-12)
    assert np.array_equal(a["psi"], b["psi"]) and all(
        np.array_equal(x, y) for x, y in zip(a["hist"], b["hist"]))
    n = 50
    rp, f = np.zeros(n + 1, np.int64), np.zeros(0, np.int32)
    lam2, mu2 = psigen.activity_profiles(n, 2, "uniform")
    r = batch_run(gpu, rp, f, lam2, mu2, 1e-12)
    for p in range(2):
        ref = oracle.power_psi(rp, f, lam2[p], mu2[p], eps=1e-12)
        assert r["Tp"][p] == ref.iterations
        assert oracle.max_rel_error(ref.psi, r["psi"][p]) <= TOL
    bad = lam.copy()
    bad[2, 5] = -1.0
    with pytest.raises(gpu.PsiError):
        gpu.PsiGraph(*to_dev(w.row_ptr, w.followers, bad, mu))


@pytest.mark.slow
def test_batch_full_size_config5(gpu):
    """Config 5 at full size (R-MAT scale 26, 1.1e9 edges), four profiles, profile 0 = the
    config's own activity: profile 0 of the batch must equal the single-profile path (itself
    pinned to the oracle at full size in test_gpu_parity) -- same T, psi to 1e-12 -- and every
    profile stops at its own T with gap <= eps."""
    import torch
    w = psigen.make_config(5)
    n = w.row_ptr.size - 1
    lam, mu = psigen.activity_profiles(n, 4, "lognormal", pure_posters=True)
    lam[0], mu[0] = w.lam, w.mu
    with gpu.PsiGraph(*to_dev(w.row_ptr, w.followers, w.lam, w.mu)) as g:
        _, T0, _ = g.iterate(w.eps)
        psi0 = g.get_psi().cpu().numpy()
    torch.cuda.empty_cache()
    r = batch_run(gpu, w.row_ptr, w.followers, lam, mu, w.eps)
    assert r["Tp"][0] == T0
    assert oracle.max_rel_error(psi0, r["psi"][0]) <= 1e-12
    assert np.all(r["gp"] <= w.eps) and np.all(r["Tp"] > 10)


def test_batch_host_inputs_equal_device_inputs(gpu):
    """psi_build_graph_batch from host (PSI_MEM_HOST) arrays = from device arrays, bitwise."""
    w = psigen.make_config(1)
    lam, mu = psigen.activity_profiles(w.row_ptr.size - 1, 3, "uniform", seed=4)
    d = batch_run(gpu, w.row_ptr, w.followers, lam, mu, 1e-12)
    with gpu.PsiGraph(w.row_ptr, w.followers, lam, mu) as g:
        g.iterate(1e-12)
        h = g.get_psi(device=False).numpy()
        Tp, _ = g.profile_stats()
    assert np.array_equal(Tp, d["Tp"]) and np.array_equal(h, d["psi"])
