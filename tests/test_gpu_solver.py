"""The three loop drivers of Alg. 2 (DESIGN.md §7 "Loop control") against the fp64 oracle (-m gpu):

  0  CUDA-graph WHILE node (k_init -> WHILE{k_heavy, k_tiles, k_fix} -> readout), the default;
  1  persistent cooperative kernel k_solve (graphs with no heavy rows and few tiles);
  2  direct launches with a host-side stop test (PSI_GRAPH=0).

Each must reproduce the oracle's psi at the oracle's T* (<= 1e-10 per entry, north_star), stop
at the same sweep in eps mode, and the drivers must agree with one another on T and psi.
"""

import numpy as np
import pytest

import oracle
import psigen

pytestmark = pytest.mark.gpu

TOL = 1e-10
DRIVERS = {
    0: {"PSI_COOP_TILES": "0"},
    1: {"PSI_COOP_TILES": str(1 << 30)},
    2: {"PSI_COOP_TILES": "0", "PSI_GRAPH": "0"},
}


def to_dev(*arrays):
    import torch
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrays]


def workload(name):
    if name == "er64":
        return psigen.make_config(0)
    if name == "c1":
        return psigen.make_config(1)
    if name == "chung_lu_s14":
        return psigen.make_config(3, scale=14)
    if name == "rmat_s15":
        return psigen.make_config(5, scale=15)
    raise KeyError(name)


def run(psi, w, eps, max_iters, driver, monkeypatch, pagerank=None):
    for k, v in DRIVERS[driver].items():
        monkeypatch.setenv(k, v)
    monkeypatch.setenv("PSI_HEAVY", "0")
    try:
        with psi.PsiGraph(*to_dev(w.row_ptr, w.followers, w.lam, w.mu)) as g:
            if pagerank is None:
                st, T, gap = g.iterate(eps, max_iters)
                out = g.get_psi().cpu().numpy()
            else:
                st, T, gap = g.pagerank(pagerank, eps, max_iters)
                out = g.get_pagerank().cpu().numpy()
            hist = g.get_residual_history()
            info = g.info()
    finally:
        for k in DRIVERS[driver]:
            monkeypatch.delenv(k, raising=False)
    assert info["last_solver"] == driver
    return dict(out=out, T=T, gap=gap, status=st, hist=hist)


@pytest.mark.parametrize("name", ["er64", "c1", "chung_lu_s14", "rmat_s15"])
def test_drivers_match_oracle(gpu, name, monkeypatch):
    w = workload(name)
    ref = oracle.power_psi(w.row_ptr, w.followers, w.lam, w.mu, eps=w.eps)
    got = {}
    for d in DRIVERS:
        r = run(gpu, w, 0.0, ref.iterations, d, monkeypatch)
        assert r["T"] == ref.iterations
        err = oracle.max_rel_error(ref.psi, r["out"])
        assert err <= TOL, (d, err)
        h_ref = np.array(ref.history)
        k = min(len(h_ref), len(r["hist"]))
        np.testing.assert_allclose(r["hist"][:k], h_ref[:k], rtol=1e-6,
                                   atol=1e-13 * np.abs(ref.s).sum())
        e = run(gpu, w, w.eps, 100_000, d, monkeypatch)
        assert abs(e["T"] - ref.iterations) <= 1 and e["gap"] <= w.eps
        got[d] = e
    # the drivers run the same arithmetic: same T, psi equal to rounding of eps_t's order
    assert got[0]["T"] == got[1]["T"] == got[2]["T"]
    assert np.array_equal(got[0]["out"], got[2]["out"])
    assert oracle.max_rel_error(got[0]["out"], got[1]["out"]) <= 1e-14


@pytest.mark.parametrize("alpha", [0.85, 0.3])
def test_persistent_pagerank(gpu, alpha, monkeypatch):
    """Eq. (22) through k_solve (no readout; x = pi / D~ after the loop)."""
    w = psigen.make_config(1)
    ref, T, _ = oracle.pagerank_power(w.row_ptr, w.followers, alpha, eps=1e-12, keep_iterates=True)
    r = run(gpu, w, 0.0, T, 1, monkeypatch, pagerank=alpha)
    assert r["T"] == T
    assert oracle.max_rel_error(ref, r["out"]) <= TOL
    g = run(gpu, w, 1e-12, 100_000, 0, monkeypatch, pagerank=alpha)
    c = run(gpu, w, 1e-12, 100_000, 1, monkeypatch, pagerank=alpha)
    assert g["T"] == c["T"] and abs(c["T"] - T) <= 1
    assert oracle.max_rel_error(g["out"], c["out"]) <= 1e-14


def test_persistent_degenerate(gpu, monkeypatch):
    """max_iters = 0 (psi from x_0 = a), eps above gap_0 (no sweep), an edgeless graph (every
    user follower-less: nothing to sweep, psi = d/N) -- the same answers as the graph driver."""
    w = psigen.make_config(0)
    for eps, mi in ((0.0, 0), (2.0, 100), (0.0, 1)):
        a = run(gpu, w, eps, mi, 0, monkeypatch)
        b = run(gpu, w, eps, mi, 1, monkeypatch)
        ref = oracle.power_psi(w.row_ptr, w.followers, w.lam, w.mu, eps=eps, max_iters=mi)
        assert a["T"] == b["T"] == ref.iterations
        assert oracle.max_rel_error(ref.psi, b["out"]) <= TOL
        assert oracle.max_rel_error(a["out"], b["out"]) <= 1e-14
    n = 100
    e = psigen.Workload("edgeless", np.zeros(n + 1, np.int64), np.zeros(0, np.int32),
                        np.full(n, 0.3), np.full(n, 0.7), 1e-12)
    ref = oracle.power_psi(e.row_ptr, e.followers, e.lam, e.mu, eps=e.eps)
    b = run(gpu, e, e.eps, 100, 1, monkeypatch)
    assert b["T"] == ref.iterations
    assert oracle.max_rel_error(ref.psi, b["out"]) <= TOL
