"""C-ABI error contract and edge cases on the device (-m gpu), include/psi.h."""

import ctypes

import numpy as np
import pytest

import psigen

pytestmark = pytest.mark.gpu


def dev(*arrays):
    import torch
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrays]


def build_status(psi, rp, f, lam, mu):
    try:
        g = psi.PsiGraph(*dev(np.asarray(rp, np.int64), np.asarray(f, np.int32),
                              np.asarray(lam, float), np.asarray(mu, float)))
        g.close()
        return psi.PSI_OK
    except psi.PsiError as e:
        return e.status


@pytest.mark.parametrize("rp,f,why", [
    ([1, 1, 2], [1, 0], "row_ptr[0] != 0"),
    ([0, 1, 3], [1, 0], "row_ptr[n] != m"),
    ([0, 2, 1], [1, 0], "decreasing"),
    ([0, 1, 2], [5, 0], "index out of range"),
    ([0, 1, 2], [-1, 0], "negative index"),
    ([0, 1, 2], [0, 0], "self loop"),
    ([0, 2, 2, 2], [2, 1, ], "unsorted row"),
    ([0, 2, 2, 2], [1, 1], "duplicate follower"),
])
def test_graph_contract(gpu, rp, f, why):
    n = len(rp) - 1
    st = build_status(gpu, rp, f, np.ones(n), np.ones(n))
    assert st == gpu.PSI_E_GRAPH, why


@pytest.mark.parametrize("lam,mu", [([np.nan, 1], [1, 1]), ([1, np.inf], [1, 1]),
                                    ([-1, 1], [1, 1]), ([0, 1], [0, 1])])
def test_activity_contract(gpu, lam, mu):
    assert build_status(gpu, [0, 1, 2], [1, 0], lam, mu) == gpu.PSI_E_ACTIVITY


def test_invalid_args(gpu):
    lib = gpu.load_library()
    ctx = ctypes.c_void_p()
    assert lib.psi_build_graph(3, 0, None, None, None, None, 1, None, ctypes.byref(ctx)) == gpu.PSI_E_INVALID_ARG
    rp, f, lam, mu = dev(np.array([0, 1, 2], np.int64), np.array([1, 0], np.int32), np.ones(2), np.ones(2))
    with gpu.PsiGraph(rp, f, lam, mu) as g:
        with pytest.raises(gpu.PsiError) as e:
            g.get_psi()
        assert e.value.status == gpu.PSI_E_STATE
        for bad in (dict(eps=-1.0), dict(eps=float("nan")), dict(max_iters=-1)):
            kw = dict(eps=1e-9, max_iters=10)
            kw.update(bad)
            with pytest.raises(gpu.PsiError) as e:
                g.iterate(**kw)
            assert e.value.status == gpu.PSI_E_INVALID_ARG
        st = lib.psi_iterate(g._ctx, 1e-9, 10, 7, None, None)
        assert st == gpu.PSI_E_INVALID_ARG


def test_not_converged_and_eps_ge_one(gpu):
    w = psigen.make_config(1)
    with gpu.PsiGraph(*dev(w.row_ptr, w.followers, w.lam, w.mu)) as g:
        st, T, gap = g.iterate(1e-12, 5)
        assert st == gpu.PSI_NOT_CONVERGED and T == 5 and gap > 1e-12
        assert len(g.get_residual_history()) == 5
        st, T, gap = g.iterate(1.0, 100)         # gap_0 = 1 is not > 1: T = 0 (Alg. 2)
        assert st == gpu.PSI_OK and T == 0 and gap == 1.0
        psi0 = g.get_psi().cpu().numpy()
        st, T, _ = g.iterate(0.0, 0)             # max_iters = 0 -> T = 0, same psi_0
        assert T == 0 and np.array_equal(g.get_psi().cpu().numpy(), psi0)
    import oracle
    ref = oracle.power_psi(w.row_ptr, w.followers, w.lam, w.mu, eps=1.0)
    assert ref.iterations == 0
    assert oracle.max_rel_error(ref.psi, psi0) < 1e-13


def test_single_user_and_edgeless(gpu):
    with gpu.PsiGraph(*dev(np.array([0, 0], np.int64), np.zeros(0, np.int32),
                           np.array([0.3]), np.array([0.7]))) as g:
        st, T, _ = g.iterate(1e-9)
        assert g.get_psi().cpu().numpy()[0] == pytest.approx(0.3)
    n = 5000
    lam = np.linspace(0.1, 1, n)
    mu = np.linspace(1, 0.1, n)
    with gpu.PsiGraph(*dev(np.zeros(n + 1, np.int64), np.zeros(0, np.int32), lam, mu)) as g:
        g.iterate(1e-9)
        np.testing.assert_allclose(g.get_psi().cpu().numpy(), lam / (lam + mu) / n, rtol=1e-15)


def test_numeric_divergence_reported(gpu):
    """A closed set whose leaders all have lambda = 0 (rho(A) = 1, reading R6): eps_t does not
    decay; the loop must stop at max_iters and say NOT_CONVERGED (never silent).  With the
    ROW norm ||B|| = 0 here (B = 0), so Alg. 2 stops after one sweep; use norm ONE."""
    rp, f = psigen.csr_from_edges(2, [(0, 1), (1, 0)])
    with gpu.PsiGraph(*dev(rp, f, np.zeros(2), np.ones(2))) as g:
        st, T, gap = g.iterate(1e-9, 50, norm="one")
        assert st == gpu.PSI_NOT_CONVERGED and T == 50
        assert np.all(g.get_residual_history() == 2.0)     # ||c^T A^t||_1 = 2 for all t
        st, T, gap = g.iterate(1e-9, 50, norm="row")
        assert st == gpu.PSI_OK and T == 1 and gap == 0.0


def test_library_pool_and_empty_cache(gpu):
    """the library allocates from its OWN pool (never the device's default pool):
    memory it caches after psi_destroy is returned by psi_empty_cache, after which torch can
    allocate it again."""
    import torch
    w = psigen.make_config(4, scale=20)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    free0, _ = torch.cuda.mem_get_info()
    d = dev(w.row_ptr, w.followers, w.lam, w.mu)
    with gpu.PsiGraph(*d) as g:
        g.iterate(w.eps)
    torch.cuda.synchronize()
    del d
    torch.cuda.empty_cache()
    free1, _ = torch.cuda.mem_get_info()
    gpu.empty_cache()
    free2, _ = torch.cuda.mem_get_info()
    assert free2 >= free1 and free0 - free2 < 64 << 20, (free0, free1, free2)
    x = torch.empty((free2 - (1 << 30)) // 8, dtype=torch.float64, device="cuda")
    del x
    torch.cuda.empty_cache()                       # give it back for the following tests


def test_power_nf_zero_iters_is_not_converged(gpu):
    """Alg. 1 with max_iters = 0 and eps < 1 leaves the loop with gap_0 = 1 > eps
    (Alg. 1 line 3), i.e. not converged, as psi_iterate reports it."""
    w = psigen.make_config(0)
    with gpu.PsiGraph(*dev(w.row_ptr, w.followers, w.lam, w.mu)) as g:
        st, p, q, it = g.power_nf([3, 5], 1e-9, 0)
        assert st == gpu.PSI_NOT_CONVERGED and list(it) == [0, 0]
        st, _, _ = g.iterate(1e-9, 0)
        assert st == gpu.PSI_NOT_CONVERGED
        st, p, q, it = g.power_nf([3], 2.0, 0)                 # eps >= 1: gap_0 <= eps
        assert st == gpu.PSI_OK


def test_history_length_counts_stored_entries(gpu):
    """psi_get_residual_history's len_out is the number of entries written."""
    w = psigen.make_config(0)
    with gpu.PsiGraph(*dev(w.row_ptr, w.followers, w.lam, w.mu)) as g:
        st, T, _ = g.iterate(0.0, 37)
        h = g.get_residual_history()
        assert T == 37 and len(h) == 37 and np.all(np.isfinite(h))
