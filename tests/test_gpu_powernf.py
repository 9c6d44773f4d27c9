"""GPU parity of batched Alg. 1 Power-NF (psi_power_nf, psi_nsystems) against
the oracle's power_nf / psi_power_nf (pinned in test_oracle_pins.py to the SPEC worked examples,
the dense balance-equation solve and Alg. 2).  Per origin: the same T, p_i and q_i to 1e-10."""

import ctypes
import json
import os

import numpy as np
import pytest

import oracle
import psigen
from oracle.power_nf import power_nf, psi_power_nf

pytestmark = pytest.mark.gpu

TOL = 1e-10
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def to_dev(*arrays):
    import torch
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrays]


def random_graph(rng, n, p):
    edges = [(i, j) for i in range(n) for j in range(n) if i != j and rng.random() < p]
    drop = set(rng.choice(n, size=max(1, n // 10), replace=False).tolist())
    edges = [(i, j) for (i, j) in edges if i not in drop]           # leaderless users
    lam, mu = rng.uniform(0.05, 1.0, n), rng.uniform(0.05, 1.0, n)
    pick = rng.permutation(n)
    mu[pick[: n // 10]] = 0.0                                        # pure posters
    lam[pick[n // 10: n // 10 + n // 20]] = 0.0                      # pure re-posters
    rp, f = psigen.csr_from_edges(n, edges)
    return rp, f, lam, mu


def check_origins(psi, rp, f, lam, mu, origins, eps, max_iters):
    with psi.PsiGraph(*to_dev(rp, f, lam, mu)) as g:
        st, p, q, iters = g.power_nf(origins, eps, max_iters)
        p, q = p.cpu().numpy(), q.cpu().numpy()
    for c, i in enumerate(origins):
        r = power_nf(rp, f, lam, mu, origin=int(i), eps=eps, max_iters=max_iters)
        assert iters[c] == r.iterations, (i, iters[c], r.iterations)
        np.testing.assert_allclose(p[c], r.p, rtol=TOL, atol=1e-16)
        np.testing.assert_allclose(q[c], r.q, rtol=TOL, atol=1e-16)
    return st


@pytest.mark.parametrize("name", ["chain", "mutual"])
def test_power_nf_spec_fixtures(gpu, name):
    with open(os.path.join(GOLD, "spec_examples.json")) as fh:
        case = json.load(fh)[name]
    rp, f = psigen.csr_from_edges(case["n"], case["edges"])
    lam, mu = np.array(case["lam"]), np.array(case["mu"])
    with gpu.PsiGraph(*to_dev(rp, f, lam, mu)) as g:
        st, p, q, iters = g.power_nf([case["power_nf_origin"]], 1e-15)
    np.testing.assert_allclose(p.cpu().numpy()[0], case["p"], atol=1e-14)
    np.testing.assert_allclose(q.cpu().numpy()[0], case["q"], atol=1e-14)


@pytest.mark.parametrize("seed", range(6))
def test_power_nf_random_fixed_count_and_eps(gpu, seed):
    """Leaderless, mu = 0 and lambda = 0 users; 40 origins = two batches (one partial)."""
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(40, 90))
    rp, f, lam, mu = random_graph(rng, n, float(rng.uniform(0.05, 0.2)))
    origins = rng.choice(n, size=min(n, 40), replace=False)
    check_origins(gpu, rp, f, lam, mu, origins, 0.0, 25)        # fixed count
    check_origins(gpu, rp, f, lam, mu, origins, 1e-10, 10_000)  # each origin's own stop
    check_origins(gpu, rp, f, lam, mu, origins[:3], 1.0, 100)   # eps >= 1: p = b_i, T = 0


def test_power_nf_config0_nsystems(gpu):
    """Config 0 (the N = 64 companion of config 1): psi by N runs of Alg. 1, same T_i sum."""
    w = psigen.make_config(0)
    ref, Ts = psi_power_nf(w.row_ptr, w.followers, w.lam, w.mu, eps=1e-12)
    with gpu.PsiGraph(*to_dev(w.row_ptr, w.followers, w.lam, w.mu)) as g:
        st, psi_v, mv = g.nsystems(1e-12)
    assert st == gpu.PSI_OK and mv == int(Ts.sum())
    assert oracle.max_rel_error(ref, psi_v.cpu().numpy()) <= TOL


def test_nsystems_config1_matches_power_psi(gpu):
    """Config 1 (N = 10,000): the N-systems psi (Alg. 1 x N, Eq. (1)) and Power-psi (Alg. 2)
    solve the same system (Eq. (12))."""
    w = psigen.make_config(1)
    with gpu.PsiGraph(*to_dev(w.row_ptr, w.followers, w.lam, w.mu)) as g:
        st, psi_nf, mv = g.nsystems(1e-13)
        g.iterate(1e-14)
        psi_v = g.get_psi().cpu().numpy()
    assert st == gpu.PSI_OK and mv > 10 * w.n
    # both against the oracle's converged Alg. 2 (not against each other): the N-systems
    # psi stops each origin at ||p - p_old||_1 <= 1e-13, so it is within ~1e-11 of the limit
    ref = oracle.power_psi(w.row_ptr, w.followers, w.lam, w.mu, eps=1e-15).psi
    assert oracle.max_rel_error(ref, psi_v) <= 1e-10
    assert oracle.max_rel_error(ref, psi_nf.cpu().numpy()) < 1e-9
    assert abs(psi_nf.cpu().numpy().sum() - 1.0) < 1e-9


def test_power_nf_host_outputs_and_errors(gpu):
    w = psigen.make_config(0)
    lib = gpu.load_library()
    with gpu.PsiGraph(*to_dev(w.row_ptr, w.followers, w.lam, w.mu)) as g:
        org = np.array([5, 7], dtype=np.int32)
        p = np.zeros((2, w.n))
        q = np.zeros((2, w.n))
        it = np.zeros(2, dtype=np.int64)
        st = lib.psi_power_nf(g._ctx, org.ctypes.data, 2, 1e-12, 1000, p.ctypes.data,
                              q.ctypes.data, gpu.PSI_MEM_HOST, it.ctypes.data)
        assert st == gpu.PSI_OK
        r = power_nf(w.row_ptr, w.followers, w.lam, w.mu, origin=7, eps=1e-12)
        np.testing.assert_allclose(q[1], r.q, rtol=TOL, atol=1e-16)
        with pytest.raises(gpu.PsiError):
            g.power_nf([w.n], 1e-9)                             # origin out of range
        with pytest.raises(gpu.PsiError):
            g.power_nf([0], -1.0)                               # bad eps
        st, p2, q2, it2 = g.power_nf([3], 0.0, 2)               # max_iters reached
        assert st == gpu.PSI_NOT_CONVERGED and it2[0] == 2
