"""Input generator (psigen) host logic: validity, determinism, thread independence."""

import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest

import psigen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def check_csr(rp, f, n):
    assert rp.dtype == np.int64 and f.dtype == np.int32
    assert rp.shape == (n + 1,) and rp[0] == 0 and rp[-1] == f.shape[0]
    deg = np.diff(rp)
    assert np.all(deg >= 0)
    assert f.size == 0 or (f.min() >= 0 and f.max() < n)
    rows = np.repeat(np.arange(n), deg)
    assert not np.any(rows == f), "self loop"
    d = np.diff(f.astype(np.int64))
    same_row = rows[1:] == rows[:-1]
    assert np.all(d[same_row] > 0), "row not strictly increasing"


@pytest.mark.parametrize("k", [0, 1, 2])
def test_er_configs_valid(k):
    w = psigen.make_config(k)
    check_csr(w.row_ptr, w.followers, w.n)
    leaders_per_user = np.bincount(w.followers, minlength=w.n)
    assert leaders_per_user.min() >= 1                       # "each user >= 1 leader"
    mean = {0: 10, 1: 10, 2: 15}[k]
    assert abs(w.m / w.n - mean) < 0.05 * mean + 0.5
    assert np.all(w.lam > 0) and np.all(w.mu > 0)
    if k == 2:
        assert np.all(w.lam == 1.0) and np.all(w.mu == 1.0)
    else:
        assert w.lam.min() >= 0.05 and w.lam.max() < 1.0


def test_chung_lu_small_exact_m_and_power_law():
    rp, f = psigen.chung_lu_graph(1 << 16, 20 << 16, 2.1, 3000.0, seed=0)
    n = 1 << 16
    check_csr(rp, f, n)
    assert f.size == 20 << 16                                # top-up to exactly M
    indeg = np.diff(rp)                                      # followers per leader
    assert indeg.max() > 50 * indeg.mean()                   # heavy tail
    assert (np.bincount(f, minlength=n) == 0).any()          # leaderless users kept


def test_rmat_small_valid():
    w = psigen.make_config(5, scale=14)
    n = 1 << 14
    check_csr(w.row_ptr, w.followers, n)
    assert np.bincount(w.followers, minlength=n).min() >= 1
    assert int((w.mu == 0).sum()) == n // 20                 # exactly floor(0.05 N)
    assert 13 * n < w.m < 16 * n


def _digest(k, scale):
    w = psigen.make_config(k, scale=scale)
    h = hashlib.sha256()
    for a in (w.row_ptr, w.followers, w.lam, w.mu):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_deterministic_and_thread_count_independent():
    ref = _digest(4, 13)
    assert _digest(4, 13) == ref
    code = ("import sys; sys.path.insert(0, %r); import psigen, hashlib, numpy as np;"
            "w = psigen.make_config(4, scale=13); h = hashlib.sha256();"
            "[h.update(np.ascontiguousarray(a).tobytes()) for a in (w.row_ptr, w.followers, w.lam, w.mu)];"
            "print(h.hexdigest())") % ROOT
    env = dict(os.environ, OMP_NUM_THREADS="1")
    out = subprocess.check_output([sys.executable, "-c", code], env=env, text=True).strip()
    assert out == ref


def test_csr_from_edges():
    rp, f = psigen.csr_from_edges(4, [(1, 0), (3, 0), (2, 0), (0, 2), (1, 0)])
    assert rp.tolist() == [0, 3, 3, 4, 4] and f.tolist() == [1, 2, 3, 0]
    with pytest.raises(ValueError):
        psigen.csr_from_edges(3, [(1, 1)])


def test_activity_profiles_seeded_and_independent():
    """Batch profiles (row 4): seeded, profile-major (k, n), valid rates, independent draws,
    exactly floor(0.05 n) pure posters per profile when asked, the same arrays on every call."""
    import psigen
    n, k = 5000, 3
    lam, mu = psigen.activity_profiles(n, k, "lognormal", pure_posters=True)
    assert lam.shape == mu.shape == (k, n) and lam.flags.c_contiguous
    assert np.all(lam > 0) and np.all(mu >= 0) and np.all(lam + mu > 0)
    assert [(mu[j] == 0).sum() for j in range(k)] == [n // 20] * k
    assert not np.array_equal(lam[0], lam[1]) and not np.array_equal(mu[1], mu[2])
    lam2, mu2 = psigen.activity_profiles(n, k, "lognormal", pure_posters=True)
    assert np.array_equal(lam, lam2) and np.array_equal(mu, mu2)
    u, v = psigen.activity_profiles(n, 2, "uniform")
    assert u.min() >= 0.05 and u.max() <= 1.0 and v.min() >= 0.05 and v.max() <= 1.0
