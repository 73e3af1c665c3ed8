"""The properties that pin ASYNCHRONOUS MB-VI (
DESIGN reading R31), checked here on a CPU model of every allowed interleaving.

Asynchronous applications are not deterministic, so the GPU results are
compared with what is unique: the Bellman (Jacobi) iterates U_k = T^k V0 and
J*, both from the oracle.  R31 lets a backup read, for every successor j, any
value j held since the application began.  For V0 with T V0 <= V0 that gives,
for every interleaving (induction on the writes; T is monotone, Lemma 3):

    J* <= V_k <= U_k,   V_k <= V_{k-1},   T V_k <= V_k,

and the mirror image for T V0 >= V0.  These tests check the sandwich on a
random-interleaving model, and that a model which reads values OLDER than the
application start (a stale-cache bug) breaks it -- so the GPU tests built on
it can tell a correct asynchronous kernel from a broken one.
"""
import numpy as np
import pytest

import oracle
from conftest import random_dense_mdp


def _T(m, V):
    return (m.c.astype(np.float64) + m.gamma * np.einsum("saj,j->sa", m.to_dense64(), V)).min(1)


def async_model(m, V, order, rng, stale=False, hist=None):
    """One asynchronous application: states in `order`; each backup reads, per
    successor j, a random value from j's history since the application began
    (its start value or its new value if already written).  stale=True also
    allows the value j had one application earlier (hist)."""
    P = m.to_dense64()
    c = m.c.astype(np.float64)
    start = V.copy()
    new = V.copy()
    written = np.zeros(m.n, bool)
    for s in order:
        r = np.where(written & (rng.random(m.n) < 0.5), new, start)
        if stale and hist is not None:
            r = np.where(rng.random(m.n) < 0.5, hist, r)
        new[s] = (c[s] + m.gamma * P[s] @ r).min()
        written[s] = True
    return new


@pytest.mark.parametrize("seed", range(12))
def test_async_sandwich_upper_start(seed):
    rng = np.random.default_rng(seed)
    m = random_dense_mdp(rng, int(rng.integers(3, 20)), int(rng.integers(1, 4)), nonneg=True)
    Jstar = oracle.vi(m, m.n, eps=1e-13, max_sweeps=100000, identity=True).V
    V0 = np.full(m.n, m.c.max() / (1 - m.gamma))
    assert (_T(m, V0) <= V0 + 1e-12).all()
    V, U = V0.copy(), V0.copy()
    for k in range(1, 25):
        Vn = async_model(m, V, oracle.partition(m.n, seed, k), rng)
        U = oracle.sweep(m, U, m.n, oracle.partition(m.n, 0, 1))[0]      # Jacobi iterate T^k V0
        tol = 1e-12 * max(1.0, np.abs(V0).max())
        assert (Vn <= U + tol).all() and (Vn >= Jstar - tol).all()
        assert (Vn <= V + tol).all()
        assert (_T(m, Vn) <= Vn + tol).all()
        V = Vn


@pytest.mark.parametrize("seed", range(8))
def test_async_sandwich_lower_start(seed):
    rng = np.random.default_rng(100 + seed)
    m = random_dense_mdp(rng, int(rng.integers(3, 20)), int(rng.integers(1, 4)), nonneg=True)
    Jstar = oracle.vi(m, m.n, eps=1e-13, max_sweeps=100000, identity=True).V
    V, U = np.zeros(m.n), np.zeros(m.n)             # c >= 0: T 0 >= 0
    for k in range(1, 25):
        Vn = async_model(m, V, oracle.partition(m.n, seed, k), rng)
        U = oracle.sweep(m, U, m.n, oracle.partition(m.n, 0, 1))[0]
        tol = 1e-12 * max(1.0, np.abs(Jstar).max())
        assert (Vn >= U - tol).all() and (Vn <= Jstar + tol).all() and (Vn >= V - tol).all()
        V = Vn


def test_stale_reads_break_the_sandwich():
    """Reading values from before the application start (what a stale L1 line
    would return) violates V_k <= V_{k-1} or V_k <= U_k on some instance."""
    broken = 0
    for seed in range(30):
        rng = np.random.default_rng(500 + seed)
        m = random_dense_mdp(rng, 8, 2, nonneg=True)
        V0 = np.full(m.n, m.c.max() / (1 - m.gamma))
        V, U, hist = V0.copy(), V0.copy(), V0.copy()
        for k in range(1, 8):
            Vn = async_model(m, V, oracle.partition(m.n, seed, k), rng, stale=True, hist=hist)
            U = oracle.sweep(m, U, m.n, oracle.partition(m.n, 0, 1))[0]
            tol = 1e-12 * V0.max()
            if (Vn > U + tol).any() or (Vn > V + tol).any():
                broken += 1
                break
            hist, V = V, Vn
    assert broken > 0


def test_gauss_seidel_and_jacobi_are_two_interleavings():
    """The two extreme interleavings are the textbook operators: all-fresh reads
    in order = Gauss-Seidel (B_1), all-start reads = Bellman T (B_n)."""
    rng = np.random.default_rng(3)
    m = random_dense_mdp(rng, 10, 3)
    V = rng.normal(size=10)
    order = oracle.partition(10, 1, 1)
    P, c = m.to_dense64(), m.c.astype(np.float64)
    fresh = V.copy()
    for s in order:
        fresh[s] = (c[s] + m.gamma * P[s] @ fresh).min()
    assert np.allclose(fresh, oracle.sweep(m, V, 1, order)[0], atol=1e-12, rtol=0)
    assert np.allclose(_T(m, V), oracle.sweep(m, V, 10, order)[0], atol=1e-12, rtol=0)
