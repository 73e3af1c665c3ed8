"""Pins for the oracle's MB-VI / MB-MPI drivers against the plain definitions
(J* by brute force / exact PI, closed forms, the Bellman-VI special case)."""
import numpy as np
import pytest

import gen
import oracle
from conftest import random_dense_mdp


def gap_mask(m, V, tol):
    """States whose best and second-best Q differ by more than tol (reading A8)."""
    Q = m.c.astype(np.float64) + m.gamma * np.einsum("saj,j->sa", m.to_dense64(), V)
    if m.A == 1:
        return np.ones(m.n, bool)
    s = np.sort(Q, axis=1)
    return (s[:, 1] - s[:, 0]) > tol * np.maximum(1.0, np.abs(s[:, 0]))


@pytest.mark.parametrize("seed", range(12))
def test_vi_reaches_brute_force_optimum(seed):
    rng = np.random.default_rng(seed)
    n, A = int(rng.integers(1, 6)), int(rng.integers(1, 4))
    m = random_dense_mdp(rng, n, A, nonneg=False)
    Jstar = oracle.brute_force(m)
    b = int(rng.integers(1, n + 1))
    res = oracle.vi(m, b, seed=seed, eps=1e-10)
    assert res.status == oracle.OK
    # certificate from Prop. 3: ||V_K - J*|| <= gamma r_K / (1 - gamma)
    bound = m.gamma * res.trace[-1] / (1 - m.gamma)
    assert np.abs(res.V - Jstar).max() <= bound + 1e-12
    # greedy policy: optimal wherever the Q-gap is resolvable
    Q = m.c + m.gamma * np.einsum("saj,j->sa", m.P, Jstar)
    mask = gap_mask(m, Jstar, 1e-6)
    assert np.array_equal(res.pi[mask], Q.argmin(1)[mask])


@pytest.mark.parametrize("seed", range(10))
def test_error_envelope_prop5(seed):
    """||V_k - J*|| <= gamma^k ||V_0 - J*|| (Prop. 3 + Lemma 4), fresh orders."""
    rng = np.random.default_rng(50 + seed)
    m = random_dense_mdp(rng, int(rng.integers(2, 7)), int(rng.integers(1, 4)), nonneg=False)
    Jstar = oracle.brute_force(m)
    V = rng.standard_normal(m.n) * 4
    e0 = np.abs(V - Jstar).max()
    b = int(rng.integers(1, m.n + 1))
    for k in range(1, 25):
        V, _, _ = oracle.sweep(m, V, b, oracle.partition(m.n, seed, k))
        assert np.abs(V - Jstar).max() <= m.gamma**k * e0 + 1e-10


def test_fixed_order_residuals_contract():
    rng = np.random.default_rng(3)
    m = random_dense_mdp(rng, 20, 4, gamma=0.9)
    res = oracle.vi(m, 6, identity=True, eps=1e-9)
    r = res.trace
    assert np.all(r[1:] <= m.gamma * r[:-1] * (1 + 1e-9) + 1e-15)


@pytest.mark.parametrize("seed", range(5))
def test_smaller_nested_b_has_smaller_error(seed):
    """Theorem 6 / Cor. 7 (nested b, fixed order, c >= 0, V0 = 0): error to J*
    after k sweeps is ordered b=1 <= b=4 <= b=n (n = 16)."""
    rng = np.random.default_rng(70 + seed)
    m = random_dense_mdp(rng, 16, 3, nonneg=True, gamma=0.95)
    Jstar, _ = oracle.policy_iteration(m)
    errs = {}
    for b in (1, 4, 16):
        V = np.zeros(16)
        e = []
        for k in range(1, 40):
            V, _, _ = oracle.sweep(m, V, b, oracle.partition(16, 0, 0, identity=True))
            e.append(np.abs(V - Jstar).max())
        errs[b] = np.array(e)
    assert np.all(errs[1] <= errs[4] + 1e-12) and np.all(errs[4] <= errs[16] + 1e-12)


def test_mpi_b_n_m1_is_bellman_vi():
    """T_{greedy(V)} V = T V: MB-MPI with b = n, m = 1 follows Bellman VI exactly."""
    rng = np.random.default_rng(11)
    m = random_dense_mdp(rng, 15, 4)
    vi = oracle.vi(m, 15, eps=1e-12, max_sweeps=30)
    V = np.zeros(15)
    pi, _, _ = oracle.improve(m, V, np.zeros(15, np.int32))
    for k in range(30):
        V, _, _ = oracle.sweep(m, V, 15, oracle.partition(15, 0, k + 1), pi)
        pi, _, _ = oracle.improve(m, V, pi)
    res = oracle.mpi(m, 15, 1, eps=1e-300, max_outer=30)
    assert np.array_equal(res.V, V)
    np.testing.assert_array_equal(res.V, oracle.vi(m, 15, eps=1e-300, max_sweeps=30).V)
    assert res.status == oracle.NOT_CONVERGED and res.outer == 30


@pytest.mark.parametrize("seed", range(8))
def test_mpi_finds_optimal_policy(seed):
    rng = np.random.default_rng(90 + seed)
    n, A = int(rng.integers(2, 6)), int(rng.integers(2, 4))
    m = random_dense_mdp(rng, n, A, nonneg=False)
    Jstar = oracle.brute_force(m)
    b = int(rng.integers(1, n + 1))
    res = oracle.mpi(m, b, int(rng.integers(1, 5)), seed=seed, eps=1e-10)
    assert res.status == oracle.OK
    assert res.changed[-1] == 0
    # ||V - J*|| <= ||TV - V|| / (1 - gamma) at the last improvement
    assert np.abs(res.V - Jstar).max() <= res.trace[-1] / (1 - m.gamma) + 1e-12
    Q = m.c + m.gamma * np.einsum("saj,j->sa", m.P, Jstar)
    mask = gap_mask(m, Jstar, 1e-6)
    assert np.array_equal(res.pi[mask], Q.argmin(1)[mask])


def test_single_state_mpi_is_vi():
    # S:L262 "single-state MDP, K=1 -> identical trace to value_iteration"
    m = oracle.MDP(1, 1, 0.9, np.array([[1.0]]), P=np.ones((1, 1, 1)))
    v = oracle.vi(m, 1, eps=1e-6)
    p = oracle.mpi(m, 1, 1, eps=1e-6)
    assert np.array_equal(p.trace.reshape(-1, 2)[:, 0], v.trace[: p.outer])
    assert p.V[0] == pytest.approx(10.0, abs=1e-4)


def test_vi_status_codes():
    m = oracle.MDP(1, 1, 0.9, np.array([[1.0]]), P=np.ones((1, 1, 1)))
    assert oracle.vi(m, 1, eps=1e-6, max_sweeps=3).status == oracle.NOT_CONVERGED
    with pytest.raises(ValueError):
        oracle.vi(m, 2)
    bad = oracle.MDP(1, 1, 0.9, np.array([[np.inf]]), P=np.ones((1, 1, 1)))
    assert oracle.vi(bad, 1).status == oracle.NONFINITE


def test_config1_instance_converges_in_expected_sweeps():
    """BASELINE config 1 (dense 50x4, gamma .9, b=10, eps 1e-6): SURVEY
    Appendix A reports ~87 sweeps on a similar instance; we pin the range and
    the certificate against exact PI."""
    P, c = gen.dense(50, 4, 1, dtype=np.float64)
    m = oracle.MDP(50, 4, 0.9, c, P=P)
    res = oracle.vi(m, 10, seed=0, eps=1e-6)
    assert res.status == oracle.OK and 60 <= res.sweeps <= 140
    Jstar, mustar = oracle.policy_iteration(m)
    assert np.abs(res.V - Jstar).max() <= 0.9 * res.trace[-1] / 0.1 + 1e-12
