"""Pins for the oracle's mini-batch operator B_b / B_{pi,b} (Eq. 12-13).

Every expected value here comes from outside oracle.c: worked examples
(golden/), closed forms, textbook special cases (b = n is the Bellman operator
T, b = 1 with ascending order the Gauss-Seidel operator F), exact
rational arithmetic, and the paper's (corrected, DESIGN readings R18) theory.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from conftest import golden, random_dense_mdp


def chain_mdp(g):
    m = g["mdp"]
    return oracle.MDP(m["n"], m["A"], m["gamma"], np.array(m["c"]), P=np.array(m["P"]))


def ident(n):
    return np.arange(n, dtype=np.uint32)


# ------------------------------------------------------------ worked example
def test_spec_chain_worked_examples():
    g = golden("spec_chain.json")
    m = chain_mdp(g)
    for case in g["cases"]:
        pi = np.array(case["policy"]) if "policy" in case else None
        V, _, _ = oracle.sweep(m, g["J"], case["b"], ident(2), pi)
        assert list(V) == case["expect"]


def test_shift_counterexample_E1():
    """Lemma 2's equality fails for b < n; the oracle must show it."""
    g = golden("spec_chain.json")
    m, ce = chain_mdp(g), g["shift_counterexample"]
    J = np.array(g["J"])
    V0, _, _ = oracle.sweep(m, J, ce["b"], ident(2))
    V1, _, _ = oracle.sweep(m, J + ce["r"], ce["b"], ident(2))
    assert list(V1 - V0) == ce["expect_shift"]


def test_ordering_counterexample_E2():
    g = golden("ordering_counterexample.json")
    n = g["n"]
    P = np.zeros((n, 1, n))
    for i in range(n - 1):
        P[i, 0, i] = 1.0
    P[n - 1, 0, n - 2] = 1.0
    m = oracle.MDP(n, 1, g["gamma"], np.ones((n, 1)), P=P)
    Vb, _, _ = oracle.sweep(m, np.zeros(n), g["b_big"], ident(n))
    Vs, _, _ = oracle.sweep(m, np.zeros(n), g["b_small"], ident(n))
    assert Vb[-1] == pytest.approx(g["expect_big_state7"], abs=1e-15)
    assert Vs[-1] == pytest.approx(g["expect_small_state7"], abs=1e-15)


# ---------------------------------------------------- textbook special cases
def bellman_T(m, J):
    """Textbook Bellman operator (Eq. 7) with numpy: min_a c + gamma P J."""
    Q = m.c.astype(np.float64) + m.gamma * np.einsum("saj,j->sa", m.to_dense64(), J)
    return Q.min(1), Q.argmin(1)


@pytest.mark.parametrize("seed", range(6))
def test_b_equals_n_is_bellman_operator(seed):
    rng = np.random.default_rng(seed)
    m = random_dense_mdp(rng, int(rng.integers(2, 30)), int(rng.integers(1, 6)), nonneg=False)
    J = rng.standard_normal(m.n) * 5
    TJ, _ = bellman_T(m, J)
    outs = []
    for k in range(3):   # any order: b = n reads only J
        V, _, r = oracle.sweep(m, J, m.n, oracle.partition(m.n, seed, k + 1))
        np.testing.assert_allclose(V, TJ, rtol=0, atol=1e-12)
        assert r == pytest.approx(np.abs(TJ - J).max(), abs=1e-12)
        outs.append(V)
    assert all(np.array_equal(outs[0], o) for o in outs)   # seed-independent, bitwise


@pytest.mark.parametrize("seed", range(4))
def test_b_equals_1_ascending_is_gauss_seidel(seed):
    """F of P:L139-143: FJ(i) uses FJ(j) for j < i and J(j) for j >= i."""
    rng = np.random.default_rng(100 + seed)
    m = random_dense_mdp(rng, int(rng.integers(2, 25)), int(rng.integers(1, 5)), nonneg=False)
    J = rng.standard_normal(m.n)
    P, c = m.to_dense64(), m.c.astype(np.float64)
    FJ = np.empty(m.n)
    for i in range(m.n):
        q = [c[i, u] + m.gamma * (P[i, u, :i] @ FJ[:i] + P[i, u, i:] @ J[i:]) for u in range(m.A)]
        FJ[i] = min(q)
    V, _, _ = oracle.sweep(m, J, 1, ident(m.n))
    np.testing.assert_allclose(V, FJ, rtol=0, atol=1e-12)


def test_policy_operator_at_b_equals_n_is_T_mu():
    rng = np.random.default_rng(7)
    m = random_dense_mdp(rng, 12, 3, nonneg=False)
    J = rng.standard_normal(12)
    mu = rng.integers(0, 3, 12).astype(np.int32)
    expect = m.c[np.arange(12), mu] + m.gamma * np.einsum("sj,j->s", m.P[np.arange(12), mu], J)
    V, arg, _ = oracle.sweep(m, J, 12, oracle.partition(12, 3, 3), mu)
    np.testing.assert_allclose(V, expect, atol=1e-12)
    assert np.array_equal(arg, mu)


def test_tie_break_lowest_index():
    # two identical actions: argmin must be 0 (reading R8)
    P = np.zeros((1, 3, 1)) + 1.0
    m = oracle.MDP(1, 3, 0.5, np.array([[2.0, 1.0, 1.0]]), P=P)
    _, arg, _ = oracle.sweep(m, np.zeros(1), 1, ident(1))
    assert arg[0] == 1


# --------------------------------------------------------------- closed forms
def test_backward_chain_closed_form():
    g = golden("backward_chain.json")
    for n, b, K in g["cases"]:
        P = np.zeros((n, 1, n))
        P[0, 0, 0] = 1.0
        for i in range(1, n):
            P[i, 0, i - 1] = 1.0
        c = np.ones((n, 1))
        c[0, 0] = 0.0
        m = oracle.MDP(n, 1, 0.5, c, P=P)
        res = oracle.vi(m, b, eps=1e-300, max_sweeps=4 * n, identity=True)
        # K sweeps reach V*, sweep K+1 has residual exactly 0
        assert res.sweeps == K + 1, (n, b, res.sweeps)
        assert res.trace[-1] == 0.0 and res.trace[-2] > 0.0
        # and the closed-form recurrence of the golden file agrees
        L, steps = 1, 0
        if b == 1:
            steps = 1
        else:
            while L < n:
                L += 1 + ((L + 1) % b == 0)
                steps += 1
        assert steps == K


@pytest.mark.parametrize("c,gamma", [(1.0, 0.95), (0.3, 0.5), (2.0, 0.99)])
def test_single_state_closed_form(c, gamma):
    m = oracle.MDP(1, 1, gamma, np.array([[c]]), P=np.ones((1, 1, 1)))
    eps = 1e-6
    res = oracle.vi(m, 1, eps=eps, max_sweeps=100000)
    K = res.sweeps
    k = np.arange(1, K + 1)
    np.testing.assert_allclose(res.trace, c * gamma ** (k - 1), rtol=1e-12, atol=64 * np.spacing(c / (1 - gamma)))
    assert c * gamma ** (K - 1) <= eps < c * gamma ** (K - 2)
    assert res.V[0] == pytest.approx(c * (1 - gamma**K) / (1 - gamma), rel=1e-13)


# ------------------------------------------------------------------- exactness
def test_rational_arithmetic_on_dyadic_instance():
    """Dyadic P (quarters), gamma = 1/2, integer costs: fp64 is exact, so the
    oracle must equal a Fraction evaluation of Eq. 12 bit for bit."""
    import gen
    n, A, b = 9, 3, 4
    P, c = gen.dense(n, A, 5, kind="dyadic", dtype=np.float64)
    m = oracle.MDP(n, A, 0.5, c, P=P)
    J = [Fraction(0)] * n
    V = np.zeros(n)
    for k in range(1, 8):
        perm = oracle.partition(n, 5, k)
        newJ = list(J)
        for lo in range(0, n, b):
            batch = [int(s) for s in perm[lo:lo + b]]
            vals = {}
            for s in batch:
                vals[s] = min(Fraction(c[s, a]) + Fraction(1, 2) * sum(
                    Fraction(P[s, a, j]) * newJ[j] for j in range(n)) for a in range(A))
            for s in batch:
                newJ[s] = vals[s]
        J = newJ
        V, _, _ = oracle.sweep(m, V, b, perm)
        assert [Fraction(v) for v in V] == J


# --------------------------------------------------- theory (sound statements)
def rand_pair(rng):
    n, A = int(rng.integers(2, 9)), int(rng.integers(1, 4))
    m = random_dense_mdp(rng, n, A, nonneg=False)
    return m, int(rng.integers(1, n + 1))


@pytest.mark.parametrize("seed", range(40))
def test_contraction_and_monotonicity(seed):
    """Prop. 3 and Lemma 1, 5 applications, fresh
    permutation per application, same permutations for both arguments."""
    rng = np.random.default_rng(seed)
    m, b = rand_pair(rng)
    J = rng.standard_normal(m.n) * 3
    Jp = J + np.abs(rng.standard_normal(m.n))          # J <= J'
    Jq = rng.standard_normal(m.n) * 3
    d0 = np.abs(J - Jq).max()
    for k in range(1, 6):
        perm = oracle.partition(m.n, seed, k)
        J, _, _ = oracle.sweep(m, J, b, perm)
        Jp, _, _ = oracle.sweep(m, Jp, b, perm)
        Jq, _, _ = oracle.sweep(m, Jq, b, perm)
        assert np.all(J <= Jp + 1e-12)
        assert np.abs(J - Jq).max() <= m.gamma**k * d0 + 1e-12


@pytest.mark.parametrize("seed", range(40))
def test_corrected_shift_bound(seed):
    """E1: for r >= 0, BJ + a^T r e <= B(J + r e) <= BJ + a r e, T = #batches;
    equality (the paper's Lemma 2) exactly when b = n."""
    rng = np.random.default_rng(1000 + seed)
    m, b = rand_pair(rng)
    J = rng.standard_normal(m.n)
    r = float(rng.uniform(0, 10))
    perm = oracle.partition(m.n, seed, 1)
    B0, _, _ = oracle.sweep(m, J, b, perm)
    B1, _, _ = oracle.sweep(m, J + r, b, perm)
    T = -(-m.n // b)
    shift = B1 - B0
    assert np.all(shift <= m.gamma * r + 1e-10)
    assert np.all(shift >= m.gamma**T * r - 1e-10)
    if b == m.n:
        np.testing.assert_allclose(shift, m.gamma * r, atol=1e-10)


@pytest.mark.parametrize("seed", range(20))
def test_fixed_point_lemma4(seed):
    """Lemma 4: J* (brute force) and J_mu are fixed points of
    B_b and B_{mu,b} for every b and order."""
    rng = np.random.default_rng(2000 + seed)
    n, A = int(rng.integers(1, 6)), int(rng.integers(1, 4))
    m = random_dense_mdp(rng, n, A, nonneg=False)
    Jstar = oracle.brute_force(m)
    mu = rng.integers(0, A, n).astype(np.int32)
    Jmu = oracle.policy_value(m, mu)
    for b in range(1, n + 1):
        perm = oracle.partition(n, seed, b)
        V, _, _ = oracle.sweep(m, Jstar, b, perm)
        assert np.abs(V - Jstar).max() <= 1e-9
        V, _, _ = oracle.sweep(m, Jmu, b, perm, mu)
        assert np.abs(V - Jmu).max() <= 1e-9


@pytest.mark.parametrize("seed", range(20))
def test_theorem6_nested_and_corollary7(seed):
    """Theorem 6 for nested b' | b (E2) and Corollary 7:
    T^k J <= B_b^k J <= F^k J <= J* for J = 0, c >= 0, same fixed order."""
    rng = np.random.default_rng(3000 + seed)
    n = int(rng.choice([4, 6, 8, 12]))
    m = random_dense_mdp(rng, n, int(rng.integers(1, 4)), nonneg=True)
    Jstar, _ = oracle.policy_iteration(m)
    perm = oracle.partition(n, seed, 1)
    divisors = [d for d in range(1, n + 1) if n % d == 0]
    Vs = {d: np.zeros(n) for d in divisors}
    for k in range(6):
        for d in divisors:
            Vs[d], _, _ = oracle.sweep(m, Vs[d], d, perm)
        for big in divisors:
            for small in divisors:
                if big % small == 0:           # nested pair
                    assert np.all(Vs[big] <= Vs[small] + 1e-12)
        assert np.all(Vs[1] <= Jstar + 1e-9)


@pytest.mark.parametrize("seed", range(20))
def test_monotone_from_below_with_fresh_permutations(seed):
    """c >= 0, V0 = 0: V_k nondecreasing and <= J* for any permutation sequence."""
    rng = np.random.default_rng(4000 + seed)
    m = random_dense_mdp(rng, int(rng.integers(2, 10)), int(rng.integers(1, 4)), nonneg=True)
    Jstar, _ = oracle.policy_iteration(m)
    b = int(rng.integers(1, m.n + 1))
    V = np.zeros(m.n)
    for k in range(1, 30):
        V2, _, _ = oracle.sweep(m, V, b, oracle.partition(m.n, seed, k))
        assert np.all(V2 >= V - 1e-13)
        assert np.all(V2 <= Jstar + 1e-9)
        V = V2


def test_csr_equals_dense_on_same_instance():
    import gen
    n, A, K = 40, 3, 8
    rp, col, val, c = gen.sparse(n, A, K, 11, dtype=np.float64)
    ms = oracle.MDP(n, A, 0.9, c, row_ptr=rp, col=col, val=val)
    md = oracle.MDP(n, A, 0.9, c, P=ms.to_dense64())
    J = np.random.default_rng(0).standard_normal(n)
    perm = oracle.partition(n, 1, 1)
    Vs, As, rs = oracle.sweep(ms, J, 7, perm)
    Vd, Ad, rd = oracle.sweep(md, J, 7, perm)
    np.testing.assert_allclose(Vs, Vd, atol=1e-13)
    assert np.array_equal(As, Ad)
