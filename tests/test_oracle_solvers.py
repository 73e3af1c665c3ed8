"""Pins for the oracle's MB-VI / MB-MPI drivers against the plain definitions
(J* by brute force / exact PI, closed forms, the Bellman-VI special case)."""
import numpy as np
import pytest

import gen
import oracle
from conftest import golden, random_dense_mdp


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


# ------------------------------------------------ policy improvement (Alg. 1)
def textbook_improve(m, V, pi):
    """Alg. 1's improvement line written with numpy: Q = c + a P V,
    pi' = argmin (np.argmin: first minimum = lowest index on ties, reading R8),
    changed = #{pi' != pi}, r_T = max |min_a Q - V| (reading R11)."""
    Q = m.c.astype(np.float64) + m.gamma * np.einsum("saj,j->sa", m.to_dense64(), V)
    new = Q.argmin(1).astype(np.int32)
    return new, float(np.abs(Q.min(1) - V).max()), int((new != pi).sum()), Q


def test_improve_worked_example():
    g = golden("improve_worked.json")
    n, A = g["mdp"]["n"], g["mdp"]["A"]
    P = np.zeros((n, A, n))
    for s in range(n):
        for a in range(A):
            P[s, a, a] = 1.0
    m = oracle.MDP(n, A, g["mdp"]["gamma"], np.array(g["mdp"]["c"]), P=P)
    pi, rT, ch = oracle.improve(m, np.array(g["V"]), np.array(g["pi_in"], np.int32))
    assert list(pi) == g["expect_pi"]
    assert rT == g["expect_bellman_resid"]
    assert ch == g["expect_changed"]


@pytest.mark.parametrize("seed", range(10))
def test_improve_matches_textbook_random(seed):
    """pi', changed and ||TV - V|| against the numpy textbook improvement on
    random dense MDPs (states whose two best Q are closer than 1e-9 relative
    are excluded from the action comparison: einsum sums in another order)."""
    rng = np.random.default_rng(300 + seed)
    n, A = int(rng.integers(2, 40)), int(rng.integers(1, 7))
    m = random_dense_mdp(rng, n, A, nonneg=bool(seed % 2))
    V = rng.standard_normal(n) * 5
    pi = rng.integers(0, A, n).astype(np.int32)
    new, rT, ch, Q = textbook_improve(m, V, pi)
    got, grT, gch = oracle.improve(m, V, pi)
    mask = gap_mask(m, V, 1e-9)
    assert np.array_equal(got[mask], new[mask])
    assert abs(grT - rT) <= 1e-12 * max(1.0, np.abs(V).max())
    if mask.all():
        assert gch == ch
    assert gch == int((got != pi).sum())


@pytest.mark.parametrize("seed", range(6))
def test_improve_matches_textbook_exact_ties(seed):
    """Dyadic instance, gamma = 1/2, dyadic V: every Q is exact in fp64, so the
    textbook improvement is exact too -- including the exact ties of
    deterministic rows; pi', changed and r_T must agree bit for bit."""
    import gen
    n, A = 24, 4
    P, c = gen.dense(n, A, seed, kind="dyadic", dtype=np.float64)
    m = oracle.MDP(n, A, 0.5, c, P=P)
    rng = np.random.default_rng(seed)
    # seed 0: V = 0, so Q = c (integer costs): exact ties are certain
    V = rng.integers(-8, 9, n).astype(np.float64) / 4 if seed else np.zeros(n)
    pi = rng.integers(0, A, n).astype(np.int32)
    new, rT, ch, Q = textbook_improve(m, V, pi)
    ties = int((np.sort(Q, 1)[:, 0] == np.sort(Q, 1)[:, 1]).sum())
    got, grT, gch = oracle.improve(m, V, pi)
    assert np.array_equal(got, new) and grT == rT and gch == ch
    if seed == 0:
        assert ties > 0  # the instance does exercise the tie rule


def test_improve_changed_counts_against_input_policy():
    """changed counts against the policy on entry (not against pi' of a
    previous call): improving twice gives changed = 0 the second time."""
    rng = np.random.default_rng(7)
    m = random_dense_mdp(rng, 30, 5)
    V = rng.random(30)
    pi0 = np.zeros(30, np.int32)
    p1, _, c1 = oracle.improve(m, V, pi0)
    p2, _, c2 = oracle.improve(m, V, p1)
    assert c1 == int((p1 != pi0).sum()) and c1 > 0
    assert c2 == 0 and np.array_equal(p1, p2)


def test_improve_csr_matches_dense():
    """The CSR improvement equals the same MDP given densely (the textbook
    improvement over the scattered rows)."""
    import gen
    n, A, K = 60, 3, 5
    rp, col, val, c = gen.sparse(n, A, K, 4, dtype=np.float64)
    ms = oracle.MDP(n, A, 0.9, c, row_ptr=rp, col=col, val=val)
    rng = np.random.default_rng(4)
    V = rng.random(n) * 3
    pi = rng.integers(0, A, n).astype(np.int32)
    new, rT, ch, Q = textbook_improve(ms, V, pi)
    got, grT, gch = oracle.improve(ms, V, pi)
    mask = gap_mask(ms, V, 1e-9)
    assert np.array_equal(got[mask], new[mask])
    assert abs(grT - rT) <= 1e-12 * max(1.0, np.abs(V).max())


# ------------------------------------------------------------ VI*
@pytest.mark.parametrize("seed", range(6))
def test_chunked_T_is_bellman_operator(seed):
    """VI*'s chunked operator (every chunk against the old values) is
    T: equal to the numpy Bellman operator to rounding and BITWISE equal to the
    one-batch sweep B_n for every chunk size and order; with a policy
    it is T_pi."""
    rng = np.random.default_rng(400 + seed)
    n, A = int(rng.integers(2, 30)), int(rng.integers(1, 5))
    m = random_dense_mdp(rng, n, A, nonneg=False)
    V = rng.standard_normal(n)
    Tn, an, rn = oracle.sweep(m, V, n, np.arange(n, dtype=np.uint32))
    Q = m.c + m.gamma * np.einsum("saj,j->sa", m.P, V)
    for c in sorted({1, 2, max(1, n // 3), n}):
        perm = oracle.partition(n, seed, c)
        Vc, ac, rc = oracle.sweep_chunked(m, V, c, perm)
        assert np.array_equal(Vc, Tn) and rc == rn
        assert np.abs(Vc - Q.min(1)).max() <= 1e-12 * max(1.0, np.abs(Q).max())
        mask = gap_mask(m, V, 1e-9)
        assert np.array_equal(ac[mask], Q.argmin(1)[mask])
    pi = rng.integers(0, A, n).astype(np.int32)
    Tp, _, _ = oracle.sweep(m, V, n, np.arange(n, dtype=np.uint32), pi)
    Vp, _, _ = oracle.sweep_chunked(m, V, max(1, n // 2), oracle.partition(n, 1, 1), pi)
    assert np.array_equal(Vp, Tp)


def test_chunked_differs_from_minibatch():
    """The chunked T is not B_b: with b < n the mini-batch operator uses the
    interim values (SPEC chain: B_1 gives (2, 2), T in chunks of 1 gives (2, 3))."""
    g = golden("spec_chain.json")
    mm = g["mdp"]
    m = oracle.MDP(mm["n"], mm["A"], mm["gamma"], np.array(mm["c"]), P=np.array(mm["P"]))
    Vc, _, _ = oracle.sweep_chunked(m, g["J"], 1, np.arange(2, dtype=np.uint32))
    assert list(Vc) == [2.0, 3.0]


def test_vi_star_equals_bellman_vi():
    rng = np.random.default_rng(5)
    m = random_dense_mdp(rng, 40, 4, gamma=0.95)
    a = oracle.vi(m, 40, eps=1e-8)
    for c in (1, 7, 40):
        s = oracle.vi(m, c, seed=3, eps=1e-8, chunked=True)
        assert s.sweeps == a.sweeps and np.array_equal(s.V, a.V) and np.array_equal(s.trace, a.trace)
        assert np.array_equal(s.pi, a.pi)


# ------------------------------------------------------- worker threads
def test_threads_are_bitwise_invisible():
    """Worker threads split one batch's states; each row sum stays sequential,
    so sweeps, improvements and whole solves are bitwise independent of W."""
    import gen
    rng = np.random.default_rng(9)
    m = random_dense_mdp(rng, 120, 6)
    rp, col, val, c = gen.sparse(300, 4, 8, 2)
    ms = oracle.MDP(300, 4, 0.97, c, row_ptr=rp, col=col, val=val)
    out = {}
    try:
        for w in (1, 4):
            oracle.set_threads(w)
            assert oracle.get_threads() == w
            out[w] = (oracle.vi(m, 17, seed=2, eps=1e-9), oracle.mpi(ms, 50, 3, seed=1, eps=1e-9),
                      oracle.improve(m, np.linspace(0, 1, 120), np.zeros(120, np.int32)),
                      oracle.sweep_chunked(m, np.ones(120), 30, oracle.partition(120, 0, 1)))
    finally:
        oracle.set_threads(1)
    a, b = out[1], out[4]
    for x, y in ((a[0], b[0]), (a[1], b[1])):
        assert x.sweeps == y.sweeps and np.array_equal(x.V, y.V) and np.array_equal(x.pi, y.pi)
        assert np.array_equal(x.trace, y.trace)
    assert np.array_equal(a[2][0], b[2][0]) and a[2][1] == b[2][1] and a[2][2] == b[2][2]
    assert np.array_equal(a[3][0], b[3][0])


def test_mpi_driver_is_alg1_composition():
    """orc_mpi is Algorithm 1 composed from the pinned primitives:
    pi_0 = greedy(V0), then per outer iteration m applications of B_{pi,b}, the
    k-th with ITS OWN partition (sweep counter k = 1, 2, ... across outer
    iterations, reading R3), then the improvement; stop when changed = 0 and
    r_T <= eps (reading R11).  Checked bitwise, b < n so the order matters."""
    rng = np.random.default_rng(21)
    n, A, b, msw, eps = 25, 3, 4, 3, 1e-9
    m = random_dense_mdp(rng, n, A, gamma=0.9)
    V = np.zeros(n)
    pi, _, _ = oracle.improve(m, V, np.zeros(n, np.int32))
    k, tr, chg = 1, [], []
    for o in range(200):
        for e in range(msw):
            V, _, r = oracle.sweep(m, V, b, oracle.partition(n, 5, k), pi)
            tr.append(r)
            k += 1
        pi, rT, ch = oracle.improve(m, V, pi)
        tr.append(rT)
        chg.append(ch)
        if ch == 0 and rT <= eps:
            break
    res = oracle.mpi(m, b, msw, seed=5, eps=eps)
    assert res.status == oracle.OK and res.outer == len(chg) and res.sweeps == k - 1
    assert np.array_equal(res.V, V) and np.array_equal(res.pi, pi)
    assert np.array_equal(res.trace, np.array(tr)) and list(res.changed) == chg


def test_vi_driver_is_composition():
    """orc_vi: sweep k uses partition k (k = 1, 2, ...), stop at the first r_k <= eps."""
    rng = np.random.default_rng(22)
    n, b, eps = 30, 7, 1e-7
    m = random_dense_mdp(rng, n, 4, gamma=0.9)
    V, tr = np.zeros(n), []
    for k in range(1, 1000):
        V, pi, r = oracle.sweep(m, V, b, oracle.partition(n, 9, k))
        tr.append(r)
        if r <= eps:
            break
    res = oracle.vi(m, b, seed=9, eps=eps)
    assert res.sweeps == len(tr) and np.array_equal(res.V, V) and np.array_equal(res.pi, pi)
    assert np.array_equal(res.trace, np.array(tr))


def test_bellman_residual_by_row_regeneration():
    """The config-5 certificate routine (rows regenerated on the host) equals
    ||T V - V|| computed from the stored instance with the numpy textbook
    Bellman operator, for f32 and f64 storage."""
    n, A, gamma = 90, 5, 0.97
    V = np.random.default_rng(0).random(n) * 30
    for f32 in (True, False):
        P, c = gen.dense(n, A, 3, dtype=np.float32 if f32 else np.float64)
        Q = c.astype(np.float64) + gamma * np.einsum("saj,j->sa", P.astype(np.float64), V)
        r, arg = oracle.bellman_residual_dense_gen(3, n, A, gamma, V, f32=f32)
        assert abs(r - np.abs(Q.min(1) - V).max()) <= 1e-12 * 30
        m = oracle.MDP(n, A, gamma, c, P=P)
        mask = gap_mask(m, V, 1e-9)
        assert np.array_equal(arg[mask], Q.argmin(1)[mask])
        r2, _ = oracle.bellman_residual_dense_gen(3, n, A, gamma, V, rows=(10, 40), f32=f32)
        assert abs(r2 - np.abs(Q.min(1) - V)[10:40].max()) <= 1e-12 * 30
