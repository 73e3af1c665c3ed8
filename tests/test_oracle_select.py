"""Pins for the oracle's state selection WITH replacement (SURVEY 8(f) row 4,
PAPER.md L605: "sampling the states with replacement and/or according to a
non-uniform distribution ... importance-sampling ... epsilon-greedy"), DESIGN
readings R28-R29, and for MB-VI / MB-MPI driven by it.

The paper gives no law for these draws, so R28-R29 fix one; these tests pin
the oracle to values that do not come from it: an independent pure-Python
reading of the R28-R29 text, numpy.searchsorted (the inverse-CDF library
routine), chi-square goodness of fit, textbook Gauss-Seidel / Jacobi sweeps
written with numpy, brute-force J* and exact policy iteration.
"""
import bisect
import itertools

import numpy as np
import pytest

import oracle
from conftest import random_dense_mdp

M64 = (1 << 64) - 1


def _mix(z):
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _py_select(n, seed, k, w=None):
    """DESIGN R28-R29 read independently: skey_k, u_i = mix64(skey_k + i),
    s = floor(u n / 2^64) or the first s whose inclusive prefix weight exceeds
    floor(u W / 2^64)."""
    key = _mix(_mix(seed) ^ k)
    skey = _mix(key ^ 0x5E1EC7105E1EC710)
    out = []
    cum = list(itertools.accumulate(int(x) for x in w)) if w is not None else None
    for i in range(n):
        u = _mix((skey + i) & M64)
        if w is None:
            out.append((u * n) >> 64)
        else:
            t = (u * cum[-1]) >> 64
            out.append(bisect.bisect_right(cum, t))
    return np.array(out, dtype=np.uint32)


@pytest.mark.parametrize("n,seed,k", [(1, 0, 1), (2, 5, 3), (10, 1, 1), (97, 42, 7), (1000, 2**63 + 5, 12)])
def test_independent_python_reading_uniform(n, seed, k):
    assert np.array_equal(oracle.select(n, seed, k), _py_select(n, seed, k))


@pytest.mark.parametrize("n,seed,k", [(1, 0, 1), (3, 9, 2), (50, 4, 4), (777, 11, 31)])
def test_independent_python_reading_weighted(n, seed, k):
    rng = np.random.default_rng(n + seed)
    w = rng.integers(1, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    assert np.array_equal(oracle.select(n, seed, k, w), _py_select(n, seed, k, [int(x) for x in w]))


def test_weighted_is_numpy_inverse_cdf():
    """s_i = searchsorted(cumsum(w), t_i, 'right') with t_i = floor(u_i W / 2^64)."""
    n, seed, k = 4099, 8, 5
    rng = np.random.default_rng(3)
    w = rng.integers(1, 1000, size=n).astype(np.uint32)
    cum = np.cumsum(w.astype(np.uint64))
    skey = _mix(_mix(_mix(seed) ^ k) ^ 0x5E1EC7105E1EC710)
    t = np.array([(_mix((skey + i) & M64) * int(cum[-1])) >> 64 for i in range(n)], dtype=np.uint64)
    assert np.array_equal(oracle.select(n, seed, k, w), np.searchsorted(cum, t, side="right").astype(np.uint32))


def test_all_ones_weights_are_uniform_draws():
    for n in (1, 7, 1000, 65_537):
        assert np.array_equal(oracle.select(n, 3, 2), oracle.select(n, 3, 2, np.ones(n, np.uint32)))


def test_zero_weight_and_bad_n_rejected():
    with pytest.raises(ValueError):
        oracle.select(4, 1, 1, np.array([1, 0, 1, 1], np.uint32))
    with pytest.raises(ValueError):
        oracle.select(0, 1, 1)


def _chi2_ok(counts, probs, alpha=1e-6):
    from scipy.stats import chisquare
    exp = probs * counts.sum()
    return chisquare(counts, exp).pvalue > alpha


def test_uniform_draws_chi_square():
    n, K = 64, 3000
    cnt = np.zeros(n)
    for k in range(1, K + 1):
        cnt += np.bincount(oracle.select(n, 17, k), minlength=n)
    assert _chi2_ok(cnt, np.full(n, 1.0 / n))
    # with replacement: the number of distinct states per sweep is ~ n(1 - (1-1/n)^n)
    d = np.mean([len(np.unique(oracle.select(n, 17, k))) for k in range(1, 401)])
    assert abs(d - n * (1 - (1 - 1 / n) ** n)) < 0.5


def test_weighted_draws_chi_square_and_extremes():
    n, K = 40, 2000
    w = np.arange(1, n + 1, dtype=np.uint32) ** 2
    cnt = np.zeros(n)
    for k in range(1, K + 1):
        cnt += np.bincount(oracle.select(n, 5, k, w), minlength=n)
    assert _chi2_ok(cnt, w / w.sum())
    # a dominant weight: P(other) = 99 / (1e9 + 99) -- essentially every draw is state 0
    w2 = np.ones(100, np.uint32)
    w2[0] = 10**9
    assert (oracle.select(100, 1, 1, w2) == 0).all()
    # a single heavy state among light ones is drawn in proportion
    w3 = np.ones(1000, np.uint32)
    w3[500] = 1000
    hits = sum(int((oracle.select(1000, 9, k, w3) == 500).sum()) for k in range(1, 101))
    assert abs(hits / 100 - 500) < 5 * np.sqrt(500)


def _q(m, V):
    return m.c.astype(np.float64) + m.gamma * np.einsum("saj,j->sa", m.to_dense64(), V)


def _textbook_sweep(m, V, b, sel, pi=None):
    """Eq. 12 / 13 over the batches of the draw sequence, with numpy backups and
    set semantics: each batch's distinct states are backed up against the same
    interim V, then written."""
    V = V.copy()
    r = 0.0
    for lo in range(0, m.n, b):
        states = sorted(set(int(s) for s in sel[lo:lo + b]))
        Q = _q(m, V)
        new = {s: (Q[s, pi[s]] if pi is not None else Q[s].min()) for s in states}
        for s, v in new.items():
            r = max(r, abs(v - V[s]))
            V[s] = v
    return V, r


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("weighted", [False, True])
def test_sweep_with_replacement_matches_textbook(seed, weighted):
    rng = np.random.default_rng(100 + seed)
    n, A = int(rng.integers(2, 30)), int(rng.integers(1, 5))
    m = random_dense_mdp(rng, n, A)
    w = rng.integers(1, 50, size=n).astype(np.uint32) if weighted else None
    sel = oracle.select(n, seed, 3, w)
    V0 = rng.normal(size=n)
    for b in sorted({1, 2, int(rng.integers(1, n + 1)), n}):
        V, _, r = oracle.sweep(m, V0, b, sel)
        Vt, rt = _textbook_sweep(m, V0, b, sel)
        assert np.allclose(V, Vt, rtol=0, atol=1e-12)
        assert abs(r - rt) <= 1e-12
        # states never drawn keep their values
        undrawn = np.setdiff1d(np.arange(n), sel)
        assert np.array_equal(V[undrawn], V0[undrawn])


def test_b1_with_replacement_is_gauss_seidel_in_draw_order():
    rng = np.random.default_rng(7)
    m = random_dense_mdp(rng, 12, 3)
    sel = oracle.select(12, 1, 1)
    V = rng.normal(size=12)
    Vgs = V.copy()
    for s in sel:                      # textbook GS: one state at a time, in place
        Vgs[s] = _q(m, Vgs)[s].min()
    assert np.allclose(oracle.sweep(m, V, 1, sel)[0], Vgs, rtol=0, atol=1e-12)


def test_bn_with_replacement_is_bellman_on_the_drawn_set():
    rng = np.random.default_rng(8)
    m = random_dense_mdp(rng, 20, 4)
    sel = oracle.select(20, 2, 5)
    V = rng.normal(size=20)
    TV = _q(m, V).min(1)
    exp = V.copy()
    drawn = np.unique(sel)
    exp[drawn] = TV[drawn]
    out, _, r = oracle.sweep(m, V, 20, sel)
    assert np.allclose(out, exp, rtol=0, atol=1e-12)
    assert abs(r - np.abs(TV[drawn] - V[drawn]).max()) <= 1e-12


@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("weighted", [False, True])
def test_vi_with_replacement_reaches_brute_force_optimum(seed, weighted):
    rng = np.random.default_rng(300 + seed)
    n, A = int(rng.integers(1, 6)), int(rng.integers(1, 4))
    m = random_dense_mdp(rng, n, A, nonneg=False)
    Jstar = oracle.brute_force(m)
    w = rng.integers(1, 9, size=n).astype(np.uint32) if weighted else None
    b = int(rng.integers(1, n + 1))
    res = oracle.vi(m, b, seed=seed, eps=1e-11, replace=True, weights=w, max_sweeps=200000)
    assert res.status == oracle.OK
    # R30: the sweep residual covers the drawn states only; the stop was
    # confirmed on all states, so ||TV - V|| <= eps and the certificate holds
    Q = _q(m, res.V)
    rT = np.abs(Q.min(1) - res.V).max()
    assert rT <= 1e-11 * (1 + 1e-9)
    assert np.abs(res.V - Jstar).max() <= rT / (1 - m.gamma) + 1e-12
    assert np.array_equal(res.pi, Q.argmin(1))   # pi = greedy(V) of the confirming pass


def test_premature_stop_is_caught_by_the_confirmation():
    """A draw sequence that misses a still-changing state: r_k <= eps but
    ||TV - V|| > eps -- the confirmation must keep sweeping (R30)."""
    rng = np.random.default_rng(307)
    seen = 0
    for seed in range(40):
        n = int(rng.integers(2, 6))
        m = random_dense_mdp(rng, n, 2, nonneg=False)
        res = oracle.vi(m, 1, seed=seed, eps=1e-11, replace=True, max_sweeps=200000)
        assert res.status == oracle.OK
        assert np.abs(_q(m, res.V).min(1) - res.V).max() <= 1e-11 * (1 + 1e-9)
        # sweeps after the first r_k <= eps exist when a confirmation failed
        first = int(np.argmax(res.trace <= 1e-11))
        seen += first < len(res.trace) - 1
    assert seen > 0


def test_vi_with_replacement_trace_and_draw_sequence():
    """orc_vi(select) applies sweep k with the draws of application k (k = 1, 2, ...)."""
    rng = np.random.default_rng(5)
    m = random_dense_mdp(rng, 15, 3)
    res = oracle.vi(m, 4, seed=9, eps=1e-300, max_sweeps=6, replace=True)
    assert res.status == oracle.NOT_CONVERGED
    V = np.zeros(15)
    for k in range(1, 7):
        V, r = _textbook_sweep(m, V, 4, oracle.select(15, 9, k))
        assert abs(r - res.trace[k - 1]) <= 1e-12
    assert np.allclose(res.V, V, rtol=0, atol=1e-12)


@pytest.mark.parametrize("seed", range(6))
def test_mpi_with_replacement_finds_policy_iteration_optimum(seed):
    rng = np.random.default_rng(500 + seed)
    m = random_dense_mdp(rng, int(rng.integers(2, 25)), int(rng.integers(2, 5)))
    Jpi, mu = oracle.policy_iteration(m)
    w = rng.integers(1, 20, size=m.n).astype(np.uint32) if seed % 2 else None
    res = oracle.mpi(m, int(rng.integers(1, m.n + 1)), 5, seed=seed, eps=1e-10, replace=True, weights=w)
    assert res.status == oracle.OK
    assert res.changed[-1] == 0
    # r_T of the last improvement is ||TV - V||, a certificate for any selection law
    assert np.abs(res.V - Jpi).max() <= res.trace[-1] / (1 - m.gamma) + 1e-12
    Q = _q(m, Jpi)
    s = np.sort(Q, axis=1)
    mask = (s[:, 1] - s[:, 0]) > 1e-9 * np.maximum(1, np.abs(s[:, 0]))
    assert np.array_equal(res.pi[mask], mu[mask])


def test_selection_rejects_chunked_and_identity():
    m = random_dense_mdp(np.random.default_rng(1), 5, 2)
    with pytest.raises(ValueError):
        oracle.vi(m, 2, replace=True, chunked=True)
    with pytest.raises(ValueError):
        oracle.vi(m, 2, replace=True, identity=True)
