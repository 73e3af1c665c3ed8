"""Edge cases of the SURVEY 8(f) row 4 variants and the error trace: tiny n
(fewer states than CTAs), one action, identity order, ragged fp64 rows,
max_sweeps reached -- each against the oracle or the R31 bounds."""
import numpy as np
import pytest
import torch

import gen
import oracle
import paper_2110_02901_b200 as rmb

pytestmark = pytest.mark.gpu


def tdev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def dense(n, A, seed, dtype=np.float32, flags=0, gamma=0.9):
    P, c = gen.dense(n, A, seed, dtype=dtype)
    return oracle.MDP(n, A, gamma, c, P=P), rmb.Problem.dense(tdev(P), tdev(c), gamma, flags=flags)


@pytest.mark.parametrize("n,A,dtype,flags", [(1, 3, np.float32, 0), (2, 1, np.float32, 0), (4, 2, np.float64, 0),
                                             (8, 5, np.float32, rmb.DENSE_NO_TMA), (7, 3, np.float64, 0),
                                             (100, 1, np.float32, 0)])
def test_async_tiny_and_degenerate(n, A, dtype, flags):
    m, prob = dense(n, A, n + A, dtype=dtype, flags=flags)
    ref = oracle.vi(m, n, eps=1e-13, max_sweeps=100000, identity=True).V
    for identity in (False, True):
        sol = prob.vi(1, eps=1e-12, max_sweeps=20000, asynchronous=True, identity=identity)
        assert sol.status == rmb.OK
        assert np.abs(sol.V.cpu().numpy() - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("n,b", [(1, 1), (2, 1), (2, 2), (5, 3)])
@pytest.mark.parametrize("kind", ["dense", "sparse"])
def test_replacement_tiny(n, b, kind):
    if kind == "dense":
        m, prob = dense(n, 3, 2 * n)
    else:
        rp, col, val, c = gen.sparse(n, 3, min(2, n), 5)
        m = oracle.MDP(n, 3, 0.9, c, row_ptr=rp, col=col, val=val)
        prob = rmb.Problem.csr(n, 3, tdev(rp), tdev(col), tdev(val), tdev(c), 0.9)
    sol = prob.vi(b, seed=1, eps=1e-10, max_sweeps=5000, select="replace")
    ref = oracle.vi(m, b, seed=1, eps=1e-10, max_sweeps=5000, replace=True)
    assert sol.status == ref.status == rmb.OK
    assert sol.stats.sweeps == ref.sweeps
    assert np.abs(sol.V.cpu().numpy() - ref.V).max() <= 1e-9 * max(1.0, np.abs(ref.V).max())


def test_error_trace_when_max_sweeps_is_reached():
    m, prob = dense(200, 4, 3)
    Vref = oracle.vi(m, 200, eps=1e-13, max_sweeps=100000, identity=True).V
    prob.set_reference(Vref)
    sol = prob.vi(20, seed=1, eps=1e-14, max_sweeps=7, trace_error=True)
    assert sol.status == rmb.NOT_CONVERGED
    assert len(sol.error) == 7
    V = np.zeros(200)
    for k in range(1, 8):
        V = oracle.sweep(m, V, 20, oracle.partition(200, 1, k))[0]
        assert abs(sol.error[k - 1] - np.abs(V - Vref).max()) <= 1e-10 * np.abs(Vref).max()


def test_weighted_selection_with_a_dominant_state():
    """All weight on one state (plus 1 elsewhere): nearly every draw is that
    state, the rest are still drawn eventually -- the stop stays confirmed."""
    m, prob = dense(32, 3, 4)
    w = np.ones(32, np.uint32)
    w[5] = 1000
    prob.set_selection_weights(w)
    sol = prob.vi(4, seed=2, eps=1e-9, max_sweeps=200000, select="weighted")
    ref = oracle.vi(m, 4, seed=2, eps=1e-9, max_sweeps=200000, replace=True, weights=w)
    assert sol.status == ref.status == rmb.OK and sol.stats.sweeps == ref.sweeps
    assert np.abs(sol.V.cpu().numpy() - ref.V).max() <= 1e-9 * max(1.0, np.abs(ref.V).max())
