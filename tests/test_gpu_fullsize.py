"""Full-length solves at BASELINE.json's full sizes against the oracle
(north_star: "oracle-matching V/pi on every config"; SURVEY 8(d) "full parity
on 1 seed per b").

The GPU solves in the launch configuration bench.py times (instances generated
on the device); the oracle solves the same instance generated on the host
(gen/, bitwise equal to the device generator: test_gpu_dense.py), with its
worker threads splitting each batch's states (every row sum stays sequential,
so the oracle's result does not depend on the thread count).

Bar: equal sweep counts (+-1 only when the stopping
residual is within rounding of eps), residual traces and V within
1e-9 * max(1, ||V||), pi bit-exact where the Q-gap exceeds 1e-9 * max(1, |Q|),
MPI changed counts equal.
"""
import os

import numpy as np
import pytest
import torch

import gen
import oracle
import paper_2110_02901_b200 as rmb

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = 1e-9


@pytest.fixture(autouse=True, scope="module")
def _oracle_threads():
    oracle.set_threads(os.cpu_count() or 1)
    yield
    oracle.set_threads(1)


def tdev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def q_gap_dense(P, c, gamma, V, chunk=2000):
    """Relative gap between the two smallest Q(s, .) against V (fp64, rows in chunks)."""
    n, A = c.shape
    gap = np.empty(n)
    for s0 in range(0, n, chunk):
        s1 = min(n, s0 + chunk)
        Q = c[s0:s1].astype(np.float64) + gamma * (P[s0:s1].reshape(-1, P.shape[2]).astype(np.float64) @ V).reshape(
            s1 - s0, A)
        q = np.sort(Q, 1)
        gap[s0:s1] = (q[:, 1] - q[:, 0]) / np.maximum(1.0, np.abs(q[:, 0]))
    return gap


def q_gap_csr(n, A, rp, col, val, c, gamma, V):
    from scipy.sparse import csr_matrix
    M = csr_matrix((val.astype(np.float64), col, rp), shape=(n * A, n))
    Q = c.astype(np.float64) + gamma * (M @ V).reshape(n, A)
    q = np.sort(Q, 1)
    return (q[:, 1] - q[:, 0]) / np.maximum(1.0, np.abs(q[:, 0]))


def assert_vi_parity(sol, ref, eps):
    scale = max(1.0, float(np.abs(ref.V).max()))
    K, Ko = sol.stats.sweeps, ref.sweeps
    if K != Ko:  # reading A17: only when the stopping residual is within rounding of eps
        assert abs(K - Ko) == 1
        kk = min(K, Ko)
        assert abs(ref.trace[kk - 1] - eps) <= 1e-12 * scale or abs(sol.trace[kk - 1] - eps) <= 1e-12 * scale
        return False
    assert sol.status == ref.status
    assert np.abs(sol.trace - ref.trace).max() <= TOL * scale
    assert np.abs(sol.V.cpu().numpy() - ref.V).max() <= TOL * scale
    return True


@pytest.mark.parametrize("b", [1000, 64])
def test_config2_full_solve(b):
    """Config 2: dense 10^4 x 16, gamma 0.99, fp32 P (6.4 GB), MB-VI to 1e-6."""
    n, A, gamma, eps = 10_000, 16, 0.99, 1e-6
    Pd, cd = rmb.generate_dense(n, A, 1)
    prob = rmb.Problem.dense(Pd, cd, gamma)
    sol = prob.vi(b, seed=11, eps=eps, max_sweeps=5000)
    prob.close()
    del Pd, cd
    torch.cuda.empty_cache()
    P, c = gen.dense(n, A, 1)
    ref = oracle.vi(oracle.MDP(n, A, gamma, c, P=P), b, seed=11, eps=eps, max_sweeps=5000)
    assert ref.status == oracle.OK and 500 < ref.sweeps < 1500
    if assert_vi_parity(sol, ref, eps):
        mask = q_gap_dense(P, c, gamma, ref.V) > TOL
        assert mask.mean() > 0.99
        assert np.array_equal(sol.pi.cpu().numpy()[mask], ref.pi[mask])


def test_config3_full_solve():
    """Config 3: sparse 10^6 x 8 x 32 (ELL fp32), gamma 0.99, MB-VI b = n/8 to 1e-6."""
    n, A, K, gamma, eps, b = 1_000_000, 8, 32, 0.99, 1e-6, 125_000
    rpd, cold, vald, cd = rmb.generate_sparse(n, A, K, 1)
    prob = rmb.Problem.csr(n, A, rpd, cold, vald, cd, gamma)
    sol = prob.vi(b, seed=4, eps=eps, max_sweeps=5000)
    prob.close()
    del rpd, cold, vald, cd
    torch.cuda.empty_cache()
    rp, col, val, c = gen.sparse(n, A, K, 1)
    ref = oracle.vi(oracle.MDP(n, A, gamma, c, row_ptr=rp, col=col, val=val), b, seed=4, eps=eps, max_sweeps=5000)
    assert ref.status == oracle.OK
    if assert_vi_parity(sol, ref, eps):
        mask = q_gap_csr(n, A, rp, col, val, c, gamma, ref.V) > TOL
        assert mask.mean() > 0.99
        assert np.array_equal(sol.pi.cpu().numpy()[mask], ref.pi[mask])


def test_config4_full_mpi_outer_iterations():
    """Config 4: 2048^2 slip gridworld, gamma 0.95, MB-MPI m = 10, b = 65536:
    the first 4 outer iterations (44 operator applications with their
    improvements), from V0 = 0 with pi_0 = greedy(V0)."""
    N, gamma, b, m, outer = 2048, 0.95, 65536, 10, 4
    n = N * N
    rpd, cold, vald, cd = rmb.generate_grid(N)
    prob = rmb.Problem.csr(n, 4, rpd, cold, vald, cd, gamma)
    sol = prob.mpi(b, m, seed=6, eps=1e-6, max_outer=outer)
    prob.close()
    del rpd, cold, vald, cd
    torch.cuda.empty_cache()
    rp, col, val, c = gen.grid(N)
    ref = oracle.mpi(oracle.MDP(n, 4, gamma, c, row_ptr=rp, col=col, val=val), b, m, seed=6, eps=1e-6,
                     max_outer=outer)
    assert ref.status == oracle.NOT_CONVERGED and ref.outer == outer
    assert sol.stats.outer_iters == outer and sol.stats.sweeps == ref.sweeps
    scale = max(1.0, float(np.abs(ref.V).max()))
    assert np.abs(sol.trace - ref.trace).max() <= TOL * scale
    assert np.abs(sol.V.cpu().numpy() - ref.V).max() <= TOL * scale
    # the grid's arithmetic is bit-exact (row mode): so are pi and changed
    assert np.array_equal(sol.pi.cpu().numpy(), ref.pi)
    assert list(sol.changed) == list(ref.changed)
