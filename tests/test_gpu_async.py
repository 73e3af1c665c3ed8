"""GPU checks of ASYNCHRONOUS MB-VI / MB-MPI (RMB_ASYNC; SURVEY 8(f) row 4,
PAPER.md L606; DESIGN reading R31), dense and sparse.

The result depends on the interleaving, so it is compared with what is
unique (tests/test_oracle_async.py pins these properties on a model of every
allowed interleaving): from V0 with T V0 <= V0 every iterate satisfies
J* <= V_k <= T^k V0 (the oracle's Bellman iterates), V_k <= V_{k-1} and
T V_k <= V_k; from V0 = 0 (costs >= 0) the mirror image.  Solves must reach
J* within the certificate ||V - J*|| <= ||TV - V|| / (1 - gamma).
"""
import numpy as np
import pytest
import torch

import gen
import oracle
import paper_2110_02901_b200 as rmb

pytestmark = pytest.mark.gpu


def tdev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def dense(n, A, seed, dtype=np.float32, gamma=0.9, flags=0):
    P, c = gen.dense(n, A, seed, dtype=dtype)
    return oracle.MDP(n, A, gamma, c, P=P), rmb.Problem.dense(tdev(P), tdev(c), gamma, flags=flags)


def sparse(name):
    if name == "grid":
        rp, col, val, c = gen.grid(20)
        n, A, gamma = 400, 4, 0.95
    else:
        n, A, gamma = 1500, 8, 0.99
        rp, col, val, c = gen.sparse(n, A, 32, 3)
    m = oracle.MDP(n, A, gamma, c, row_ptr=rp, col=col, val=val)
    return m, rmb.Problem.csr(n, A, tdev(rp), tdev(col), tdev(val), tdev(c), gamma)


CASES = {
    "dense_f32": lambda: dense(600, 16, 5),
    "dense_f32_ragged": lambda: dense(257, 5, 6),            # n % 4 != 0: scalar loads
    "dense_f64": lambda: dense(300, 12, 7, dtype=np.float64),
    "dense_A40": lambda: dense(200, 40, 8),                  # three row units per state (16 + 16 + 8)
    "dense_A3": lambda: dense(128, 3, 9),                    # units narrower than a row group of 4
    "dense_f32_regs": lambda: dense(400, 16, 10, flags=rmb.DENSE_NO_TMA),  # register-streaming kernel
    "sparse_ell": lambda: sparse("ell"),
    "sparse_grid": lambda: sparse("grid"),
}


def jacobi(m, V):
    return oracle.sweep(m, V, m.n, oracle.partition(m.n, 0, 1))[0]


def tol_of(V):
    return 1e-10 * max(1.0, float(np.abs(V).max()))


@pytest.mark.parametrize("name", list(CASES))
def test_async_iterates_upper_sandwich(name):
    m, prob = CASES[name]()
    Jstar = oracle.vi(m, m.n, eps=1e-12, max_sweeps=100000, identity=True).V
    V0 = np.full(m.n, float(m.c.max()) / (1 - m.gamma))
    V = tdev(V0)
    U, prev = V0.copy(), V0.copy()
    tol = tol_of(V0)
    for k in range(1, 16):
        V, arg, r = prob.apply(m.n, 3, k, V, asynchronous=True)
        Vk = V.cpu().numpy()
        U = jacobi(m, U)
        assert (Vk <= U + tol).all(), k
        assert (Vk >= Jstar - tol).all(), k
        assert (Vk <= prev + tol).all(), k
        assert abs(r - np.abs(Vk - prev).max()) <= tol
        TV = jacobi(m, Vk)
        assert (TV <= Vk + tol).all(), k
        prev = Vk


@pytest.mark.parametrize("name", ["dense_f32", "sparse_grid"])
def test_async_iterates_lower_sandwich(name):
    m, prob = CASES[name]()
    Jstar = oracle.vi(m, m.n, eps=1e-12, max_sweeps=100000, identity=True).V
    V = torch.zeros(m.n, dtype=torch.float64, device="cuda")
    U, prev = np.zeros(m.n), np.zeros(m.n)
    tol = tol_of(Jstar)
    for k in range(1, 16):
        V, _, _ = prob.apply(m.n, 3, k, V, asynchronous=True)
        Vk = V.cpu().numpy()
        U = jacobi(m, U)
        assert (Vk >= U - tol).all() and (Vk <= Jstar + tol).all() and (Vk >= prev - tol).all(), k
        prev = Vk


@pytest.mark.parametrize("name", list(CASES))
def test_async_vi_reaches_optimum(name):
    m, prob = CASES[name]()
    ref = oracle.vi(m, m.n, eps=1e-12, max_sweeps=100000, identity=True)
    sol = prob.vi(1, seed=2, eps=1e-10, max_sweeps=20000, asynchronous=True)
    assert sol.status == rmb.OK
    V = sol.V.cpu().numpy()
    pi = torch.zeros(m.n, dtype=torch.int32, device="cuda")
    _, rT, _ = prob.improve(sol.V, pi)
    assert np.abs(V - ref.V).max() <= rT / (1 - m.gamma) + 1e-9 * max(1.0, np.abs(ref.V).max())
    assert np.abs(V - ref.V).max() <= 1e-7 * max(1.0, np.abs(ref.V).max())
    # async reads at least the sweep-start values: never more sweeps than Bellman VI (b = n)
    bell = oracle.vi(m, m.n, eps=1e-10, max_sweeps=100000, identity=True)
    assert sol.stats.sweeps <= bell.sweeps + 1


@pytest.mark.parametrize("name", ["dense_f32", "dense_f64", "sparse_grid"])
def test_async_mpi_finds_optimal_policy(name):
    m, prob = CASES[name]()
    ref = oracle.mpi(m, m.n, 5, seed=1, eps=1e-10)
    sol = prob.mpi(m.n, 5, seed=1, eps=1e-10, asynchronous=True)
    assert sol.status == rmb.OK and ref.status == oracle.OK
    assert sol.changed[-1] == 0
    V = sol.V.cpu().numpy()
    assert np.abs(V - ref.V).max() <= 1e-7 * max(1.0, np.abs(ref.V).max())
    P = m.to_dense64()
    Q = m.c.astype(np.float64) + m.gamma * np.einsum("saj,j->sa", P, ref.V)
    s = np.sort(Q, 1)
    mask = (s[:, 1] - s[:, 0]) > 1e-6 * np.maximum(1, np.abs(s[:, 0]))
    assert np.array_equal(sol.pi.cpu().numpy()[mask], ref.pi[mask])


def test_async_policy_value_is_J_pi():
    m, prob = CASES["dense_f32"]()
    pi = np.random.default_rng(0).integers(0, m.A, m.n).astype(np.int32)
    sol = prob.policy_value(tdev(pi), eps=1e-12, asynchronous=True)
    assert sol.status == rmb.OK
    assert np.abs(sol.V.cpu().numpy() - oracle.policy_value(m, pi)).max() <= 1e-9


def test_async_rejections():
    m, prob = CASES["dense_f32"]()
    with pytest.raises(rmb.RmbError):
        prob.vi(8, asynchronous=True, chunked=True)
    with pytest.raises(rmb.RmbError):
        prob.vi(8, asynchronous=True, select="replace")
