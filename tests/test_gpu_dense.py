"""GPU parity: the sm_100a dense path (through the C ABI) vs the CPU oracle.

Tolerances: both sides accumulate in fp64 but in
different orders, so V agrees to ~n*u*|V|; we require
  single application: |V_gpu - V_or| <= 1e-11 * max(1, |V|_inf)
  full solves:        |V_gpu - V_or| <= 1e-9  * max(1, |V|_inf)   (north_star)
  residual traces:    same bound per sweep, same number of sweeps
  policies:           bit-exact wherever the oracle's Q-gap exceeds 1e-9 * scale
  dyadic instances:   bit-exact (every product and sum is exact in fp64)
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


def make(n, A, seed, dtype=np.float64, kind="random", gamma=0.9):
    P, c = gen.dense(n, A, seed, kind=kind, dtype=dtype)
    m = oracle.MDP(n, A, gamma, c, P=P)
    prob = rmb.Problem.dense(tdev(P), tdev(c), gamma)
    return m, prob, P, c


def qgap(m, V):
    Q = m.c.astype(np.float64) + m.gamma * np.einsum("saj,j->sa", m.to_dense64(), V)
    if m.A == 1:
        return np.full(m.n, np.inf)
    s = np.sort(Q, 1)
    return (s[:, 1] - s[:, 0]) / np.maximum(1.0, np.abs(s[:, 0]))


def assert_close(a, b, rel):
    scale = max(1.0, float(np.abs(b).max()))
    assert np.abs(np.asarray(a) - np.asarray(b)).max() <= rel * scale, np.abs(np.asarray(a) - np.asarray(b)).max()


# ------------------------------------------------------------ partition
@pytest.mark.parametrize("n,seed,k", [(1, 0, 1), (3, 1, 2), (50, 42, 7), (10_000, 5, 100), (1_000_000, 7, 3)])
def test_device_partition_matches_oracle(n, seed, k):
    d = rmb.partition_device(n, seed, k).cpu().numpy().view(np.uint32)
    assert np.array_equal(d, oracle.partition(n, seed, k))


# ----------------------------------------------------------- generators
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("kind", ["random", "dyadic"])
def test_device_dense_generator_is_bitwise_host(dtype, kind):
    Pd, cd = rmb.generate_dense(77, 5, 3, kind=kind, dtype=dtype)
    Ph, ch = gen.dense(77, 5, 3, kind=kind, dtype=np.float32 if dtype == torch.float32 else np.float64)
    assert np.array_equal(Pd.cpu().numpy(), Ph) and np.array_equal(cd.cpu().numpy(), ch)
    Pr, cr = rmb.generate_dense(77, 5, 3, kind=kind, dtype=dtype, rows=(10, 20))
    assert np.array_equal(Pr.cpu().numpy(), Ph[10:20])


def test_device_sparse_and_grid_generators_are_bitwise_host():
    out = rmb.generate_sparse(500, 8, 32, 9)
    ref = gen.sparse(500, 8, 32, 9)
    for a, b in zip(out, ref):
        assert np.array_equal(a.cpu().numpy(), b)
    out = rmb.generate_grid(13, dtype=torch.float64)
    ref = gen.grid(13, dtype=np.float64)
    for a, b in zip(out, ref):
        assert np.array_equal(a.cpu().numpy(), b)


# ----------------------------------------------------- single application
CASES = [  # n, A, b, dtype, identity
    (1, 1, 1, np.float64, False),
    (2, 3, 1, np.float32, True),
    (50, 4, 10, np.float64, False),
    (50, 4, 7, np.float32, False),       # n % 4 != 0 -> scalar loads
    (257, 5, 1, np.float32, False),      # ragged everything, A % 4 != 0
    (257, 6, 19, np.float64, False),
    (600, 16, 600, np.float32, False),   # Bellman T
    (600, 16, 64, np.float32, False),
    (1000, 40, 33, np.float32, False),   # A > 32
    (2048, 8, 1, np.float32, True),      # Gauss-Seidel F, ascending
    (4096, 3, 4096, np.float64, False),
]


@pytest.mark.parametrize("n,A,b,dtype,identity", CASES)
@pytest.mark.parametrize("policy", [False, True])
def test_apply_matches_oracle(n, A, b, dtype, identity, policy):
    m, prob, P, c = make(n, A, seed=n + A, dtype=dtype)
    rng = np.random.default_rng(n)
    V0 = rng.standard_normal(n) * 3
    pi = rng.integers(0, A, n).astype(np.int32) if policy else None
    sweep = 5
    Vg, argg, rg = prob.apply(b, 11, sweep, tdev(V0), pi=tdev(pi) if policy else None, identity=identity)
    perm = oracle.partition(n, 11, sweep, identity=identity)
    Vo, argo, ro = oracle.sweep(m, V0, b, perm, pi)
    assert_close(Vg.cpu().numpy(), Vo, 1e-11)
    assert abs(rg - ro) <= 1e-11 * max(1.0, np.abs(Vo).max())
    mask = qgap(m, Vo) > 1e-9
    assert np.array_equal(argg.cpu().numpy()[mask], argo[mask])


@pytest.mark.parametrize("b", [1, 3, 8, 13])
def test_dyadic_instance_is_bitwise(b):
    n, A = 13, 3
    m, prob, P, c = make(n, A, seed=4, kind="dyadic", gamma=0.5)
    V = torch.zeros(n, dtype=torch.float64, device="cuda")
    Vo = np.zeros(n)
    # each batch can add 3 fraction bits (gamma/4 = 1/8) to the values it reads:
    # stay within 45 bits so every product and sum is exact in fp64
    T = -(-n // b)
    for k in range(1, max(1, 45 // (3 * T)) + 1):
        V, arg, r = prob.apply(b, 2, k, V)
        Vo, argo, ro = oracle.sweep(m, Vo, b, oracle.partition(n, 2, k))
        assert np.array_equal(V.cpu().numpy(), Vo) and r == ro
        assert np.array_equal(arg.cpu().numpy(), argo)


def test_spec_chain_worked_example():
    # two-state chain, gamma 0.5, J = (4,4)
    P = np.array([[[1.0, 0.0]], [[1.0, 0.0]]])
    c = np.array([[0.0], [1.0]])
    prob = rmb.Problem.dense(tdev(P), tdev(c), 0.5)
    J = tdev(np.array([4.0, 4.0]))
    assert prob.apply(2, 0, 1, J, identity=True)[0].tolist() == [2.0, 3.0]
    assert prob.apply(1, 0, 1, J, identity=True)[0].tolist() == [2.0, 2.0]


# ------------------------------------------------------------- solves
def test_config1_vi_parity():
    # BASELINE config 1: dense 50 x 4, gamma 0.9, b = 10, eps 1e-6, fp64
    m, prob, P, c = make(50, 4, seed=1)
    for seed in range(3):
        sol = prob.vi(10, seed=seed, eps=1e-6)
        ref = oracle.vi(m, 10, seed=seed, eps=1e-6)
        assert sol.status == rmb.OK and sol.stats.sweeps == ref.sweeps
        assert_close(sol.trace, ref.trace, 1e-9)
        assert_close(sol.V.cpu().numpy(), ref.V, 1e-9)
        assert np.array_equal(sol.pi.cpu().numpy(), ref.pi)


@pytest.mark.parametrize("b", [1, 64, 1000, 2000])
def test_config2_shape_vi_parity_scaled(b):
    """Config 2 shape (|A| = 16, gamma 0.99, fp32 P) at n = 2000, 40 sweeps."""
    n, A = 2000, 16
    m, prob, P, c = make(n, A, seed=2, dtype=np.float32, gamma=0.99)
    sol = prob.vi(b, seed=3, eps=1e-6, max_sweeps=40)
    ref = oracle.vi(m, b, seed=3, eps=1e-6, max_sweeps=40)
    assert sol.status == rmb.NOT_CONVERGED and ref.status == oracle.NOT_CONVERGED
    assert_close(sol.trace, ref.trace, 1e-10)
    assert_close(sol.V.cpu().numpy(), ref.V, 1e-10)
    mask = qgap(m, ref.V) > 1e-9
    assert np.array_equal(sol.pi.cpu().numpy()[mask], ref.pi[mask])


def test_vi_to_convergence_small_b_sweep():
    n, A = 300, 8
    m, prob, P, c = make(n, A, seed=5, dtype=np.float32, gamma=0.95)
    for b in (1, 37, 300):
        sol = prob.vi(b, seed=1, eps=1e-8)
        ref = oracle.vi(m, b, seed=1, eps=1e-8)
        assert sol.status == rmb.OK
        assert abs(sol.stats.sweeps - ref.sweeps) <= 1
        k = min(sol.stats.sweeps, ref.sweeps)
        assert_close(sol.trace[:k], ref.trace[:k], 1e-9)
        if sol.stats.sweeps == ref.sweeps:
            assert_close(sol.V.cpu().numpy(), ref.V, 1e-9)


@pytest.mark.parametrize("b,msweeps", [(1, 3), (37, 5), (300, 1), (300, 10)])
def test_mpi_parity(b, msweeps):
    n, A = 300, 8
    m, prob, P, c = make(n, A, seed=6, dtype=np.float32, gamma=0.95)
    sol = prob.mpi(b, msweeps, seed=4, eps=1e-8)
    ref = oracle.mpi(m, b, msweeps, seed=4, eps=1e-8)
    assert sol.status == rmb.OK and ref.status == oracle.OK
    assert sol.stats.outer_iters == ref.outer
    assert_close(sol.trace, ref.trace, 1e-9)
    assert np.array_equal(sol.changed, ref.changed)
    assert_close(sol.V.cpu().numpy(), ref.V, 1e-9)
    assert np.array_equal(sol.pi.cpu().numpy(), ref.pi)


def test_improve_parity():
    n, A = 500, 7
    m, prob, P, c = make(n, A, seed=8, dtype=np.float32)
    V = np.random.default_rng(1).standard_normal(n)
    pi0 = np.zeros(n, np.int32)
    pig = tdev(pi0)
    _, r, ch = prob.improve(tdev(V), pig)
    pio, ro, cho = oracle.improve(m, V, pi0)
    assert np.array_equal(pig.cpu().numpy(), pio) and ch == cho
    assert abs(r - ro) <= 1e-11 * max(1, np.abs(V).max())


# ---------------------------------------------------------- API behaviour
def test_host_buffers_equal_device_buffers():
    n, A = 400, 6
    P, c = gen.dense(n, A, 3, dtype=np.float32)
    ph = rmb.Problem.dense(P, c, 0.97)                       # host numpy
    pd = rmb.Problem.dense(tdev(P), tdev(c), 0.97)
    Vh, pih = np.zeros(n), np.zeros(n, np.int32)
    sh = ph.vi(17, seed=2, eps=1e-7, V=Vh, pi=pih)
    sd = pd.vi(17, seed=2, eps=1e-7)
    assert np.array_equal(Vh, sd.V.cpu().numpy()) and np.array_equal(pih, sd.pi.cpu().numpy())
    assert np.array_equal(sh.trace, sd.trace)


def test_bitwise_reproducible():
    n, A = 1500, 16
    m, prob, P, c = make(n, A, seed=9, dtype=np.float32, gamma=0.99)
    a = prob.vi(50, seed=1, eps=1e-6, max_sweeps=30)
    b = prob.vi(50, seed=1, eps=1e-6, max_sweeps=30)
    assert np.array_equal(a.V.cpu().numpy(), b.V.cpu().numpy()) and np.array_equal(a.trace, b.trace)


def test_errors():
    n, A = 20, 2
    m, prob, P, c = make(n, A, seed=1)
    with pytest.raises(rmb.RmbError) as e:
        prob.vi(0)
    assert e.value.status == rmb.INVALID_ARG
    with pytest.raises(rmb.RmbError):
        prob.vi(n + 1)
    with pytest.raises(rmb.RmbError):
        prob.mpi(5, 0)
    cbad = c.copy()
    cbad[3, :] = np.inf          # every action infinite -> V(3) = inf (min ignores a single inf)
    bad = rmb.Problem.dense(tdev(P), tdev(cbad), 0.9)
    sol = bad.vi(5, eps=1e-6, max_sweeps=10)
    assert sol.status == rmb.NONFINITE
    with pytest.raises(rmb.RmbError) as e:
        rmb.Problem.dense(tdev(P * 1.01), tdev(c), 0.9, validate=True)
    assert e.value.status == rmb.INVALID_MDP


def test_single_state_closed_form():
    prob = rmb.Problem.dense(tdev(np.ones((1, 1, 1))), tdev(np.array([[1.0]])), 0.95)
    sol = prob.vi(1, eps=1e-6)
    K = sol.stats.sweeps
    assert 1.0 * 0.95 ** (K - 1) <= 1e-6 < 0.95 ** (K - 2)
    assert sol.V.item() == pytest.approx((1 - 0.95**K) / 0.05, rel=1e-13)


@pytest.mark.slow
@pytest.mark.parametrize("b", [1, 64, 1000, 10_000])
def test_config2_full_size_sampled(b):
    """BASELINE config 2 at full size (n = 10^4, |A| = 16, fp32 P generated on
    device), one application at the bench's launch configuration; 64 sampled
    states recomputed one by one by the oracle from host-generated rows and the
    interim V (pre/post snapshots assembled with the oracle's partition)."""
    n, A, gamma = 10_000, 16, 0.99
    P, c = rmb.generate_dense(n, A, 1)
    prob = rmb.Problem.dense(P, c, gamma)
    V0 = np.random.default_rng(0).random(n) * 50
    V1, arg, r = prob.apply(b, 7, 3, tdev(V0))
    V1 = V1.cpu().numpy()
    arg = arg.cpu().numpy()
    perm = oracle.partition(n, 7, 3)
    pos = np.empty(n, np.int64)
    pos[perm] = np.arange(n)
    rng = np.random.default_rng(b)
    for s in rng.choice(n, 64, replace=False):
        t = pos[s] // b
        earlier = (pos // b) < t
        Vint = np.where(earlier, V1, V0)
        Ph, ch = gen.dense(n, A, 1, rows=(s, s + 1))
        assert np.array_equal(Ph[0], P[s].cpu().numpy())
        q, a = oracle.backup_dense_row(Ph[0], ch[0], gamma, Vint)
        assert abs(V1[s] - q) <= 1e-11 * max(1.0, abs(q))
        assert arg[s] == a
    assert r == pytest.approx(np.abs(V1 - V0).max(), abs=0)


@pytest.mark.parametrize("b", [1, 50, 400])
def test_policy_value_matches_linear_solve(b):
    """rmb_policy_value: B_{pi,b} iterated to eps reaches J_pi (Eq. 4, Lemma 4),
    the oracle's dense linear solve, within the certificate gamma r/(1-gamma)."""
    n, A, gamma = 400, 6, 0.95
    m, prob, P, c = make(n, A, seed=12, dtype=np.float64, gamma=gamma)
    pi = np.random.default_rng(3).integers(0, A, n).astype(np.int32)
    sol = prob.policy_value(tdev(pi), b=b, seed=1, eps=1e-11)
    assert sol.status == rmb.OK
    J = oracle.policy_value(m, pi)
    r = sol.stats.final_residual
    assert np.abs(sol.V.cpu().numpy() - J).max() <= gamma * r / (1 - gamma) + 1e-9
    # and the sweep-by-sweep trajectory is the oracle's B_{pi,b} iteration
    V = np.zeros(n)
    for k in range(1, 6):
        V, _, ro = oracle.sweep(m, V, b, oracle.partition(n, 1, k), pi)
        assert abs(sol.trace[k - 1] - ro) <= 1e-11 * max(1.0, np.abs(V).max())


# ------------------------------------------- TMA ring path vs warp path
@pytest.mark.parametrize("n,A,b,dtype", [(600, 16, 64, np.float32), (1000, 6, 1, np.float32),
                                         (2048, 16, 2048, np.float32), (512, 5, 37, np.float64),
                                         (4096, 40, 500, np.float32)])
def test_tma_path_matches_warp_path_and_oracle(n, A, b, dtype):
    """The default dense path (cp.async.bulk ring, producer warp running one
    batch ahead) and the register-streaming warp path (RMB_DENSE_NO_TMA) solve
    the same MB-VI: same sweep count, V within rounding, and the oracle."""
    m, prob, P, c = make(n, A, seed=31 + n, dtype=dtype, gamma=0.95)
    warp = rmb.Problem.dense(tdev(P), tdev(c), 0.95, tma=False)
    s1 = prob.vi(b, seed=4, eps=1e-8, max_sweeps=400)
    s2 = warp.vi(b, seed=4, eps=1e-8, max_sweeps=400)
    ref = oracle.vi(m, b, seed=4, eps=1e-8, max_sweeps=400)
    assert s1.stats.sweeps == s2.stats.sweeps == ref.sweeps
    assert_close(s1.V.cpu().numpy(), s2.V.cpu().numpy(), 1e-12)
    assert_close(s1.V.cpu().numpy(), ref.V, 1e-9)
    mask = qgap(m, ref.V) > 1e-9
    assert np.array_equal(s1.pi.cpu().numpy()[mask], ref.pi[mask])


@pytest.mark.parametrize("b,msweeps", [(1, 2), (100, 5), (1024, 3)])
def test_tma_path_mpi_matches_oracle(b, msweeps):
    """MB-MPI on the TMA path: evaluation sweeps right after an improvement are
    fenced (their rows depend on the new pi); outer iterations, V, pi match."""
    n, A = 1024, 8
    m, prob, P, c = make(n, A, seed=77, dtype=np.float32, gamma=0.95)
    sol = prob.mpi(b, msweeps, seed=2, eps=1e-7, max_outer=200)
    ref = oracle.mpi(m, b, msweeps, seed=2, eps=1e-7, max_outer=200)
    assert sol.stats.outer_iters == ref.outer
    assert_close(sol.V.cpu().numpy(), ref.V, 1e-9)
    assert np.array_equal(sol.pi.cpu().numpy(), ref.pi)


# ------------------------------------- global-V TMA mode (large dense n)
@pytest.mark.parametrize("n,A,b,dtype", [(600, 16, 64, np.float32), (1000, 6, 1, np.float32),
                                         (2048, 16, 2048, np.float32), (512, 5, 37, np.float64),
                                         (4096, 40, 500, np.float32)])
def test_global_v_mode_matches_oracle(n, A, b, dtype):
    """RMB_DENSE_VGLOBAL: V and pi read from L2 by the compute warps, each state
    finished and written by one CTA, grid-reduced residual — the mode large n
    (V > shared memory) takes automatically.  Same sweeps, trace, V, pi."""
    m, _, P, c = make(n, A, seed=41 + n, dtype=dtype, gamma=0.95)
    prob = rmb.Problem.dense(tdev(P), tdev(c), 0.95, vglobal=True)
    sol = prob.vi(b, seed=5, eps=1e-8, max_sweeps=400)
    ref = oracle.vi(m, b, seed=5, eps=1e-8, max_sweeps=400)
    assert sol.stats.sweeps == ref.sweeps
    assert_close(sol.trace, ref.trace, 1e-9)
    assert_close(sol.V.cpu().numpy(), ref.V, 1e-9)
    mask = qgap(m, ref.V) > 1e-9
    assert np.array_equal(sol.pi.cpu().numpy()[mask], ref.pi[mask])


@pytest.mark.parametrize("b,msweeps", [(1, 2), (100, 5), (1024, 3)])
def test_global_v_mode_mpi_matches_oracle(b, msweeps):
    n, A = 1024, 8
    m, _, P, c = make(n, A, seed=78, dtype=np.float32, gamma=0.95)
    prob = rmb.Problem.dense(tdev(P), tdev(c), 0.95, vglobal=True)
    sol = prob.mpi(b, msweeps, seed=2, eps=1e-7, max_outer=200)
    ref = oracle.mpi(m, b, msweeps, seed=2, eps=1e-7, max_outer=200)
    assert sol.stats.outer_iters == ref.outer
    assert np.array_equal(sol.changed, ref.changed)
    assert_close(sol.V.cpu().numpy(), ref.V, 1e-9)
    assert np.array_equal(sol.pi.cpu().numpy(), ref.pi)


@pytest.mark.slow
@pytest.mark.parametrize("b", [1, 1000, 30_000])
def test_large_n_dense_sampled(b):
    """n = 30 000 > the shared-memory V limit (|A| = 2, fp32 P 7.2 GB generated
    on device): one application in the automatic global-V mode, 48 sampled
    states recomputed by the oracle from host-generated rows."""
    n, A, gamma = 30_000, 2, 0.99
    P, c = rmb.generate_dense(n, A, 3)
    prob = rmb.Problem.dense(P, c, gamma)
    V0 = np.random.default_rng(1).random(n) * 50
    V1, arg, r = prob.apply(b, 9, 2, tdev(V0))
    V1 = V1.cpu().numpy()
    arg = arg.cpu().numpy()
    perm = oracle.partition(n, 9, 2)
    pos = np.empty(n, np.int64)
    pos[perm] = np.arange(n)
    for s in np.random.default_rng(b).choice(n, 48, replace=False):
        earlier = (pos // b) < pos[s] // b
        Vint = np.where(earlier, V1, V0)
        Ph, ch = gen.dense(n, A, 3, rows=(s, s + 1))
        q, a = oracle.backup_dense_row(Ph[0], ch[0], gamma, Vint)
        assert abs(V1[s] - q) <= 1e-11 * max(1.0, abs(q))
        assert arg[s] == a
    assert r == pytest.approx(np.abs(V1 - V0).max(), abs=0)


# ------------------------------ certificate of the returned policy (NEXT #2)
@pytest.mark.parametrize("b", [1, 60, 600])
def test_returned_policy_optimality_gap_certificate(b):
    """evaluate the pi returned by MB-VI exactly on the GPU
    (rmb_policy_value, B_{pi,b} to 1e-12) and certify it.  With r_K the last
    residual, ||V_K - J*|| <= a r_K / (1 - a) (reading R6, contraction), and a
    policy greedy w.r.t. V_K satisfies ||J_pi - J*|| <= 2 a ||V_K - J*|| / (1 - a)
    (the standard greedy-policy bound behind P:L99).  J* and J_pi also come
    from the oracle's linear solves (Eq. 4) for the comparison."""
    n, A, gamma = 600, 16, 0.95
    m, prob, P, c = make(n, A, seed=90, dtype=np.float32, gamma=gamma)
    sol = prob.vi(b, seed=7, eps=1e-4)
    rK = float(sol.trace[-1])
    pi = sol.pi.clone()
    Jpi = prob.policy_value(pi, b=b, seed=3, eps=1e-12).V.cpu().numpy()
    Jpi_or = oracle.policy_value(m, pi.cpu().numpy())
    assert_close(Jpi, Jpi_or, 1e-9)
    Jstar, _ = oracle.policy_iteration(m)  # exact J* (finite PI, linear solves)
    dV = np.abs(sol.V.cpu().numpy() - Jstar).max()
    assert dV <= gamma * rK / (1 - gamma) * (1 + 1e-9) + 1e-12
    gap = np.abs(Jpi - Jstar).max()
    assert gap <= 2 * gamma * dV / (1 - gamma) + 1e-9


# ------------------------------------------------------------ VI*
@pytest.mark.parametrize("path", ["tma", "warp", "vglobal"])
@pytest.mark.parametrize("b", [1, 7, 64, 150])
def test_chunked_T_apply_is_bellman(path, b):
    """RMB_CHUNKED_T on every dense path: T in chunks of b states against the
    sweep-start values = the one-batch sweep B_n (to rounding: the dense
    column-chunk plan depends on b, so sums may be split differently), and the
    oracle's chunked T to 1e-11."""
    n, A = 300, 6
    P, c = gen.dense(n, A, 21, dtype=np.float32)
    m = oracle.MDP(n, A, 0.95, c, P=P)
    prob = rmb.Problem.dense(tdev(P), tdev(c), 0.95, tma=path != "warp", vglobal=path == "vglobal")
    V0 = np.random.default_rng(b).random(n) * 10
    Vc, ac, rc = prob.apply(b, 3, 5, tdev(V0), chunked=True)
    Vn, an, rn = prob.apply(n, 3, 5, tdev(V0))
    assert_close(Vc.cpu().numpy(), Vn.cpu().numpy(), 1e-12)
    assert abs(rc - rn) <= 1e-12 * 10
    Vo, ao, ro = oracle.sweep_chunked(m, V0, b, oracle.partition(n, 3, 5))
    assert_close(Vc.cpu().numpy(), Vo, 1e-11)
    mask = qgap(m, V0) > 1e-9
    assert np.array_equal(ac.cpu().numpy()[mask], ao[mask])


@pytest.mark.parametrize("b", [1, 40, 333])
def test_vi_star_solve_equals_bellman_vi(b):
    """VI* to eps: the trajectory of Bellman VI (b = n) to rounding, with
    ceil(n/b) barriers per sweep; the oracle's VI* within the solve bar."""
    n, A = 500, 8
    m, prob, P, c = make(n, A, seed=13, dtype=np.float32, gamma=0.97)
    star = prob.vi(b, seed=1, eps=1e-7, max_sweeps=2000, chunked=True)
    bell = prob.vi(n, seed=1, eps=1e-7, max_sweeps=2000)
    assert star.status == rmb.OK and star.stats.sweeps == bell.stats.sweeps
    assert_close(star.trace, bell.trace, 1e-9)
    assert_close(star.V.cpu().numpy(), bell.V.cpu().numpy(), 1e-9)
    assert star.stats.batches == star.stats.sweeps * -(-n // b)
    ref = oracle.vi(m, b, seed=1, eps=1e-7, max_sweeps=2000, chunked=True)
    assert ref.sweeps == star.stats.sweeps
    assert_close(star.V.cpu().numpy(), ref.V, 1e-9)


def test_dense_apply_rejects_out_of_range_policy():
    n, A = 64, 4
    m, prob, P, c = make(n, A, seed=2)
    pi = np.zeros(n, np.int32)
    pi[5] = 4
    with pytest.raises(rmb.RmbError) as e:
        prob.apply(8, 1, 1, tdev(np.zeros(n)), pi=tdev(pi))
    assert e.value.status == rmb.INVALID_ARG
    with pytest.raises(rmb.RmbError):
        prob.apply(8, 1, 1, np.zeros(n), pi=pi)  # host buffers: same check
    assert prob.vi(8, eps=1e-6).status == rmb.OK  # the context is intact


def test_binding_rejects_wrong_vector_types():
    n, A = 32, 3
    m, prob, P, c = make(n, A, seed=3)
    with pytest.raises(TypeError):
        prob.vi(4, V=torch.zeros(n, device="cuda"))          # float32 V
    with pytest.raises(ValueError):
        prob.vi(4, V=torch.zeros(n - 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(TypeError):
        prob.vi(4, pi=np.zeros(n, np.int64))
    with pytest.raises(TypeError):
        prob.apply(4, 0, 1, np.zeros(n, np.float32))


# ---------------------------------------- one-cluster path for tiny batches
@pytest.mark.parametrize("n,A,b,dtype", [(1000, 16, 1, np.float32), (2000, 4, 3, np.float32),
                                         (512, 8, 2, np.float64), (10_000, 16, 1, np.float32)])
def test_cluster_path_matches_grid_path_and_oracle(n, A, b, dtype):
    """Tiny batches (<= 2 MB of P, <= 256 rows) run on one thread-block cluster
    (DSMEM combine, hardware cluster barrier).  Its trajectory equals the
    148-CTA grid solver's (RMB_DENSE_NO_CLUSTER) to fp64 rounding and the
    oracle's within the solve bar; single applications (B_b and B_{pi,b}) to 1e-11."""
    P, c = gen.dense(n, A, 17, dtype=dtype)
    gamma = 0.95
    clu = rmb.Problem.dense(tdev(P), tdev(c), gamma)
    grid = rmb.Problem.dense(tdev(P), tdev(c), gamma, flags=rmb.DENSE_NO_CLUSTER)
    sweeps = 3 if n >= 10_000 else 12
    a = clu.vi(b, seed=4, eps=1e-300, max_sweeps=sweeps)
    g = grid.vi(b, seed=4, eps=1e-300, max_sweeps=sweeps)
    assert a.stats.batches == g.stats.batches == sweeps * -(-n // b)
    # barriers: one cluster barrier per batch plus one at each end (cluster path)
    # vs one grid barrier per batch plus the start (grid path): both paths ran
    assert clu.last_phase_times()[3] == a.stats.batches + 2
    assert grid.last_phase_times()[3] == g.stats.batches + 1
    assert_close(a.V.cpu().numpy(), g.V.cpu().numpy(), 1e-12)
    assert_close(a.trace, g.trace, 1e-12)
    if n <= 2000:
        m = oracle.MDP(n, A, gamma, c, P=P)
        ref = oracle.vi(m, b, seed=4, eps=1e-300, max_sweeps=sweeps)
        assert_close(a.V.cpu().numpy(), ref.V, 1e-10)
        assert_close(a.trace, ref.trace, 1e-10)
        mask = qgap(m, ref.V) > 1e-9
        assert np.array_equal(a.pi.cpu().numpy()[mask], ref.pi[mask])
        V0 = np.random.default_rng(1).random(n) * 10
        pi = np.random.default_rng(2).integers(0, A, n).astype(np.int32)
        for pol in (None, pi):
            V1, arg, r = clu.apply(b, 9, 2, tdev(V0), pi=None if pol is None else tdev(pol))
            Vo, ao, ro = oracle.sweep(m, V0, b, oracle.partition(n, 9, 2), pol)
            assert_close(V1.cpu().numpy(), Vo, 1e-11)
            assert abs(r - ro) <= 1e-11 * 10


def test_cluster_path_policy_value_and_convergence():
    n, A, b = 800, 6, 1
    m, prob, P, c = make(n, A, seed=23, dtype=np.float32, gamma=0.9)
    sol = prob.vi(b, seed=1, eps=1e-8, max_sweeps=2000)
    ref = oracle.vi(m, b, seed=1, eps=1e-8, max_sweeps=2000)
    assert sol.status == rmb.OK and sol.stats.sweeps == ref.sweeps
    assert_close(sol.V.cpu().numpy(), ref.V, 1e-9)
    pi = np.random.default_rng(3).integers(0, A, n).astype(np.int32)
    pv = prob.policy_value(tdev(pi), b=b, seed=2, eps=1e-10)
    J = oracle.policy_value(m, pi)
    assert np.abs(pv.V.cpu().numpy() - J).max() <= 0.9 * pv.stats.final_residual / 0.1 + 1e-9
