"""GPU parity of the sparse (CSR / ELL) persistent solver vs the CPU oracle.

Same bar as test_gpu_dense.py: single applications to 1e-11 * max(1,|V|),
solves to 1e-9 * max(1,|V|), identical sweep counts and residual traces,
policies bit-exact where the Q-gap exceeds 1e-9.
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


def assert_close(a, b, rel):
    scale = max(1.0, float(np.abs(b).max()))
    d = np.abs(np.asarray(a) - np.asarray(b)).max()
    assert d <= rel * scale, d


def sparse_instance(n, A, K, seed, dtype=np.float32, gamma=0.99):
    rp, col, val, c = gen.sparse(n, A, K, seed, dtype=dtype)
    m = oracle.MDP(n, A, gamma, c, row_ptr=rp, col=col, val=val)
    prob = rmb.Problem.csr(n, A, tdev(rp), tdev(col), tdev(val), tdev(c), gamma)
    return m, prob


def grid_instance(N, dtype=np.float32, gamma=0.95):
    rp, col, val, c = gen.grid(N, dtype=dtype)
    n = N * N
    m = oracle.MDP(n, 4, gamma, c, row_ptr=rp, col=col, val=val)
    prob = rmb.Problem.csr(n, 4, tdev(rp), tdev(col), tdev(val), tdev(c), gamma)
    return m, prob


def ragged_instance(n, A, seed, gamma=0.9):
    """General CSR with 1..40 successors per row (strided mode, row_ptr path)."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 41, n * A)
    rp = np.zeros(n * A + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32)
    val = rng.random(rp[-1]) + 0.01
    for r in range(n * A):
        val[rp[r]:rp[r + 1]] /= val[rp[r]:rp[r + 1]].sum()
    c = rng.random((n, A))
    m = oracle.MDP(n, A, gamma, c, row_ptr=rp, col=col, val=val)
    prob = rmb.Problem.csr(n, A, tdev(rp), tdev(col), tdev(val), tdev(c), gamma, validate=True)
    return m, prob


def qgap(m, V):
    P = m.to_dense64() if m.n <= 3000 else None
    if P is None:
        return None
    Q = m.c.astype(np.float64) + m.gamma * np.einsum("saj,j->sa", P, V)
    s = np.sort(Q, 1)
    return (s[:, 1] - s[:, 0]) / np.maximum(1.0, np.abs(s[:, 0]))


INSTANCES = {
    "ell32": lambda: sparse_instance(1500, 8, 32, 3),
    "ell32_f64": lambda: sparse_instance(900, 5, 32, 4, dtype=np.float64, gamma=0.9),
    "ell12": lambda: sparse_instance(700, 3, 12, 5, gamma=0.9),
    "grid": lambda: grid_instance(20),
    "ragged": lambda: ragged_instance(400, 6, 6),
}


@pytest.mark.parametrize("name", list(INSTANCES))
@pytest.mark.parametrize("bfrac", [0, 0.013, 0.25, 1.0])
@pytest.mark.parametrize("policy", [False, True])
def test_apply_matches_oracle(name, bfrac, policy):
    m, prob = INSTANCES[name]()
    b = max(1, int(round(bfrac * m.n)))
    rng = np.random.default_rng(b)
    V0 = rng.standard_normal(m.n) * 2
    pi = rng.integers(0, m.A, m.n).astype(np.int32) if policy else None
    Vg, argg, rg = prob.apply(b, 9, 4, tdev(V0), pi=tdev(pi) if policy else None)
    Vo, argo, ro = oracle.sweep(m, V0, b, oracle.partition(m.n, 9, 4), pi)
    assert_close(Vg.cpu().numpy(), Vo, 1e-11)
    assert abs(rg - ro) <= 1e-11 * max(1.0, np.abs(Vo).max())
    gap = qgap(m, Vo)
    mask = gap > 1e-9 if gap is not None else np.ones(m.n, bool)
    assert np.array_equal(argg.cpu().numpy()[mask], argo[mask])


@pytest.mark.parametrize("b", [1, 50, 1500])
def test_config3_shape_vi(b):
    m, prob = sparse_instance(1500, 8, 32, 7)
    sol = prob.vi(b, seed=2, eps=1e-6, max_sweeps=60)
    ref = oracle.vi(m, b, seed=2, eps=1e-6, max_sweeps=60)
    assert sol.stats.sweeps == ref.sweeps
    assert_close(sol.trace, ref.trace, 1e-10)
    assert_close(sol.V.cpu().numpy(), ref.V, 1e-10)


@pytest.mark.parametrize("b,msweeps", [(1, 10), (25, 10), (400, 10), (400, 1)])
def test_config4_shape_mpi(b, msweeps):
    """Gridworld (config 4 law) at 20 x 20, MPI m = 10 (and m = 1)."""
    m, prob = grid_instance(20)
    sol = prob.mpi(b, msweeps, seed=1, eps=1e-8)
    ref = oracle.mpi(m, b, msweeps, seed=1, eps=1e-8)
    assert sol.status == rmb.OK and ref.status == oracle.OK
    assert sol.stats.outer_iters == ref.outer
    assert_close(sol.trace, ref.trace, 1e-9)
    assert np.array_equal(sol.changed, ref.changed)
    assert_close(sol.V.cpu().numpy(), ref.V, 1e-9)
    gap = qgap(m, ref.V)
    assert np.array_equal(sol.pi.cpu().numpy()[gap > 1e-9], ref.pi[gap > 1e-9])


def test_ragged_vi_and_improve():
    m, prob = ragged_instance(300, 4, 11)
    sol = prob.vi(17, seed=3, eps=1e-9)
    ref = oracle.vi(m, 17, seed=3, eps=1e-9)
    assert sol.status == rmb.OK and abs(sol.stats.sweeps - ref.sweeps) <= 1
    k = min(sol.stats.sweeps, ref.sweeps)
    assert_close(sol.trace[:k], ref.trace[:k], 1e-9)
    V = np.random.default_rng(0).standard_normal(300)
    pig = tdev(np.zeros(300, np.int32))
    _, r, ch = prob.improve(tdev(V), pig)
    pio, ro, cho = oracle.improve(m, V, np.zeros(300, np.int32))
    assert np.array_equal(pig.cpu().numpy(), pio) and ch == cho and abs(r - ro) < 1e-11 * max(1, np.abs(V).max())


def test_sparse_device_generator_instance_equals_host():
    rp, col, val, c = rmb.generate_sparse(3000, 8, 32, 1)
    prob = rmb.Problem.csr(3000, 8, rp, col, val, c, 0.99)
    m, _ = sparse_instance(3000, 8, 32, 1)
    sol = prob.vi(300, seed=5, eps=1e-6, max_sweeps=25)
    ref = oracle.vi(m, 300, seed=5, eps=1e-6, max_sweeps=25)
    assert_close(sol.V.cpu().numpy(), ref.V, 1e-10)


@pytest.mark.slow
@pytest.mark.parametrize("b", [1_000_000, 125_000, 4096])
def test_config3_full_size_sampled(b):
    """BASELINE config 3 at full size (10^6 x 8 x 32, fp32, generated on device),
    one application at the launch configuration of the solver; 64 sampled
    states recomputed by the oracle from host-generated rows and the interim V."""
    n, A, K, gamma = 1_000_000, 8, 32, 0.99
    rp, col, val, c = rmb.generate_sparse(n, A, K, 1)
    prob = rmb.Problem.csr(n, A, rp, col, val, c, gamma)
    V0 = np.random.default_rng(0).random(n) * 50
    V1, arg, r = prob.apply(b, 3, 2, tdev(V0))
    V1, arg = V1.cpu().numpy(), arg.cpu().numpy()
    perm = oracle.partition(n, 3, 2)
    pos = np.empty(n, np.int64)
    pos[perm] = np.arange(n)
    bat = pos // b
    for s in np.random.default_rng(b).choice(n, 64, replace=False):
        Vint = np.where(bat < bat[s], V1, V0)
        hrp, hcol, hval, hc = gen.sparse(n, A, K, 1, rows=(s, s + 1))
        q, a = oracle.backup_csr_row(n, hrp, hcol, hval, hc[0], gamma, Vint)
        assert abs(V1[s] - q) <= 1e-11 * max(1.0, abs(q))
        assert arg[s] == a
    assert r == np.abs(V1 - V0).max()


@pytest.mark.slow
def test_config4_full_size_sampled_eval():
    """BASELINE config 4 grid (2048^2 states) one B_{pi,b} application, b = 65536."""
    N, b, gamma = 2048, 65536, 0.95
    n = N * N
    rp, col, val, c = rmb.generate_grid(N)
    prob = rmb.Problem.csr(n, 4, rp, col, val, c, gamma)
    rng = np.random.default_rng(0)
    V0 = rng.random(n) * 20
    pi = rng.integers(0, 4, n).astype(np.int32)
    V1, _, r = prob.apply(b, 5, 7, tdev(V0), pi=tdev(pi))
    V1 = V1.cpu().numpy()
    perm = oracle.partition(n, 5, 7)
    pos = np.empty(n, np.int64)
    pos[perm] = np.arange(n)
    bat = pos // b
    for s in rng.choice(n, 64, replace=False):
        Vint = np.where(bat < bat[s], V1, V0)
        hrp, hcol, hval, hc = gen.grid(N, rows=(s, s + 1))
        q, _ = oracle.backup_csr_row(n, hrp, hcol, hval, hc[0], gamma, Vint, pi_a=int(pi[s]))
        assert abs(V1[s] - q) <= 1e-11 * max(1.0, abs(q))


def test_policy_value_on_grid():
    m, prob = grid_instance(16, dtype=np.float64)
    pi = np.random.default_rng(0).integers(0, 4, m.n).astype(np.int32)
    sol = prob.policy_value(tdev(pi), b=37, seed=2, eps=1e-11)
    assert sol.status == rmb.OK
    J = oracle.policy_value(m, pi)
    assert np.abs(sol.V.cpu().numpy() - J).max() <= 0.95 * sol.stats.final_residual / 0.05 + 1e-9
    V = np.zeros(m.n)
    for k in range(1, 6):
        V, _, ro = oracle.sweep(m, V, 37, oracle.partition(m.n, 2, k), pi)
        assert abs(sol.trace[k - 1] - ro) <= 1e-11 * max(1.0, np.abs(V).max())


def _instance_with_flags(name, flags):
    """Rebuild INSTANCES[name]'s CSR arrays into a handle created with `flags`."""
    m, _ = INSTANCES[name]()
    prob = rmb.Problem.csr(m.n, m.A, tdev(m.row_ptr), tdev(m.col), tdev(m.val), tdev(m.c), m.gamma, flags=flags)
    return m, prob


@pytest.mark.parametrize("name", ["ell32", "grid", "ragged"])
@pytest.mark.parametrize("b", [1, 37, None])
def test_full_grid_is_bitwise_single_cta(name, b):
    """Tiny batches run on one CTA by default; forced onto the full 148-CTA grid
    (RMB_SPARSE_FULL_GRID) every result is bitwise the same (per-state
    arithmetic is grid-free), for VI and MPI, and within the bar of the oracle."""
    m, p1 = _instance_with_flags(name, 0)
    _, p2 = _instance_with_flags(name, rmb.SPARSE_FULL_GRID)
    b = m.n if b is None else b
    for solve in (lambda p: p.vi(b, seed=5, eps=1e-8, max_sweeps=40),
                  lambda p: p.mpi(b, 3, seed=5, eps=1e-8, max_outer=6)):
        one, two = solve(p1), solve(p2)
        assert one.stats.sweeps == two.stats.sweeps
        assert np.array_equal(one.trace, two.trace)
        assert np.array_equal(one.V.cpu().numpy(), two.V.cpu().numpy())
        assert np.array_equal(one.pi.cpu().numpy(), two.pi.cpu().numpy())
    ref = oracle.vi(m, b, seed=5, eps=1e-8, max_sweeps=40)
    assert_close(p2.vi(b, seed=5, eps=1e-8, max_sweeps=40).V.cpu().numpy(), ref.V, 1e-9)


# ------------------------------------------------------------ VI*
@pytest.mark.parametrize("name", list(INSTANCES))
@pytest.mark.parametrize("bfrac", [0, 0.013, 0.25])
def test_chunked_T_apply_is_bellman(name, bfrac):
    """RMB_CHUNKED_T: T in chunks of b states against the sweep-start values.
    Bitwise equal to the one-batch sweep B_n on the device (both read only the
    old values; per-state arithmetic identical) and to the oracle's chunked T."""
    m, prob = INSTANCES[name]()
    b = max(1, int(bfrac * m.n))
    V0 = np.random.default_rng(1).random(m.n) * 10
    Vc, ac, rc = prob.apply(b, 4, 2, tdev(V0), chunked=True)
    Vn, an, rn = prob.apply(m.n, 4, 2, tdev(V0))
    assert np.array_equal(Vc.cpu().numpy(), Vn.cpu().numpy()) and np.array_equal(ac.cpu().numpy(), an.cpu().numpy())
    assert rc == rn
    Vo, ao, ro = oracle.sweep_chunked(m, V0, b, oracle.partition(m.n, 4, 2))
    assert_close(Vc.cpu().numpy(), Vo, 1e-11)


@pytest.mark.parametrize("name", ["ell32", "grid"])
def test_vi_star_solve_equals_bellman_vi(name):
    m, prob = INSTANCES[name]()
    b = max(1, m.n // 7)
    star = prob.vi(b, seed=2, eps=1e-8, max_sweeps=3000, chunked=True)
    bell = prob.vi(m.n, seed=2, eps=1e-8, max_sweeps=3000)
    assert star.stats.sweeps == bell.stats.sweeps and np.array_equal(star.trace, bell.trace)
    assert np.array_equal(star.V.cpu().numpy(), bell.V.cpu().numpy())
    assert star.stats.batches == star.stats.sweeps * -(-m.n // b)  # one barrier per chunk
    ref = oracle.vi(m, b, seed=2, eps=1e-8, max_sweeps=3000, chunked=True)
    assert star.stats.sweeps == ref.sweeps
    assert_close(star.V.cpu().numpy(), ref.V, 1e-9)


def test_apply_rejects_out_of_range_policy():
    m, prob = INSTANCES["grid"]()
    pi = np.zeros(m.n, np.int32)
    pi[m.n // 2] = m.A  # one action past the end
    with pytest.raises(rmb.RmbError) as e:
        prob.apply(10, 1, 1, tdev(np.zeros(m.n)), pi=tdev(pi))
    assert e.value.status == rmb.INVALID_ARG
    pi[m.n // 2] = -1
    with pytest.raises(rmb.RmbError):
        prob.policy_value(tdev(pi))
    # the handle is still usable afterwards (no device fault)
    assert prob.vi(m.n, eps=1e-6).status == rmb.OK
