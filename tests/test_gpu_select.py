"""GPU parity of state selection WITH replacement (PAPER.md
L605; DESIGN readings R28-R30) on every solver path, against the CPU oracle
(tests/test_oracle_select.py pins the oracle).

Same bar as the partition paths: single applications to 1e-11 * max(1,|V|),
solves to 1e-9, the same sweep counts and residual traces, policies bit-exact
where the Q-gap exceeds 1e-9; dyadic instances bit-exact.  The draws are
integer-only, so the device draws are bitwise the oracle's.
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


def qgap(m, V):
    Q = m.c.astype(np.float64) + m.gamma * np.einsum("saj,j->sa", m.to_dense64(), V)
    if m.A == 1:
        return np.full(m.n, np.inf)
    s = np.sort(Q, 1)
    return (s[:, 1] - s[:, 0]) / np.maximum(1.0, np.abs(s[:, 0]))


def weights(n, seed):
    return np.random.default_rng(seed).integers(1, 50, size=n).astype(np.uint32)


def dense(n, A, seed, dtype=np.float32, kind="random", gamma=0.9, flags=0):
    P, c = gen.dense(n, A, seed, kind=kind, dtype=dtype)
    m = oracle.MDP(n, A, gamma, c, P=P)
    return m, rmb.Problem.dense(tdev(P), tdev(c), gamma, flags=flags)


def sparse(name, flags=0):
    if name == "grid":
        rp, col, val, c = gen.grid(20)
        n, A, gamma = 400, 4, 0.95
    elif name == "ell32":
        n, A, gamma = 1500, 8, 0.99
        rp, col, val, c = gen.sparse(n, A, 32, 3)
    elif name == "ell12":
        n, A, gamma = 700, 3, 0.9
        rp, col, val, c = gen.sparse(n, A, 12, 5)
    else:  # ragged CSR: strided mode
        rng = np.random.default_rng(6)
        n, A, gamma = 400, 6, 0.9
        lens = rng.integers(1, 41, n * A)
        rp = np.zeros(n * A + 1, np.int64)
        rp[1:] = np.cumsum(lens)
        col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32)
        val = rng.random(rp[-1]) + 0.01
        for r in range(n * A):
            val[rp[r]:rp[r + 1]] /= val[rp[r]:rp[r + 1]].sum()
        c = rng.random((n, A))
    m = oracle.MDP(n, A, gamma, c, row_ptr=rp, col=col, val=val)
    return m, rmb.Problem.csr(n, A, tdev(rp), tdev(col), tdev(val), tdev(c), gamma, flags=flags)


def _sel(prob, m, weighted, seed=0):
    w = weights(m.n, seed + 1) if weighted else None
    if weighted:
        prob.set_selection_weights(tdev(w.view(np.int32)))
    return ("weighted" if weighted else "replace"), w


# ------------------------------------------------------------- the draws
@pytest.mark.parametrize("n", [1, 5, 1000, 65_537])
@pytest.mark.parametrize("weighted", [False, True])
def test_device_draws_match_oracle(n, weighted):
    rp = np.arange(n + 1, dtype=np.int64)          # any handle of n states serves the draw kernel
    prob = rmb.Problem.csr(n, 1, tdev(rp), tdev(np.arange(n, dtype=np.int32)), tdev(np.ones(n, np.float32)),
                           tdev(np.ones((n, 1), np.float32)), 0.5)
    w = weights(n, 7) if weighted else None
    if weighted:
        prob.set_selection_weights(w)              # host weights
    for k in (1, 2, 99):
        d = prob.select_device(5, k, weighted=weighted).cpu().numpy().view(np.uint32)
        assert np.array_equal(d, oracle.select(n, 5, k, w))


# ------------------------------------------------------ dense applications
DENSE_CASES = [  # (n, A, b, dtype)
    (64, 4, 1, np.float32),
    (64, 4, 7, np.float64),
    (257, 5, 19, np.float32),     # ragged
    (600, 16, 64, np.float32),
    (600, 16, 600, np.float32),   # b = n: one batch of n draws (not a permutation)
    (1000, 40, 33, np.float32),   # A > 32
]
DENSE_FLAGS = {"default": 0, "grid": rmb.DENSE_NO_CLUSTER, "warp": rmb.DENSE_NO_TMA,
               "vglobal": rmb.DENSE_VGLOBAL | rmb.DENSE_NO_CLUSTER}


@pytest.mark.parametrize("n,A,b,dtype", DENSE_CASES)
@pytest.mark.parametrize("path", list(DENSE_FLAGS))
@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("policy", [False, True])
def test_dense_apply_matches_oracle(n, A, b, dtype, path, weighted, policy):
    if path == "vglobal" and n % (4 if dtype == np.float32 else 2):
        pytest.skip("the global-V TMA path needs 16-byte rows")
    m, prob = dense(n, A, n + A, dtype=dtype, flags=DENSE_FLAGS[path])
    sel, w = _sel(prob, m, weighted)
    rng = np.random.default_rng(n)
    V0 = rng.standard_normal(n) * 3
    pi = rng.integers(0, A, n).astype(np.int32) if policy else None
    Vg, argg, rg = prob.apply(b, 11, 5, tdev(V0), pi=tdev(pi) if policy else None, select=sel)
    Vo, argo, ro = oracle.sweep(m, V0, b, oracle.select(n, 11, 5, w), pi)
    assert_close(Vg.cpu().numpy(), Vo, 1e-11)
    assert abs(rg - ro) <= 1e-11 * max(1.0, np.abs(Vo).max())
    drawn = np.zeros(n, bool)
    drawn[oracle.select(n, 11, 5, w)] = True
    mask = (qgap(m, Vo) > 1e-9) & drawn        # undrawn states: argmin output is unspecified
    assert np.array_equal(argg.cpu().numpy()[mask], argo[mask])


@pytest.mark.parametrize("b", [1, 3, 8, 13])
@pytest.mark.parametrize("path", ["default", "grid"])
def test_dense_dyadic_with_replacement_is_bitwise(b, path):
    """Duplicates inside a batch and across batches, exact arithmetic: bitwise."""
    n, A = 13, 3
    m, prob = dense(n, A, 4, dtype=np.float64, kind="dyadic", gamma=0.5, flags=DENSE_FLAGS[path])
    V = torch.zeros(n, dtype=torch.float64, device="cuda")
    Vo = np.zeros(n)
    T = -(-n // b)
    for k in range(1, max(1, 45 // (3 * T)) + 1):
        V, arg, r = prob.apply(b, 2, k, V, select="replace")
        Vo, argo, ro = oracle.sweep(m, Vo, b, oracle.select(n, 2, k))
        assert np.array_equal(V.cpu().numpy(), Vo) and r == ro


# ---------------------------------------------------------- dense solves
@pytest.mark.parametrize("n,A,b", [(50, 4, 10), (300, 8, 1), (300, 8, 37), (600, 16, 600)])
@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("path", ["default", "grid"])
def test_dense_vi_with_replacement_matches_oracle(n, A, b, weighted, path):
    m, prob = dense(n, A, 3 * n + A, flags=DENSE_FLAGS[path])
    sel, w = _sel(prob, m, weighted, seed=n)
    sol = prob.vi(b, seed=4, eps=1e-8, max_sweeps=3000, select=sel)
    ref = oracle.vi(m, b, seed=4, eps=1e-8, max_sweeps=3000, replace=True, weights=w)
    assert sol.status == rmb.OK and ref.status == oracle.OK
    assert sol.stats.sweeps == ref.sweeps
    assert_close(sol.trace, ref.trace, 1e-9)
    assert_close(sol.V.cpu().numpy(), ref.V, 1e-9)
    # R30: the stop was confirmed on all states -- pi = greedy(V), ||TV - V|| <= eps
    assert sol.stats.final_residual <= 1e-8
    mask = qgap(m, ref.V) > 1e-9
    assert np.array_equal(sol.pi.cpu().numpy()[mask], ref.pi[mask])


@pytest.mark.parametrize("weighted", [False, True])
def test_dense_mpi_with_replacement_matches_oracle(weighted):
    m, prob = dense(400, 8, 12)
    sel, w = _sel(prob, m, weighted, seed=2)
    sol = prob.mpi(40, 5, seed=3, eps=1e-8, select=sel)
    ref = oracle.mpi(m, 40, 5, seed=3, eps=1e-8, replace=True, weights=w)
    assert sol.status == rmb.OK and ref.status == oracle.OK
    assert sol.stats.outer_iters == ref.outer
    assert_close(sol.trace, ref.trace, 1e-9)
    assert np.array_equal(sol.changed, ref.changed)
    assert_close(sol.V.cpu().numpy(), ref.V, 1e-9)


# ----------------------------------------------------------------- sparse
SPARSE_NAMES = ["ell32", "ell12", "grid", "ragged"]


@pytest.mark.parametrize("name", SPARSE_NAMES)
@pytest.mark.parametrize("bfrac", [0, 0.013, 0.25, 1.0])
@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("full_grid", [False, True])
def test_sparse_apply_matches_oracle(name, bfrac, weighted, full_grid):
    m, prob = sparse(name, rmb.SPARSE_FULL_GRID if full_grid else 0)
    sel, w = _sel(prob, m, weighted)
    b = max(1, int(round(bfrac * m.n)))
    rng = np.random.default_rng(b)
    V0 = rng.standard_normal(m.n) * 2
    Vg, argg, rg = prob.apply(b, 9, 4, tdev(V0), select=sel)
    Vo, argo, ro = oracle.sweep(m, V0, b, oracle.select(m.n, 9, 4, w))
    assert_close(Vg.cpu().numpy(), Vo, 1e-11)
    assert abs(rg - ro) <= 1e-11 * max(1.0, np.abs(Vo).max())


@pytest.mark.parametrize("name", SPARSE_NAMES)
@pytest.mark.parametrize("b", [1, 37, 150, None])
@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("full_grid", [False, True])
def test_sparse_vi_with_replacement_matches_oracle(name, b, weighted, full_grid):
    """Carry mode (b <= lane groups), generic re-copies (b > lane groups, e.g.
    b = 150 on one CTA of 128 groups) and b = n: every one must let a batch's
    new values supersede the carried / re-copied ones of the same state."""
    m, prob = sparse(name, rmb.SPARSE_FULL_GRID if full_grid else 0)
    sel, w = _sel(prob, m, weighted, seed=b or 0)
    b = m.n if b is None else b
    sol = prob.vi(b, seed=6, eps=1e-8, max_sweeps=4000, select=sel)
    ref = oracle.vi(m, b, seed=6, eps=1e-8, max_sweeps=4000, replace=True, weights=w)
    assert sol.status == ref.status
    assert sol.stats.sweeps == ref.sweeps
    assert_close(sol.trace, ref.trace, 1e-9)
    assert_close(sol.V.cpu().numpy(), ref.V, 1e-9)


@pytest.mark.parametrize("b", [5000, 20_000])
def test_sparse_recopy_mode_full_grid(b):
    """b above the grid's lane groups (148 x 32 for 16-lane groups): the generic
    re-copy path, with duplicate states within and across batches."""
    n, A = 20_000, 3
    rp, col, val, c = gen.sparse(n, A, 12, 8)
    m = oracle.MDP(n, A, 0.9, c, row_ptr=rp, col=col, val=val)
    prob = rmb.Problem.csr(n, A, tdev(rp), tdev(col), tdev(val), tdev(c), 0.9)
    sol = prob.vi(b, seed=2, eps=1e-8, max_sweeps=2000, select="replace")
    ref = oracle.vi(m, b, seed=2, eps=1e-8, max_sweeps=2000, replace=True)
    assert sol.status == ref.status == rmb.OK
    assert sol.stats.sweeps == ref.sweeps
    assert_close(sol.trace, ref.trace, 1e-9)
    assert_close(sol.V.cpu().numpy(), ref.V, 1e-9)


@pytest.mark.parametrize("b,msweeps", [(1, 10), (25, 10), (400, 3)])
@pytest.mark.parametrize("weighted", [False, True])
def test_sparse_mpi_with_replacement_matches_oracle(b, msweeps, weighted):
    m, prob = sparse("grid")
    sel, w = _sel(prob, m, weighted, seed=b)
    sol = prob.mpi(b, msweeps, seed=1, eps=1e-8, select=sel)
    ref = oracle.mpi(m, b, msweeps, seed=1, eps=1e-8, replace=True, weights=w)
    assert sol.status == rmb.OK and ref.status == oracle.OK
    assert sol.stats.outer_iters == ref.outer
    assert_close(sol.trace, ref.trace, 1e-9)
    assert np.array_equal(sol.changed, ref.changed)
    assert_close(sol.V.cpu().numpy(), ref.V, 1e-9)


# ------------------------------------------------------------ rejections
def test_selection_rejections():
    m, prob = dense(64, 4, 1)
    V = torch.zeros(64, dtype=torch.float64, device="cuda")
    with pytest.raises(rmb.RmbError):      # no weights set
        prob.vi(8, select="weighted")
    with pytest.raises(rmb.RmbError):
        prob.vi(8, select="replace", chunked=True)
    with pytest.raises(rmb.RmbError):
        prob.vi(8, select="replace", identity=True)
    with pytest.raises(rmb.RmbError):
        prob.set_selection_weights(np.zeros(64, np.uint32))
    with pytest.raises(rmb.RmbError):
        prob.apply(8, 1, 1, V, select="replace", chunked=True)
    pi = torch.zeros(64, dtype=torch.int32, device="cuda")
    flags = rmb.SELECT_REPLACE | rmb.V0_ZERO
    tr = np.zeros(10)
    st = rmb.Stats()
    s = rmb.lib().rmb_policy_value(prob._h, rmb._ptr(pi), 8, 0, 1e-6, 10, flags, rmb._ptr(V), rmb._ptr(tr),
                                   rmb.ctypes.byref(st))
    assert s == rmb.UNSUPPORTED
