"""GPU: the sharded (multi-GPU) protocol on one device.

* logical groups of G shard handles (device-copy exchange) give V, pi and the
  residual trace bitwise identical to the single-handle solve (G-invariance),
  and within the north-star tolerance of the oracle;
* the real NCCL path (rmb_vi / rmb_mpi on a handle with nccl_comm, 1 rank)
  runs and matches bitwise as well.
"""
import numpy as np
import pytest
import torch

import gen
import oracle
import paper_2110_02901_b200 as rmb

pytestmark = pytest.mark.gpu
# the sharded paths reproduce the single-GPU GRID solver bit for bit; tiny
# batches on one GPU default to the one-cluster path (another fixed summation
# order, equal to rounding), so the single-GPU references pin the grid solver
GRID = rmb.DENSE_NO_CLUSTER


def tdev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def shards(P, c, gamma, G, comm=None, flags=0):
    n = P.shape[0]
    out = []
    for g in range(G):
        r0, r1 = rmb.shard_range(n, G, g)
        out.append(rmb.Problem.dense(tdev(P[r0:r1]), tdev(c[r0:r1]), gamma, n=n, row_range=(r0, r1),
                                     nccl_comm=comm, flags=flags))
    return out


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("b", [1, 37, 300])
def test_group_vi_is_bitwise_single_gpu(G, b):
    n, A, gamma = 300, 8, 0.95
    P, c = gen.dense(n, A, 3, dtype=np.float32)
    single = rmb.Problem.dense(tdev(P), tdev(c), gamma, flags=GRID)
    ref = single.vi(b, seed=2, eps=1e-8, max_sweeps=40)
    sol = rmb.vi_group(shards(P, c, gamma, G), b, seed=2, eps=1e-8, max_sweeps=40)
    assert sol.stats.sweeps == ref.stats.sweeps
    assert np.array_equal(sol.trace, ref.trace)
    assert np.array_equal(sol.V.cpu().numpy(), ref.V.cpu().numpy())
    assert np.array_equal(sol.pi.cpu().numpy(), ref.pi.cpu().numpy())


@pytest.mark.parametrize("G", [2, 5])
def test_group_mpi_matches_oracle_and_single(G):
    n, A, gamma, b, m = 300, 8, 0.95, 37, 5
    P, c = gen.dense(n, A, 6, dtype=np.float32)
    single = rmb.Problem.dense(tdev(P), tdev(c), gamma, flags=GRID).mpi(b, m, seed=4, eps=1e-8)
    sol = rmb.mpi_group(shards(P, c, gamma, G), b, m, seed=4, eps=1e-8)
    assert sol.status == rmb.OK and sol.stats.outer_iters == single.stats.outer_iters
    assert np.array_equal(sol.V.cpu().numpy(), single.V.cpu().numpy())
    assert np.array_equal(sol.pi.cpu().numpy(), single.pi.cpu().numpy())
    assert np.array_equal(sol.changed, single.changed)
    ref = oracle.mpi(oracle.MDP(n, A, gamma, c, P=P), b, m, seed=4, eps=1e-8)
    assert np.abs(sol.V.cpu().numpy() - ref.V).max() <= 1e-9 * max(1, np.abs(ref.V).max())
    assert np.array_equal(sol.pi.cpu().numpy(), ref.pi)


def test_config2_shape_group_of_8():
    """Config-2 shape (|A| = 16, gamma 0.99, fp32) at n = 2048, b = n/8, 8 shards."""
    n, A, gamma = 2048, 16, 0.99
    P, c = gen.dense(n, A, 1, dtype=np.float32)
    ref = rmb.Problem.dense(tdev(P), tdev(c), gamma, flags=GRID).vi(n // 8, seed=0, eps=1e-6, max_sweeps=30)
    sol = rmb.vi_group(shards(P, c, gamma, 8), n // 8, seed=0, eps=1e-6, max_sweeps=30)
    assert np.array_equal(sol.V.cpu().numpy(), ref.V.cpu().numpy())
    assert np.array_equal(sol.trace, ref.trace)


def test_nccl_single_rank_path():
    """rmb_vi / rmb_mpi on a shard handle with a real (1-rank) NCCL communicator."""
    n, A, gamma = 257, 5, 0.9
    P, c = gen.dense(n, A, 8, dtype=np.float64)
    comm = rmb.nccl_comm_init(1, 0, rmb.nccl_unique_id())
    try:
        (h,) = shards(P, c, gamma, 1, comm=comm)
        sol = h.vi(19, seed=1, eps=1e-9)
        ref = rmb.Problem.dense(tdev(P), tdev(c), gamma, flags=GRID).vi(19, seed=1, eps=1e-9)
        assert sol.status == rmb.OK and np.array_equal(sol.V.cpu().numpy(), ref.V.cpu().numpy())
        assert np.array_equal(sol.trace, ref.trace)
        solm = h.mpi(19, 3, seed=1, eps=1e-9)
        refm = rmb.Problem.dense(tdev(P), tdev(c), gamma, flags=GRID).mpi(19, 3, seed=1, eps=1e-9)
        assert np.array_equal(solm.V.cpu().numpy(), refm.V.cpu().numpy())
        assert np.array_equal(solm.pi.cpu().numpy(), refm.pi.cpu().numpy())
        h.close()
    finally:
        rmb.nccl_comm_destroy(comm)


# ------------------------------------------------------------- sparse shards
def csr_shards(rp, col, val, c, n, A, gamma, G, comm=None, flags=0):
    """Owned-row slices of a CSR instance: row_ptr rebased to 0, col kept global."""
    out = []
    for g in range(G):
        r0, r1 = rmb.shard_range(n, G, g)
        e0, e1 = rp[r0 * A], rp[r1 * A]
        out.append(rmb.Problem.csr(n, A, tdev(rp[r0 * A:r1 * A + 1] - e0), tdev(col[e0:e1]), tdev(val[e0:e1]),
                                   tdev(c[r0:r1]), gamma, row_range=(r0, r1), nccl_comm=comm, flags=flags))
    return out


def ragged_csr(n, A, seed):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 41, n * A)
    rp = np.zeros(n * A + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32)
    val = rng.random(rp[-1]) + 0.01
    for r in range(n * A):
        val[rp[r]:rp[r + 1]] /= val[rp[r]:rp[r + 1]].sum()
    return rp, col, val, rng.random((n, A))


@pytest.mark.parametrize("G", [1, 2, 3, 8])
@pytest.mark.parametrize("kind", ["vec", "row", "strided"])
def test_sparse_group_vi_is_bitwise_single_gpu(G, kind):
    """Sparse shards (ELL vec mode, grid row mode, ragged CSR): V, pi, trace bitwise = one handle."""
    if kind == "vec":
        n, A, gamma, b = 600, 8, 0.99, 75
        rp, col, val, c = gen.sparse(n, A, 32, 5, dtype=np.float32)
    elif kind == "row":
        N, A, gamma = 24, 4, 0.95
        n, b = N * N, 100
        rp, col, val, c = gen.grid(N, dtype=np.float32)
    else:
        n, A, gamma, b = 200, 3, 0.9, 31
        rp, col, val, c = ragged_csr(n, A, 9)
    ref = rmb.Problem.csr(n, A, tdev(rp), tdev(col), tdev(val), tdev(c), gamma).vi(b, seed=3, eps=1e-8,
                                                                                  max_sweeps=60)
    sol = rmb.vi_group(csr_shards(rp, col, val, c, n, A, gamma, G), b, seed=3, eps=1e-8, max_sweeps=60)
    assert sol.stats.sweeps == ref.stats.sweeps
    assert np.array_equal(sol.trace, ref.trace)
    assert np.array_equal(sol.V.cpu().numpy(), ref.V.cpu().numpy())
    assert np.array_equal(sol.pi.cpu().numpy(), ref.pi.cpu().numpy())


@pytest.mark.parametrize("G", [2, 4])
def test_sparse_group_mpi_matches_oracle_and_single(G):
    """Config-4-shaped gridworld MPI (m = 5) over G sparse shards: bitwise = one handle; oracle parity."""
    N, A, gamma, b, m = 20, 4, 0.95, 57, 5
    n = N * N
    rp, col, val, c = gen.grid(N, dtype=np.float32)
    single = rmb.Problem.csr(n, A, tdev(rp), tdev(col), tdev(val), tdev(c), gamma).mpi(b, m, seed=4, eps=1e-8)
    sol = rmb.mpi_group(csr_shards(rp, col, val, c, n, A, gamma, G), b, m, seed=4, eps=1e-8)
    assert sol.status == rmb.OK and sol.stats.outer_iters == single.stats.outer_iters
    assert np.array_equal(sol.V.cpu().numpy(), single.V.cpu().numpy())
    assert np.array_equal(sol.pi.cpu().numpy(), single.pi.cpu().numpy())
    assert np.array_equal(sol.changed, single.changed)
    ref = oracle.mpi(oracle.MDP(n, A, gamma, c, row_ptr=rp, col=col, val=val), b, m, seed=4, eps=1e-8)
    assert np.abs(sol.V.cpu().numpy() - ref.V).max() <= 1e-9 * max(1, np.abs(ref.V).max())
    assert np.array_equal(sol.pi.cpu().numpy(), ref.pi)


def test_sparse_nccl_single_rank_path():
    """rmb_vi on a sparse shard handle with a real (1-rank) NCCL communicator (config-3 shape, small n)."""
    n, A, gamma = 1000, 8, 0.99
    rp, col, val, c = gen.sparse(n, A, 32, 2, dtype=np.float32)
    comm = rmb.nccl_comm_init(1, 0, rmb.nccl_unique_id())
    try:
        (h,) = csr_shards(rp, col, val, c, n, A, gamma, 1, comm=comm)
        sol = h.vi(n // 8, seed=1, eps=1e-7)
        ref = rmb.Problem.csr(n, A, tdev(rp), tdev(col), tdev(val), tdev(c), gamma).vi(n // 8, seed=1, eps=1e-7)
        assert sol.status == rmb.OK and np.array_equal(sol.V.cpu().numpy(), ref.V.cpu().numpy())
        assert np.array_equal(sol.trace, ref.trace)
        h.close()
    finally:
        rmb.nccl_comm_destroy(comm)


@pytest.mark.parametrize("sparse", [False, True])
def test_graph_replayed_sweeps_equal_eager(sparse):
    """The sharded sweep's batch sequence replayed from a CUDA graph (default)
    equals the eager launch sequence (RMB_SHARD_NO_GRAPH) bit for bit, VI and
    MPI -- and the graph really was replayed (rmb_last_graph_launches)."""
    if sparse:
        N, A, gamma = 16, 4, 0.95
        n = N * N
        rp, col, val, c = gen.grid(N, dtype=np.float32)
        make = lambda f: csr_shards(rp, col, val, c, n, A, gamma, 3, flags=f)  # noqa: E731
    else:
        n, A, gamma = 240, 6, 0.95
        P, c = gen.dense(n, A, 12, dtype=np.float32)
        make = lambda f: shards(P, c, gamma, 3, flags=f)  # noqa: E731
    b = 23
    he, hg = make(rmb.SHARD_NO_GRAPH), make(0)
    ev = rmb.vi_group(he, b, seed=6, eps=1e-9, max_sweeps=50)
    assert he[0].last_graph_launches() == 0
    gv = rmb.vi_group(hg, b, seed=6, eps=1e-9, max_sweeps=50)
    assert hg[0].last_graph_launches() == gv.stats.sweeps - 1  # every sweep after the eager warm-up one
    em = rmb.mpi_group(he, b, 4, seed=6, eps=1e-9)
    gm = rmb.mpi_group(hg, b, 4, seed=6, eps=1e-9)
    assert hg[0].last_graph_launches() > 0
    for e, g in ((ev, gv), (em, gm)):
        assert e.stats.sweeps == g.stats.sweeps and e.stats.batches == g.stats.batches
        assert np.array_equal(e.trace, g.trace)
        assert np.array_equal(e.V.cpu().numpy(), g.V.cpu().numpy())
        assert np.array_equal(e.pi.cpu().numpy(), g.pi.cpu().numpy())


@pytest.mark.parametrize("G", [2, 4])
def test_sparse_skewed_shards_keep_single_gpu_layout(G):
    """Shards whose own row lengths differ from the whole problem's (rank 0:
    long ragged rows, the rest: short rows) must still use the layout -- and
    hence the summation order -- of one handle over all rows (layout
    consensus): bitwise equal V, pi, trace."""
    n, A, gamma, b = 240, 3, 0.9, 29
    rng = np.random.default_rng(17)
    r0, r1 = rmb.shard_range(n, G, 0)
    lens = np.where(np.arange(n * A) < r1 * A, rng.integers(30, 41, n * A), rng.integers(1, 4, n * A))
    rp = np.zeros(n * A + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32)
    val = rng.random(rp[-1]) + 0.01
    for r in range(n * A):
        val[rp[r]:rp[r + 1]] /= val[rp[r]:rp[r + 1]].sum()
    c = rng.random((n, A))
    ref = rmb.Problem.csr(n, A, tdev(rp), tdev(col), tdev(val), tdev(c), gamma).vi(b, seed=3, eps=1e-9,
                                                                                  max_sweeps=80)
    sol = rmb.vi_group(csr_shards(rp, col, val, c, n, A, gamma, G), b, seed=3, eps=1e-9, max_sweeps=80)
    assert sol.stats.sweeps == ref.stats.sweeps
    assert np.array_equal(sol.trace, ref.trace)
    assert np.array_equal(sol.V.cpu().numpy(), ref.V.cpu().numpy())
    assert np.array_equal(sol.pi.cpu().numpy(), ref.pi.cpu().numpy())


def test_group_rejects_out_of_range_given_policy():
    n, A, gamma = 120, 4, 0.9
    P, c = gen.dense(n, A, 2, dtype=np.float32)
    pi = np.zeros(n, np.int32)
    pi[-1] = A
    with pytest.raises(rmb.RmbError) as e:
        rmb.mpi_group(shards(P, c, gamma, 2), 10, 2, pi=tdev(pi), pi_given=True)
    assert e.value.status == rmb.INVALID_ARG


# --------------------------------------------- fused exchange (K8f, RMB_FUSED)
@pytest.mark.parametrize("G", [1, 2, 3, 8])
@pytest.mark.parametrize("b", [1, 37, 300])
def test_fused_group_vi_is_bitwise_single_gpu(G, b):
    """The fused multi-rank kernel (G logical ranks in one launch: each rank
    backs up its states of a batch, stores the results into every rank's
    exchange arrays, in-kernel cross-rank barrier) = the single-GPU solve bit
    for bit, and the oracle within the solve bar."""
    n, A, gamma = 300, 8, 0.95
    P, c = gen.dense(n, A, 3, dtype=np.float32)
    ref = rmb.Problem.dense(tdev(P), tdev(c), gamma, flags=GRID).vi(b, seed=2, eps=1e-8, max_sweeps=40)
    sol = rmb.vi_group(shards(P, c, gamma, G), b, seed=2, eps=1e-8, max_sweeps=40, fused=True)
    assert sol.stats.sweeps == ref.stats.sweeps and sol.status == ref.status
    assert np.array_equal(sol.trace, ref.trace)
    assert np.array_equal(sol.V.cpu().numpy(), ref.V.cpu().numpy())
    assert np.array_equal(sol.pi.cpu().numpy(), ref.pi.cpu().numpy())
    orc = oracle.vi(oracle.MDP(n, A, gamma, c, P=P), b, seed=2, eps=1e-8, max_sweeps=40)
    assert np.abs(sol.V.cpu().numpy() - orc.V).max() <= 1e-9 * max(1, np.abs(orc.V).max())


@pytest.mark.parametrize("G", [2, 5, 8])
@pytest.mark.parametrize("vglobal", [False, True])
def test_fused_group_mpi_is_bitwise_single_gpu(G, vglobal):
    """MB-MPI through the fused path (improvement on owned states, cross-rank
    reduction of ||TV - V|| and the changed counts), smem-V and global-V modes."""
    n, A, gamma, b, m = 240, 6, 0.95, 29, 4
    P, c = gen.dense(n, A, 6, dtype=np.float32)
    single = rmb.Problem.dense(tdev(P), tdev(c), gamma, vglobal=vglobal, flags=GRID).mpi(b, m, seed=4, eps=1e-8)
    hs = []
    for g in range(G):
        r0, r1 = rmb.shard_range(n, G, g)
        hs.append(rmb.Problem.dense(tdev(P[r0:r1]), tdev(c[r0:r1]), gamma, n=n, row_range=(r0, r1),
                                    vglobal=vglobal))
    sol = rmb.mpi_group(hs, b, m, seed=4, eps=1e-8, fused=True)
    assert sol.status == rmb.OK and sol.stats.outer_iters == single.stats.outer_iters
    assert np.array_equal(sol.V.cpu().numpy(), single.V.cpu().numpy())
    assert np.array_equal(sol.pi.cpu().numpy(), single.pi.cpu().numpy())
    assert np.array_equal(sol.changed, single.changed)
    assert np.array_equal(sol.trace, single.trace)


def test_fused_repeated_solves_on_the_same_handles():
    """The cross-rank counters are monotonic across launches: consecutive fused
    solves (VI, MPI, VI) on the same handles agree with fresh single-GPU solves."""
    n, A, gamma = 200, 4, 0.9
    P, c = gen.dense(n, A, 9, dtype=np.float32)
    hs = shards(P, c, gamma, 4)
    one = rmb.Problem.dense(tdev(P), tdev(c), gamma, flags=GRID)
    for b, mode in ((17, "vi"), (50, "mpi"), (200, "vi"), (3, "mpi")):
        if mode == "vi":
            a, r = rmb.vi_group(hs, b, seed=b, eps=1e-7, fused=True), one.vi(b, seed=b, eps=1e-7)
        else:
            a, r = rmb.mpi_group(hs, b, 3, seed=b, eps=1e-7, fused=True), one.mpi(b, 3, seed=b, eps=1e-7)
        assert a.stats.sweeps == r.stats.sweeps
        assert np.array_equal(a.V.cpu().numpy(), r.V.cpu().numpy())


def test_fused_nccl_single_rank_path():
    """rmb_vi / rmb_mpi with RMB_FUSED on a shard handle with a real (1-rank)
    NCCL communicator: the per-rank fused kernel, peers mapped through the
    handle's communicator (here only the rank itself)."""
    n, A, gamma = 400, 8, 0.95
    P, c = gen.dense(n, A, 8, dtype=np.float32)
    comm = rmb.nccl_comm_init(1, 0, rmb.nccl_unique_id())
    try:
        (h,) = shards(P, c, gamma, 1, comm=comm)
        one = rmb.Problem.dense(tdev(P), tdev(c), gamma, flags=GRID)
        sol, ref = h.vi(23, seed=1, eps=1e-9, fused=True), one.vi(23, seed=1, eps=1e-9)
        assert sol.status == rmb.OK and np.array_equal(sol.V.cpu().numpy(), ref.V.cpu().numpy())
        assert np.array_equal(sol.trace, ref.trace) and h.last_launch_count() == 1
        solm, refm = h.mpi(23, 3, seed=1, eps=1e-9, fused=True), one.mpi(23, 3, seed=1, eps=1e-9)
        assert np.array_equal(solm.V.cpu().numpy(), refm.V.cpu().numpy())
        assert np.array_equal(solm.pi.cpu().numpy(), refm.pi.cpu().numpy())
        h.close()
    finally:
        rmb.nccl_comm_destroy(comm)


def test_fused_config2_shape_group_of_8():
    """Config-2 shape (|A| = 16, gamma 0.99, fp32) at n = 2048, b = n/8, 8 fused logical ranks."""
    n, A, gamma = 2048, 16, 0.99
    P, c = gen.dense(n, A, 1, dtype=np.float32)
    ref = rmb.Problem.dense(tdev(P), tdev(c), gamma, flags=GRID).vi(n // 8, seed=0, eps=1e-6, max_sweeps=30)
    sol = rmb.vi_group(shards(P, c, gamma, 8), n // 8, seed=0, eps=1e-6, max_sweeps=30, fused=True)
    assert np.array_equal(sol.V.cpu().numpy(), ref.V.cpu().numpy())
    assert np.array_equal(sol.trace, ref.trace)
