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


def tdev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def shards(P, c, gamma, G, comm=None):
    n = P.shape[0]
    out = []
    for g in range(G):
        r0, r1 = rmb.shard_range(n, G, g)
        out.append(rmb.Problem.dense(tdev(P[r0:r1]), tdev(c[r0:r1]), gamma, n=n, row_range=(r0, r1),
                                     nccl_comm=comm))
    return out


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("b", [1, 37, 300])
def test_group_vi_is_bitwise_single_gpu(G, b):
    n, A, gamma = 300, 8, 0.95
    P, c = gen.dense(n, A, 3, dtype=np.float32)
    single = rmb.Problem.dense(tdev(P), tdev(c), gamma)
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
    single = rmb.Problem.dense(tdev(P), tdev(c), gamma).mpi(b, m, seed=4, eps=1e-8)
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
    ref = rmb.Problem.dense(tdev(P), tdev(c), gamma).vi(n // 8, seed=0, eps=1e-6, max_sweeps=30)
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
        ref = rmb.Problem.dense(tdev(P), tdev(c), gamma).vi(19, seed=1, eps=1e-9)
        assert sol.status == rmb.OK and np.array_equal(sol.V.cpu().numpy(), ref.V.cpu().numpy())
        assert np.array_equal(sol.trace, ref.trace)
        solm = h.mpi(19, 3, seed=1, eps=1e-9)
        refm = rmb.Problem.dense(tdev(P), tdev(c), gamma).mpi(19, 3, seed=1, eps=1e-9)
        assert np.array_equal(solm.V.cpu().numpy(), refm.V.cpu().numpy())
        assert np.array_equal(solm.pi.cpu().numpy(), refm.pi.cpu().numpy())
        h.close()
    finally:
        rmb.nccl_comm_destroy(comm)
