"""GPU parity on the paper's own environments (gen/envs.py):
FrozenLake 8x8, Taxi, 2D-Maze N = 80 — through the C ABI, CSR (sparse solver)
and dense (TMA path) forms, against the CPU oracle on the same instances."""
import numpy as np
import pytest
import torch

import oracle
import paper_2110_02901_b200 as rmb
from gen import envs

pytestmark = pytest.mark.gpu
GAMMA = 0.95


def tdev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


ENVS = {"frozenlake": envs.frozenlake, "taxi": envs.taxi, "maze80": lambda: envs.maze(80)}


def build(name, dense=False):
    n, A, rp, col, val, c, info = ENVS[name]()
    if dense:
        P = envs.dense_from_csr(n, A, rp, col, val)
        m = oracle.MDP(n, A, GAMMA, c, P=P)
        prob = rmb.Problem.dense(tdev(P), tdev(c), GAMMA, validate=True)
    else:
        m = oracle.MDP(n, A, GAMMA, c, row_ptr=rp, col=col, val=val)
        prob = rmb.Problem.csr(n, A, tdev(rp), tdev(col), tdev(val), tdev(c), GAMMA, validate=True)
    return m, prob


def close(a, b, rel):
    scale = max(1.0, float(np.abs(b).max()))
    return np.abs(np.asarray(a) - np.asarray(b)).max() <= rel * scale


@pytest.mark.parametrize("name", list(ENVS))
@pytest.mark.parametrize("frac", [0, 0.1, 1.0])
def test_env_vi_matches_oracle(name, frac):
    m, prob = build(name)
    b = max(1, int(frac * m.n))
    sol = prob.vi(b, seed=3, eps=1e-8, max_sweeps=5000)
    ref = oracle.vi(m, b, seed=3, eps=1e-8, max_sweeps=5000)
    assert sol.stats.sweeps == ref.sweeps
    assert close(sol.trace, ref.trace, 1e-9)
    assert close(sol.V.cpu().numpy(), ref.V, 1e-9)


@pytest.mark.parametrize("name", ["frozenlake", "taxi"])
@pytest.mark.parametrize("b", [1, 50])
def test_env_dense_path_matches_oracle(name, b):
    m, prob = build(name, dense=True)
    sol = prob.vi(b, seed=1, eps=1e-8, max_sweeps=5000)
    ref = oracle.vi(m, b, seed=1, eps=1e-8, max_sweeps=5000)
    assert sol.stats.sweeps == ref.sweeps
    assert close(sol.V.cpu().numpy(), ref.V, 1e-9)


def test_maze_mpi_matches_oracle():
    m, prob = build("maze80")
    sol = prob.mpi(616, 10, seed=2, eps=1e-8, max_outer=500)
    ref = oracle.mpi(m, 616, 10, seed=2, eps=1e-8, max_outer=500)
    assert sol.stats.outer_iters == ref.outer
    assert close(sol.V.cpu().numpy(), ref.V, 1e-9)
