import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device) and the built librmb.so")
    config.addinivalue_line("markers", "slow: long-running (full-size) check")


@pytest.fixture(scope="session", autouse=True)
def _build_host_libs():
    import gen
    import oracle
    gen.build()
    oracle.build()


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def random_dense_mdp(rng, n, A, gamma=None, nonneg=True, density=1.0, dtype=np.float64):
    """Small random MDP for property tests (numpy RNG; not the bench generator)."""
    import oracle
    P = rng.random((n, A, n))
    if density < 1.0:
        P *= rng.random((n, A, n)) < density
        P[np.arange(n), :, rng.integers(0, n, n)] += 1e-3
    P /= P.sum(-1, keepdims=True)
    c = rng.random((n, A)) if nonneg else rng.standard_normal((n, A))
    g = float(rng.uniform(0.5, 0.99)) if gamma is None else gamma
    return oracle.MDP(n, A, g, c.astype(dtype), P=P.astype(dtype))
