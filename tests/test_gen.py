"""The shared instance generators (gen/) produce valid MDPs of the stated shapes."""
import numpy as np

import gen


def test_dense_rows_are_distributions():
    P, c = gen.dense(37, 5, 3, dtype=np.float64)
    assert P.shape == (37, 5, 37) and c.shape == (37, 5)
    np.testing.assert_allclose(P.sum(-1), 1.0, atol=1e-13)
    assert P.min() > 0 and 0 <= c.min() and c.max() < 1


def test_dense_f32_is_rounded_f64():
    P64, c64 = gen.dense(20, 3, 9, dtype=np.float64)
    P32, c32 = gen.dense(20, 3, 9, dtype=np.float32)
    assert np.array_equal(P64.astype(np.float32), P32)
    assert np.array_equal(c64.astype(np.float32), c32)


def test_dense_row_block_matches_full():
    P, c = gen.dense(30, 2, 4)
    Pb, cb = gen.dense(30, 2, 4, rows=(11, 17))
    assert np.array_equal(P[11:17], Pb) and np.array_equal(c[11:17], cb)


def test_dyadic_is_quarters():
    P, c = gen.dense(13, 3, 2, kind="dyadic", dtype=np.float64)
    assert np.all(P * 4 == np.round(P * 4)) and np.all(P.sum(-1) == 1.0)
    assert set(np.unique(c)) <= {0.0, 1.0, 2.0, 3.0}


def test_sparse_successors_distinct_sorted():
    rp, col, val, c = gen.sparse(1000, 8, 32, 5, dtype=np.float64)
    col = col.reshape(-1, 32)
    assert np.all(np.diff(col, axis=1) > 0) and col.min() >= 0 and col.max() < 1000
    np.testing.assert_allclose(val.reshape(-1, 32).sum(-1), 1.0, atol=1e-13)
    assert np.array_equal(rp, np.arange(8001) * 32)


def test_grid_law():
    N = 6
    rp, col, val, c = gen.grid(N, dtype=np.float64)
    val = val.reshape(N * N, 4, 5)
    col = col.reshape(N * N, 4, 5)
    np.testing.assert_allclose(val.sum(-1), 1.0, atol=1e-14)
    assert np.all(val[0, :, 0] == 1.0) and c[0].tolist() == [0, 0, 0, 0]
    s = 2 * N + 3   # interior: intended 0.7, 4 others (3 nbrs + stay) 0.075
    assert val[s, 0, 1] == 0.7 and val[s, 0, 0] == 0.3 / 4
    assert col[s, 0, 1] == s - N and col[s, 3, 4] == s + 1
    s = N - 1       # top-right corner, moving N is blocked: stay 0.7 + 0.3/3
    assert val[s, 0, 0] == 0.7 + 0.3 / 3 and val[s, 0, 1] == 0.0
