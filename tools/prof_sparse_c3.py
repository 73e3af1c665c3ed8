"""One config-3 MB-VI solve (b = n/8, 10 sweeps) for an ncu --set full capture
of sparse_solver_kernel (run under ncu -k regex:sparse_solver_kernel -c 1)."""
import sys
sys.path.insert(0, '.')
import paper_2110_02901_b200 as rmb  # noqa: E402

n, A, K = 1_000_000, 8, 32
rp, col, val, c = rmb.generate_sparse(n, A, K, 1)
prob = rmb.Problem.csr(n, A, rp, col, val, c, 0.99, flags=0)
s = prob.vi(n // 8, seed=0, eps=1e-300, max_sweeps=10)
print(f"sweeps {s.stats.sweeps} ms {s.stats.seconds * 1e3:.3f} algorithmic bytes/sweep {n * A * K * 8 + n * A * 4 + 16 * n}")
