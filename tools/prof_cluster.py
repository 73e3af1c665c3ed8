"""Config-2 MB-VI at b = 1 on the one-cluster path: 1 sweep (10^4 batches) for an
ncu --set full capture of dense_cluster_kernel."""
import sys
sys.path.insert(0, '.')
import paper_2110_02901_b200 as rmb  # noqa: E402

P, c = rmb.generate_dense(10_000, 16, 1)
prob = rmb.Problem.dense(P, c, 0.99)
s = prob.vi(1, seed=0, eps=1e-300, max_sweeps=1)
print(f"ms {s.stats.seconds * 1e3:.3f} phases {prob.last_phase_times()}")
