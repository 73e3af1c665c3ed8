"""Short dense MB-VI run for ncu captures (config 2 instance, a few sweeps)."""
import sys
sys.path.insert(0, '.')
import paper_2110_02901_b200 as rmb
b = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
P, c = rmb.generate_dense(10_000, 16, 1)
prob = rmb.Problem.dense(P, c, 0.99)
sol = prob.vi(b, seed=0, eps=1e-6, max_sweeps=sweeps)
print(f"b={b} sweeps={sol.stats.sweeps} ms/sweep={sol.stats.seconds*1e3/sol.stats.sweeps:.3f} phases={prob.last_phase_times()}")
