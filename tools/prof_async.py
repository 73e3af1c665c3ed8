"""Short asynchronous dense MB-VI run (config 2 instance) for ncu captures."""
import sys
sys.path.insert(0, '.')
import paper_2110_02901_b200 as rmb
apps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
P, c = rmb.generate_dense(10_000, 16, 1)
prob = rmb.Problem.dense(P, c, 0.99)
sol = prob.vi(1, seed=0, eps=1e-12, max_sweeps=apps, asynchronous=True)
print(f"async applications={sol.stats.sweeps} ms/app={sol.stats.seconds*1e3/sol.stats.sweeps:.3f}")
