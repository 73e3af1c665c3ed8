import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2110_02901_b200 as rmb
N = int(sys.argv[1]); n = N * N
rp, col, val, c = rmb.generate_grid(N)
prob = rmb.Problem.csr(n, 4, rp, col, val, c, 0.95)
pi = torch.from_numpy(np.random.default_rng(0).integers(0, 4, n).astype(np.int32)).cuda()
b = max(1, n // 64)
prob.policy_value(pi, b=b, seed=0, eps=1e-300, max_sweeps=3)
s = prob.policy_value(pi, b=b, seed=0, eps=1e-300, max_sweeps=10)
print(f"N={N} n={n} b={b}: {s.stats.seconds/10*1e3:.3f} ms/sweep, {s.stats.seconds/10/n*1e12:.1f} ps/state")
