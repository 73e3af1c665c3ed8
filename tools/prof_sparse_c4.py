"""Config-4 kernels for ncu captures (run under ncu -k regex:sparse_solver_kernel -c 1):
  mpi  : one MB-MPI solve (2048^2 grid, b = 65536, m = 10, 1 outer iteration)
  eval : 10 B_{pi,b} sweeps (b = 65536) of a fixed policy (rmb_policy_value)"""
import sys
sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2110_02901_b200 as rmb  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "mpi"
N = 2048
n = N * N
rp, col, val, c = rmb.generate_grid(N)
prob = rmb.Problem.csr(n, 4, rp, col, val, c, 0.95)
if what == "mpi":
    s = prob.mpi(65536, 10, seed=0, eps=1e-6, max_outer=1)
else:
    pi = torch.from_numpy(np.random.default_rng(0).integers(0, 4, n).astype(np.int32)).cuda()
    s = prob.policy_value(pi, b=65536, seed=0, eps=1e-300, max_sweeps=10)
print(f"{what}: sweeps {s.stats.sweeps} ms {s.stats.seconds * 1e3:.3f} phases {prob.last_phase_times()}")
