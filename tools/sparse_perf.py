"""Per-sweep timing of the sparse solver on BASELINE configs 3 and 4."""
import sys
import time
sys.path.insert(0, '.')
import torch
import paper_2110_02901_b200 as rmb

# config 3: 10^6 x 8 x 32, fp32, gamma .99, VI
n, A, K = 1_000_000, 8, 32
rp, col, val, c = rmb.generate_sparse(n, A, K, 1)
prob = rmb.Problem.csr(n, A, rp, col, val, c, 0.99)
bytes3 = n * A * K * 8 + n * A * 4 + 16 * n
prob.vi(n, seed=0, eps=1e-6, max_sweeps=5)
for b in (n, n // 8, n // 64, 4096):
    s = prob.vi(b, seed=0, eps=1e-6, max_sweeps=20)
    t = s.stats.seconds / s.stats.sweeps
    print(f"cfg3 VI b={b}: {t*1e3:.3f} ms/sweep, {bytes3/t/1e9:.0f} GB/s (algorithmic {bytes3/1e9:.2f} GB/sweep), "
          f"{n*A/t:.3e} backups/s, phases={prob.last_phase_times()}", flush=True)
s = prob.vi(n // 8, seed=0, eps=1e-6, max_sweeps=5000)
print(f"cfg3 VI b=n/8 full solve: {s.stats.sweeps} sweeps, status {s.status}, {s.stats.seconds:.3f} s", flush=True)
del prob, rp, col, val, c
torch.cuda.empty_cache()

# config 4: 2048^2 gridworld, MPI m=10, gamma .95
N = 2048
n = N * N
rp, col, val, c = rmb.generate_grid(N)
prob = rmb.Problem.csr(n, 4, rp, col, val, c, 0.95)
vi_bytes = n * 4 * 5 * 8 + n * 4 * 4 + 16 * n
ev_bytes = n * (5 * 8 + 4 + 4) + 16 * n
for b in (n, n // 16, 65536):
    s = prob.mpi(b, 10, seed=0, eps=1e-6, max_outer=3)
    t = s.stats.seconds
    print(f"cfg4 MPI b={b}: 3 outer = {s.stats.sweeps} eval sweeps + {s.stats.outer_iters + 1} improvements in {t*1e3:.1f} ms, "
          f"phases={prob.last_phase_times()}", flush=True)
s = prob.vi(n, seed=0, eps=1e-6, max_sweeps=20)
t = s.stats.seconds / s.stats.sweeps
print(f"cfg4 VI b=n: {t*1e3:.3f} ms/sweep, {vi_bytes/t/1e9:.0f} GB/s", flush=True)
t0 = time.time()
s = prob.mpi(65536, 10, seed=0, eps=1e-6, max_outer=2000)
print(f"cfg4 MPI b=65536 full solve: outer {s.stats.outer_iters}, eval sweeps {s.stats.sweeps}, status {s.status}, "
      f"{s.stats.seconds:.3f} s, changed tail {list(s.changed[-5:])}", flush=True)
