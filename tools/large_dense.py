"""Global-V TMA mode at config-5 per-GPU scale: n = 50 000 dense fp32 on one GPU
(|A| = 4: 40 GB = one rank's 6250 x 32 x 50 000 share of BASELINE config 5),
MB-MPI m = 10, b = n/8; plus config 2 forced into global-V mode for comparison."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_2110_02901_b200 as rmb

n, A = 10_000, 16
P, c = rmb.generate_dense(n, A, 1)
for vg in (False, True):
    prob = rmb.Problem.dense(P, c, 0.99, vglobal=vg)
    prob.vi(1000, seed=0, eps=1e-6, max_sweeps=3)
    for b in (10_000, 1000):
        s = prob.vi(b, seed=0, eps=1e-6, max_sweeps=30)
        t = s.stats.seconds / s.stats.sweeps
        print(f"config2 vglobal={vg} b={b}: {t*1e3:.3f} ms/sweep {6.4008e9/t/1e9:.0f} GB/s", flush=True)
    prob.close()
del P, c
torch.cuda.empty_cache()
n, A = 50_000, 4
P, c = rmb.generate_dense(n, A, 5)
prob = rmb.Problem.dense(P, c, 0.99)
bps = n * A * n * 4
s = prob.vi(n // 8, seed=0, eps=1e-6, max_sweeps=5)
t = s.stats.seconds / s.stats.sweeps
print(f"n=50000 A=4 (40 GB) VI b=n/8: {t*1e3:.2f} ms/sweep, {bps/t/1e9:.0f} GB/s", flush=True)
s = prob.mpi(n // 8, 10, seed=0, eps=1e-6, max_outer=3)
print(f"n=50000 A=4 MPI m=10 b=n/8: {s.stats.outer_iters} outer, {s.stats.sweeps} eval sweeps, "
      f"{s.stats.seconds*1e3:.1f} ms, status {s.status}", flush=True)
