"""Where the e2e step's time goes (config 2, host P/c pinned): create (cudaMalloc +
H2D), the solve, destroy -- against a plain torch H2D copy of the same bytes."""
import time
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2110_02901_b200 as rmb

n, A = 10_000, 16
P, c = rmb.generate_dense(n, A, 1)
Ph = torch.empty(P.shape, dtype=P.dtype, pin_memory=True)
ch = torch.empty(c.shape, dtype=c.dtype, pin_memory=True)
Ph.copy_(P)
ch.copy_(c)
del P
torch.cuda.empty_cache()
Vh = np.zeros(n)
pih = np.zeros(n, np.int32)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Pd = Ph.to("cuda", non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    del Pd
    torch.cuda.empty_cache()
    t2 = time.perf_counter()
    p2 = rmb.Problem.dense(Ph, ch, 0.99)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    sol = p2.vi(1000, seed=rep, eps=1e-6, max_sweeps=200_000, V=Vh, pi=pih, v0_zero=True)
    t4 = time.perf_counter()
    p2.close()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"torch H2D {t1-t0:.3f} s ({Ph.numel()*4/(t1-t0)/1e9:.1f} GB/s) | create {t3-t2:.3f} s | vi {t4-t3:.3f} s "
          f"(device {sol.stats.seconds:.3f}) | destroy {t5-t4:.3f} s", flush=True)
