"""Stress of the b = 1 look-ahead cluster kernel's stop path: many solves that
stop on convergence at different sweeps (and one with replacement draws),
each checked against the oracle's sweep count."""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import torch
import gen
import oracle
import paper_2110_02901_b200 as rmb

t0 = time.perf_counter()
bad = 0
runs = 0
for n, A in ((64, 4), (300, 16), (1000, 8), (2048, 16)):
    P, c = gen.dense(n, A, n, dtype=np.float32)
    m = oracle.MDP(n, A, 0.9, c, P=P)
    prob = rmb.Problem.dense(torch.from_numpy(P).cuda(), torch.from_numpy(c).cuda(), 0.9)
    for seed in range(12 if n < 2000 else 4):
        for eps in (1e-4, 1e-7):
            sel = "replace" if seed % 4 == 3 else None
            sol = prob.vi(1, seed=seed, eps=eps, max_sweeps=2000, select=sel)
            ref = oracle.vi(m, 1, seed=seed, eps=eps, max_sweeps=2000, replace=sel is not None)
            runs += 1
            if sol.stats.sweeps != ref.sweeps or np.abs(sol.V.cpu().numpy() - ref.V).max() > 1e-9 * max(1, np.abs(ref.V).max()):
                bad += 1
                print("mismatch", n, A, seed, eps, sel, sol.stats.sweeps, ref.sweeps, flush=True)
print(f"{runs} solves, {bad} mismatches, {time.perf_counter() - t0:.1f} s", flush=True)
