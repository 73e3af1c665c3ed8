"""A/B: TMA ring path vs register-streaming warp path on the config-2 instance
(per-b ms/sweep over a fixed number of sweeps, CTA-0 phase breakdown)."""
import sys
sys.path.insert(0, '.')
import paper_2110_02901_b200 as rmb
n, A = 10_000, 16
BS = tuple(int(x) for x in sys.argv[1].split(',')) if len(sys.argv) > 1 else (10000, 2000, 1000, 250, 64, 1)
P, c = rmb.generate_dense(n, A, 1)
probs = {"tma": rmb.Problem.dense(P, c, 0.99, flags=rmb.DENSE_NO_CLUSTER), "warp": rmb.Problem.dense(P, c, 0.99, tma=False),
         "cluster": rmb.Problem.dense(P, c, 0.99)}
for name, prob in probs.items():
    prob.vi(1000, seed=0, eps=1e-6, max_sweeps=3)
for b in BS:
    for name, prob in probs.items():
        ms = 30 if b > 1 else 3
        best = None
        for rep in range(2):
            sol = prob.vi(b, seed=0, eps=1e-6, max_sweeps=ms)
            t = sol.stats.seconds / sol.stats.sweeps
            if best is None or t < best[0]:
                best = (t, prob.last_phase_times(), sol.stats.batches, sol.stats.sweeps)
        t, (comp, bar, comb, nb), batches, sw = best
        print(f"{name:5s} b={b}: {t*1e3:.3f} ms/sweep, {6.4e9/t/1e9:.0f} GB/s | CTA0: compute {comp/1e6:.2f} ms, "
              f"barrier {bar/1e6:.2f} ms, combine {comb/1e6:.2f} ms, {(comp+bar+comb)/max(1,batches)/1e3:.2f} us/batch",
              flush=True)
import numpy as np
for b in (1000, 64):
    s1 = probs["tma"].vi(b, seed=3, eps=1e-6, max_sweeps=50)
    s2 = probs["warp"].vi(b, seed=3, eps=1e-6, max_sweeps=50)
    d = (s1.V - s2.V).abs().max().item()
    print(f"b={b} tma vs warp: max|dV| = {d:.3e}, pi equal frac = {(s1.pi == s2.pi).float().mean().item():.6f}")
