"""Quick per-b timing of MB-VI on the config-2 instance with CTA-0 phase breakdown."""
import sys
sys.path.insert(0, '.')
import paper_2110_02901_b200 as rmb
n, A = 10_000, 16
P, c = rmb.generate_dense(n, A, 1)
prob = rmb.Problem.dense(P, c, 0.99)
prob.vi(1000, seed=0, eps=1e-6, max_sweeps=5)
BS = tuple(int(x) for x in sys.argv[1].split(',')) if len(sys.argv) > 1 else (10000, 1000, 64, 1)
for b in BS:
    ms = 30 if b > 1 else 2
    sol = prob.vi(b, seed=0, eps=1e-6, max_sweeps=ms)
    t = sol.stats.seconds / sol.stats.sweeps
    comp, bar, comb, nb = prob.last_phase_times()
    print(f"b={b}: {sol.stats.sweeps} sweeps, {t*1e3:.3f} ms/sweep, {6.4e9/t/1e9:.0f} GB/s, batches={sol.stats.batches} "
          f"| CTA0: compute {comp/1e6:.2f} ms, barrier {bar/1e6:.2f} ms, combine {comb/1e6:.2f} ms, {nb} barriers, "
          f"{(comp+bar+comb)/max(1,sol.stats.batches)/1e3:.2f} us/batch", flush=True)
if len(sys.argv) <= 2:
    sol = prob.vi(1000, seed=0, eps=1e-6)
    print("full solve b=1000:", sol.stats.sweeps, sol.status, sol.stats.seconds)
