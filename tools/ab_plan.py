"""A/B of the dense TMA plan (column split C for statically dealt batches,
redundant-combine volume) on config 2: ms/sweep per b, per library build.

  python tools/ab_plan.py build   (CPU)      python tools/ab_plan.py run   (GPU)
"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.ab_build import build_variants, lib_path  # noqa: E402

VARIANTS = {"base": [], "bal4_r4096": ["RMB_AB_BALANCE=4", "RMB_AB_REDMAX=4096"],
            "bal8_r8192": ["RMB_AB_BALANCE=8", "RMB_AB_REDMAX=8192"], "r4096": ["RMB_AB_REDMAX=4096"]}
BS = (32, 64, 100, 128, 250, 500, 1000)


def one():
    import paper_2110_02901_b200 as rmb
    n, A = 10_000, 16
    P, c = rmb.generate_dense(n, A, 1)
    prob = rmb.Problem.dense(P, c, 0.99, flags=rmb.DENSE_NO_CLUSTER)
    prob.vi(1000, eps=1e-6, max_sweeps=3)
    out = {"lib": os.path.basename(os.environ.get("RMB_LIB_PATH", ""))}
    for b in BS:
        best = 1e9
        for rep in range(2):
            sol = prob.vi(b, seed=0, eps=1e-9, max_sweeps=20)
            best = min(best, sol.stats.seconds / sol.stats.sweeps)
        out[b] = round(best * 1e3, 4)
        out[f"us_per_batch_{b}"] = round(best * 1e6 / -(-n // b), 2)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build_variants("dense.cu", VARIANTS)
    elif sys.argv[1] == "one":
        one()
    else:
        for name in VARIANTS:
            subprocess.run([sys.executable, __file__, "one"], env=dict(os.environ, RMB_LIB_PATH=lib_path(name)))
