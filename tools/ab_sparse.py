"""A/B of sparse-solver build variants on configs 3 and 4 (timing + CTA-0 phases).
  python tools/ab_sparse.py build      # here: cross-compile the variant .so files
  python tools/ab_sparse.py run        # on the GPU box: time every variant"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SK = ["RMB_AB_SKIP_RECOPY=0", "RMB_AB_SKIP_GATHER=0", "RMB_AB_SKIP_ROWS=0"]
VARIANTS = {
    "product": [],
} if len(sys.argv) > 2 and sys.argv[2] == "product" else {
    "product": [],
    "no_recopy": ["RMB_AB_SKIP_RECOPY=1", "RMB_AB_SKIP_GATHER=0", "RMB_AB_SKIP_ROWS=0"],
    "no_gather": ["RMB_AB_SKIP_RECOPY=0", "RMB_AB_SKIP_GATHER=1", "RMB_AB_SKIP_ROWS=0"],
    "no_rows": ["RMB_AB_SKIP_RECOPY=0", "RMB_AB_SKIP_GATHER=0", "RMB_AB_SKIP_ROWS=1"],
    "no_all3": ["RMB_AB_SKIP_RECOPY=1", "RMB_AB_SKIP_GATHER=1", "RMB_AB_SKIP_ROWS=1"],
}


def so(name):
    return os.path.join(ROOT, "paper_2110_02901_b200", f"build_ab_{name}", f"librmb_{name}.so")


if sys.argv[1] == "build":
    from paper_2110_02901_b200 import _build
    for name, d in VARIANTS.items():
        if name != "product":
            os.makedirs(os.path.dirname(so(name)), exist_ok=True)
            _build.build(force=True, defines=d, out=so(name))
            print("built", so(name))
    sys.exit(0)

if sys.argv[1] == "run":
    for name in VARIANTS:
        env = dict(os.environ)
        if name != "product":
            env["RMB_LIB_PATH"] = so(name)
        r = subprocess.run([sys.executable, __file__, "one", name], env=env, capture_output=True, text=True)
        print(r.stdout + r.stderr[-2000:], flush=True)
    sys.exit(0)

import paper_2110_02901_b200 as rmb  # noqa: E402
name = sys.argv[2]
n, A, K = 1_000_000, 8, 32
rp, col, val, c = rmb.generate_sparse(n, A, K, 1)
if len(sys.argv) > 3:
    p = rmb.Problem.csr(n, A, rp, col, val, c, 0.99)
    p.vi(n // 8, seed=0, eps=1e-300, max_sweeps=3)
    s = p.vi(n // 8, seed=1, eps=1e-300, max_sweeps=20)
    print(f"[{name}] cfg3 VI b=n/8: {s.stats.seconds / s.stats.sweeps * 1e3:.3f} ms/sweep  phases={p.last_phase_times()}")
    del p
del rp, col, val, c
N = 2048
rp, col, val, c = rmb.generate_grid(N)
p = rmb.Problem.csr(N * N, 4, rp, col, val, c, 0.95)
p.mpi(65536, 10, seed=0, eps=1e-6, max_outer=1)
best = min((p.mpi(65536, 10, seed=1, eps=1e-6, max_outer=3) for _ in range(3)), key=lambda s: s.stats.seconds)
print(f"[{name}] cfg4 MPI b=65536 3 outer: {best.stats.seconds * 1e3:.1f} ms  phases={p.last_phase_times()}")
ev = p.policy_value(best.pi, b=65536, seed=1, eps=1e-300, max_sweeps=30)
print(f"[{name}] cfg4 eval sweeps b=65536: {ev.stats.seconds / ev.stats.sweeps * 1e3:.3f} ms/sweep  phases={p.last_phase_times()}")
best = min((p.vi(N * N, seed=1, eps=1e-300, max_sweeps=10) for _ in range(3)), key=lambda s: s.stats.seconds)
print(f"[{name}] cfg4 VI b=n: {best.stats.seconds / best.stats.sweeps * 1e3:.3f} ms/sweep")
