"""SURVEY 8(f) row 4 measurements on B200: state selection with replacement
(uniform / weighted, R28-R30) and asynchronous MB-VI (R31) against MB-VI with
partitions, on config 2 (dense 10^4 x 16), config 3 (sparse 10^6 x 8 x 32)
and the N=100 maze.  Prints one JSON object per row.

  python tools/f4_perf.py [c2] [c3] [maze]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_02901_b200 as rmb  # noqa: E402


def peak():
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
        return float(json.load(f)["hbm_gbs"])


def row(name, sol, bytes_per_sweep, extra=None):
    st = sol.stats
    gbs = st.sweeps * bytes_per_sweep / st.seconds / 1e9
    d = {"row": name, "status": int(sol.status), "sweeps": st.sweeps, "time_to_eps_ms": round(st.seconds * 1e3, 3),
         "ms_per_sweep": round(st.seconds * 1e3 / max(1, st.sweeps), 4), "GB_per_s": round(gbs, 1),
         "frac": round(gbs / peak(), 4), "final_residual": st.final_residual}
    if extra:
        d.update(extra)
    print(json.dumps(d), flush=True)
    return d


def importance_weights(c, eps=0.1):
    """R29's epsilon-greedy importance law from a priority rho_s = |min_a c(s, a)|
    (the Bellman residual at V0 = 0): w = ceil(2^20 ((1-eps) rho/max rho + eps))."""
    rho = np.abs(c.min(1).astype(np.float64))
    w = np.ceil(2.0**20 * ((1 - eps) * rho / max(rho.max(), 1e-300) + eps)).astype(np.uint32)
    return np.maximum(w, 1)


def c2():
    n, A = 10_000, 16
    P, c = rmb.generate_dense(n, A, 1)
    prob = rmb.Problem.dense(P, c, 0.99)
    bps = n * A * n * 4 + n * A * 4 + 2 * n * 8
    V = torch.zeros(n, dtype=torch.float64, device="cuda")
    pi = torch.zeros(n, dtype=torch.int32, device="cuda")
    prob.vi(1000, eps=1e-6, max_sweeps=3, V=V, pi=pi, v0_zero=True)
    prob.vi(1000, eps=1e-6, max_sweeps=3, V=V, pi=pi, v0_zero=True, asynchronous=True)
    w = importance_weights(c.cpu().numpy())
    prob.set_selection_weights(w)
    for b in (n, 1000):
        row(f"c2 MB-VI partition b={b}", prob.vi(b, seed=3, eps=1e-6, max_sweeps=100_000, V=V, pi=pi, v0_zero=True), bps)
        row(f"c2 MB-VI with replacement b={b}",
            prob.vi(b, seed=3, eps=1e-6, max_sweeps=100_000, V=V, pi=pi, v0_zero=True, select="replace"), bps)
        row(f"c2 MB-VI weighted (eps-greedy importance) b={b}",
            prob.vi(b, seed=3, eps=1e-6, max_sweeps=100_000, V=V, pi=pi, v0_zero=True, select="weighted"), bps)
    for rep in range(2):
        row("c2 async MB-VI", prob.vi(1, seed=3 + rep, eps=1e-6, max_sweeps=100_000, V=V, pi=pi, v0_zero=True,
                                      asynchronous=True), bps)
    row("c2 MB-MPI partition b=n m=10", prob.mpi(n, 10, seed=3, eps=1e-6, V=V, pi=pi, v0_zero=True), bps)
    row("c2 async MB-MPI m=10", prob.mpi(n, 10, seed=3, eps=1e-6, V=V, pi=pi, v0_zero=True, asynchronous=True), bps)


def c3():
    n, A, K = 1_000_000, 8, 32
    rp, col, val, c = rmb.generate_sparse(n, A, K, 1)
    prob = rmb.Problem.csr(n, A, rp, col, val, c, 0.99)
    bps = n * A * K * 8 + n * A * 4 + 16 * n
    prob.vi(n // 8, eps=1e-6, max_sweeps=3)
    for b in (n // 8,):
        row(f"c3 MB-VI partition b={b}", prob.vi(b, seed=0, eps=1e-6, max_sweeps=100_000), bps)
        row(f"c3 MB-VI with replacement b={b}", prob.vi(b, seed=0, eps=1e-6, max_sweeps=100_000, select="replace"), bps)
    row("c3 MB-VI partition b=n", prob.vi(n, seed=0, eps=1e-6, max_sweeps=100_000), bps)
    for rep in range(2):
        row("c3 async MB-VI", prob.vi(1, seed=rep, eps=1e-6, max_sweeps=100_000, asynchronous=True), bps)


def maze():
    from gen import envs
    n, A, rp, col, val, c, _ = envs.maze(100)
    dev = lambda x: torch.from_numpy(x).cuda()  # noqa: E731
    prob = rmb.Problem.csr(n, A, dev(rp), dev(col), dev(val), dev(c), 0.95)
    bps = int(len(val)) * 8 + n * A * 4 + 16 * n
    prob.vi(n, eps=1e-6, max_sweeps=3)
    for b in (1, 512, n):
        row(f"maze100 MB-VI partition b={b}", prob.vi(b, seed=0, eps=1e-6, max_sweeps=100_000), bps)
    row("maze100 MB-VI with replacement b=512", prob.vi(512, seed=0, eps=1e-6, max_sweeps=100_000, select="replace"), bps)
    for rep in range(3):
        row("maze100 async MB-VI", prob.vi(1, seed=rep, eps=1e-6, max_sweeps=100_000, asynchronous=True), bps)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c2", "c3", "maze"]
    for w in which:
        {"c2": c2, "c3": c3, "maze": maze}[w]()
