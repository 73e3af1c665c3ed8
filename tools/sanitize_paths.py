"""Small solves on every kernel path, for compute-sanitizer (memcheck /
racecheck / synccheck): dense grid TMA (b = 1, 7, n), global-V, warp path,
one-cluster path, sparse vec / row / strided (1 CTA and full grid), the
asynchronous kernels (TMA and register), draws with replacement, and a fused
2-rank logical group.  Each solve is checked against the oracle loosely (the
point is the sanitizer's report, not parity)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch

import gen
import oracle
import paper_2110_02901_b200 as rmb


def tdev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def check(name, V, ref):
    d = float(np.abs(V.cpu().numpy() - ref).max())
    print(f"{name:40s} max|V - oracle| = {d:.2e}", flush=True)
    assert d < 1e-6 * max(1.0, np.abs(ref).max()), name


def main():
    n, A = 256, 8
    P, c = gen.dense(n, A, 3, dtype=np.float32)
    m = oracle.MDP(n, A, 0.9, c, P=P)
    for flags, tag in ((rmb.DENSE_NO_CLUSTER, "grid"), (0, "cluster"), (rmb.DENSE_NO_TMA, "warp"),
                       (rmb.DENSE_VGLOBAL | rmb.DENSE_NO_CLUSTER, "vglobal")):
        prob = rmb.Problem.dense(tdev(P), tdev(c), 0.9, flags=flags)
        for b in (1, 7, n):
            sol = prob.vi(b, seed=1, eps=1e-9, max_sweeps=400)
            check(f"dense {tag} b={b}", sol.V, oracle.vi(m, b, seed=1, eps=1e-9, max_sweeps=400).V)
        sol = prob.mpi(16, 3, seed=1, eps=1e-9)
        check(f"dense {tag} mpi b=16", sol.V, oracle.mpi(m, 16, 3, seed=1, eps=1e-9).V)
        sol = prob.vi(7, seed=1, eps=1e-9, max_sweeps=400, select="replace")
        check(f"dense {tag} with replacement b=7", sol.V,
              oracle.vi(m, 7, seed=1, eps=1e-9, max_sweeps=400, replace=True).V)
    ref = oracle.vi(m, n, eps=1e-12, max_sweeps=10000, identity=True).V
    for flags, tag in ((0, "tma"), (rmb.DENSE_NO_TMA, "regs")):
        prob = rmb.Problem.dense(tdev(P), tdev(c), 0.9, flags=flags)
        check(f"dense async {tag}", prob.vi(1, eps=1e-11, max_sweeps=2000, asynchronous=True).V, ref)
    # sparse: vec (K = 32), row (grid), strided (K = 12)
    for tag, (rp, col, val, cc), nn, AA, g in (
            ("vec", gen.sparse(600, 8, 32, 2), 600, 8, 0.95), ("row", gen.grid(12), 144, 4, 0.95),
            ("strided", gen.sparse(500, 3, 12, 4), 500, 3, 0.9)):
        ms = oracle.MDP(nn, AA, g, cc, row_ptr=rp, col=col, val=val)
        for flags in (0, rmb.SPARSE_FULL_GRID):
            prob = rmb.Problem.csr(nn, AA, tdev(rp), tdev(col), tdev(val), tdev(cc), g, flags=flags)
            for b in (1, 37, nn):
                sol = prob.vi(b, seed=2, eps=1e-9, max_sweeps=2000)
                check(f"sparse {tag} flags={flags} b={b}", sol.V, oracle.vi(ms, b, seed=2, eps=1e-9, max_sweeps=2000).V)
            sol = prob.vi(37, seed=2, eps=1e-9, max_sweeps=2000, select="replace")
            check(f"sparse {tag} flags={flags} replace b=37", sol.V,
                  oracle.vi(ms, 37, seed=2, eps=1e-9, max_sweeps=2000, replace=True).V)
            sol = prob.mpi(37, 4, seed=2, eps=1e-9)
            check(f"sparse {tag} flags={flags} mpi b=37", sol.V, oracle.mpi(ms, 37, 4, seed=2, eps=1e-9).V)
        ref = oracle.vi(ms, nn, eps=1e-12, max_sweeps=100000, identity=True).V
        check(f"sparse {tag} async", prob.vi(1, eps=1e-11, max_sweeps=5000, asynchronous=True).V, ref)
    # fused logical group (2 ranks in one launch)
    hs = []
    for g in range(2):
        r0, r1 = rmb.shard_range(n, 2, g)
        hs.append(rmb.Problem.dense(tdev(P[r0:r1]), tdev(c[r0:r1]), 0.9, n=n, row_range=(r0, r1)))
    sol = rmb.vi_group(hs, 16, seed=1, eps=1e-9, max_sweeps=400, fused=True)
    check("dense fused group G=2 b=16", sol.V, oracle.vi(m, 16, seed=1, eps=1e-9, max_sweeps=400).V)
    print("all paths ok", flush=True)


if __name__ == "__main__":
    main()
