#!/usr/bin/env python
"""bench.py — time-to-eps of MB-VI on BASELINE config 2 (B200, sm_100a).

Workload (BASELINE.json configs[1], the metric's own config, fits one GPU):
random dense MDP |S| = 10 000, |A| = 16, gamma = 0.99, P stored fp32
(6.4 GB, > L2), fp64 accumulation and V, eps = 1e-6, V0 = 0.

One STEP = one complete MB-VI solve to eps at the headline batch size b
(default 1000): every sweep's partition draw, all batches with their
interim-V reads and barriers, residual and stop test, V/pi outputs — all of
SURVEY 8(a) a1-a5, a8 — in one persistent kernel launch.
value = state-action backups per second = sweeps * |S| * |A| / time.

Also reported: the roofline of the solver kernel (algorithmic HBM bytes per
launch / event-timed launch duration vs MEASURED_PEAKS.json), time-to-eps
for every b in {1, 64, 1000, 10000} (Gauss-Seidel -> Bellman), the e2e number
through the C ABI with host buffers, and the CPU oracle baseline.

  python bench.py [--gpus N --steps K --warmup W --b B]
  python bench.py --impl reference   # the CPU oracle arm (host cores)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "state-action backups/sec (HBM GB/s vs peak) and time-to-ε vs batch size, 1/2/4/8 B200"
UNIT = "state-action backups/s"
N_STATES, N_ACTIONS, GAMMA, EPS, INST_SEED = 10_000, 16, 0.99, 1e-6, 1
WORKLOAD = ("BASELINE config 2: random dense MDP |S|=10000 |A|=16 gamma=0.99, MB-VI to eps=1e-6 "
            "(residual stop), V0=0, P fp32 (6.4 GB) + fp64 accumulation/V")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def algo_bytes_per_sweep(n, A, psz, b):
    """P + c + V read/write (+ the 4n-byte permutation when b < n)."""
    return n * A * n * psz + n * A * psz + 2 * n * 8 + (4 * n if b < n else 0)


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, idx):
        self.idx, self.p = idx, None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out = self.p.communicate(timeout=5)[0]
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU oracle
def cpu_model():
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_sample(seconds_target=8.0, n_rows=200):
    """The oracle as it stands, ONE thread, on a bounded sample of the config-2
    workload: full Bellman backups (16 actions x 10^4 successors) of `n_rows`
    states, repeated until ~seconds_target.  Returns (backups/s, sample)."""
    import numpy as np

    import gen
    import oracle
    Ph, ch = gen.dense(N_STATES, N_ACTIONS, INST_SEED, rows=(0, n_rows))
    V = np.random.default_rng(0).random(N_STATES) * 50
    done, t0 = 0, time.perf_counter()
    while True:
        for s in range(n_rows):
            oracle.backup_dense_row(Ph[s], ch[s], GAMMA, V)
        done += n_rows
        el = time.perf_counter() - t0
        if el >= seconds_target:
            break
    return done * N_ACTIONS / el, (f"oracle.backup_dense_row, 1 thread, states 0..{n_rows - 1} of the config-2 "
                                   f"instance: {done} state backups x 16 actions x 10^4 successors in {el:.1f} s")


class OracleSweeps:
    """The oracle's B_b sweep over the WHOLE config-2 instance (host-generated,
    6.4 GB fp32) with W worker threads over each batch's states -- one sweep is
    one unit of the GPU arm's solve."""

    def __init__(self, threads):
        import numpy as np

        import gen
        import oracle
        self.oracle, self.np = oracle, np
        P, c = gen.dense(N_STATES, N_ACTIONS, INST_SEED)
        self.m = oracle.MDP(N_STATES, N_ACTIONS, GAMMA, c, P=P)
        self.V = np.zeros(N_STATES)
        self.threads = threads
        self.k = 1

    def sweep(self, b):
        self.oracle.set_threads(self.threads)
        try:
            self.V, _, r = self.oracle.sweep(self.m, self.V, b, self.oracle.partition(N_STATES, 0, self.k))
        finally:
            self.oracle.set_threads(1)
        self.k += 1
        return r


def arm_config(b, parallelism, extra=None):
    cfg = {"workload": WORKLOAD, "b": b,
           "l2": "inputs larger than L2 (P 6.4 GB) + 256 MB flush between GPU solves",
           "parallelism": parallelism}
    cfg.update(extra or {})
    return cfg


def run_reference(args):
    """--impl reference: the CPU oracle as it stands (oracle/, plain C + OpenMP
    workers over a batch's states) on the same workload and metric.  One step =
    one B_b sweep (b = args.b) of the full config-2 instance on all host cores;
    value = state-action backups / s."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    W = os.cpu_count() or 1
    ora = OracleSweeps(W)
    for _ in range(args.warmup):
        ora.sweep(args.b)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ora.sweep(args.b)
    el = time.perf_counter() - t0
    value = args.steps * N_STATES * N_ACTIONS / el
    sample = (f"each step = one oracle B_b sweep (b={args.b}) over all 10^4 states x 16 actions x 10^4 successors "
              f"of the config-2 instance, {W} OpenMP threads over each batch's states ({cpu_model()})")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": arm_config(args.b, f"cpu{W}"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": W, "kind": "oracle", "sample": sample,
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baselines(b):
    """cpu_baseline of the GPU arm: the oracle at W = 1 (a row sample) and at
    W = nproc (whole B_b sweeps of the config-2 instance)."""
    r1, s1 = oracle_sample()
    W = os.cpu_count() or 1
    ora = OracleSweeps(W)
    ora.sweep(b)
    t0 = time.perf_counter()
    k = 0
    while time.perf_counter() - t0 < 8.0 or k < 2:
        ora.sweep(b)
        k += 1
    el = time.perf_counter() - t0
    rW = k * N_STATES * N_ACTIONS / el
    del ora
    return {"value": rW, "unit": UNIT, "cores": W, "kind": "oracle", "cpu": cpu_model(),
            "sample": f"{k} oracle B_b sweeps (b={b}) of the whole config-2 instance with {W} OpenMP threads "
                      f"over each batch's states, {el:.1f} s",
            "w1": {"value": r1, "cores": 1, "sample": s1}}


def vi_star_rows(rmb, torch, prob_c2, V, pi):
    """SURVEY 8(f) row 3 / PAPER.md L577: VI* (the Bellman operator computed in
    chunks of c states against the old values, RMB_CHUNKED_T) against MB-VI with
    batches of the same size -- the same barriers and bytes per sweep, so the
    time-to-eps ratio is the paper's equal-parallelism comparison."""
    out = []
    for b in (1000, 5000):
        row = {"instance": "config 2 (dense 10^4 x 16, gamma 0.99, eps 1e-6)", "chunk_or_batch": b}
        for name, ch in (("mb_vi", False), ("vi_star", True)):
            sol = prob_c2.vi(b, seed=3, eps=EPS, max_sweeps=200_000, V=V, pi=pi, v0_zero=True, chunked=ch)
            row[name] = {"sweeps": sol.stats.sweeps, "barriers_per_sweep": -(-N_STATES // b),
                         "time_to_eps_ms": sol.stats.seconds * 1e3}
        row["speedup_mb_vi_over_vi_star"] = row["vi_star"]["time_to_eps_ms"] / row["mb_vi"]["time_to_eps_ms"]
        out.append(row)
    from gen import envs
    n, A, rp, col, val, c, _ = envs.maze(100)
    dev = lambda x: torch.from_numpy(x).cuda()  # noqa: E731
    prob = rmb.Problem.csr(n, A, dev(rp), dev(col), dev(val), dev(c), 0.95)
    for b in (-(-n // 2), 512):  # the paper's 2 chunks of 4853 (N=100 maze) and its MB-VI m=512
        row = {"instance": f"2D-Maze N=100 (n={n}, gamma 0.95, eps 1e-6)", "chunk_or_batch": b}
        for name, ch in (("mb_vi", False), ("vi_star", True)):
            sol = prob.vi(b, seed=3, eps=1e-6, max_sweeps=100_000, chunked=ch)
            row[name] = {"sweeps": sol.stats.sweeps, "barriers_per_sweep": -(-n // b),
                         "time_to_eps_ms": sol.stats.seconds * 1e3}
        row["speedup_mb_vi_over_vi_star"] = row["vi_star"]["time_to_eps_ms"] / row["mb_vi"]["time_to_eps_ms"]
        row["paper"] = "x2.57 (m=4853) / x3.04 (m=512) on a GTX 1650 Ti, P:L577"
        out.append(row)
    prob.close()
    return out


def f4_rows(rmb, torch, prob_c2, V, pi):
    """SURVEY 8(f) row 4 (DESIGN R28-R31) on config 2: MB-VI with
    the paper's partitions vs draws with replacement (uniform, and an
    epsilon-greedy importance law, R29) vs asynchronous MB-VI (no batch
    barrier, R31); time-to-eps 1e-6 from V0 = 0."""
    import numpy as np
    peak, _ = peaks()
    bps = algo_bytes_per_sweep(N_STATES, N_ACTIONS, 4, N_STATES)
    c = rmb.generate_dense(N_STATES, N_ACTIONS, INST_SEED)[1].cpu().numpy()
    rho = np.abs(c.min(1).astype(np.float64))
    prob_c2.set_selection_weights(np.maximum(np.ceil(2.0**20 * (0.9 * rho / rho.max() + 0.1)), 1).astype(np.uint32))
    out = []

    def add(name, sol, note=None):
        st = sol.stats
        gbs = st.sweeps * bps / st.seconds / 1e9
        out.append({"variant": name, "status": int(sol.status), "sweeps": st.sweeps,
                    "time_to_eps_ms": st.seconds * 1e3, "ms_per_sweep": st.seconds * 1e3 / max(1, st.sweeps),
                    "GB_per_s": gbs, "frac": gbs / peak, **({"note": note} if note else {})})

    kw = dict(seed=3, eps=EPS, max_sweeps=200_000, V=V, pi=pi, v0_zero=True)
    prob_c2.vi(1, eps=EPS, max_sweeps=3, V=V, pi=pi, v0_zero=True, asynchronous=True)
    add("MB-VI, partition (paper), b=1000", prob_c2.vi(1000, **kw))
    add("MB-VI, with replacement, b=1000", prob_c2.vi(1000, select="replace", **kw),
        "r_k covers the drawn states only: stop confirmed by ||TV-V|| (R30)")
    add("MB-VI, eps-greedy importance (w ~ 0.9 |min_a c| / max + 0.1), b=1000", prob_c2.vi(1000, select="weighted", **kw))
    add("MB-VI, partition, b=n (Bellman)", prob_c2.vi(N_STATES, **kw))
    add("asynchronous MB-VI (no batch barrier; one state per CTA, rows by TMA, finisher warp)",
        prob_c2.vi(1, asynchronous=True, **kw),
        "dense_async_tma_kernel: not deterministic; pinned by the J* <= V_k <= T^k V0 sandwich")
    prob_c2.set_selection_weights(None)
    return out


def config5_line(rmb, torch, dist, comm, world, rank, dev):
    """BASELINE config 5 (dense |S|=50 000, |A|=32, fp32, MB-MPI m=10, b=n/8,
    gamma 0.99): P is 320 GB, sharded 8 ways = 40 GB per GPU.  On N GPUs the
    instance has n_N = 50 000 sqrt(N/8) states (the same 40 GB per GPU; n_8 is
    config 5 itself), each rank generating its rows on the device.  N = 1 adds
    the certificate ||TV - V||_inf with every row regenerated on the host."""
    A, gamma = 32, 0.99
    n = int(round(50_000 * (world / 8) ** 0.5 / 8)) * 8
    b = n // 8
    rows = rmb.shard_range(n, world, rank) if world > 1 else (0, n)
    P, c = rmb.generate_dense(n, A, 5, rows=rows)
    if world > 1:
        prob = rmb.Problem.dense(P, c, gamma, n=n, row_range=rows, nccl_comm=comm)
    else:
        prob = rmb.Problem.dense(P, c, gamma)
    fused = world > 1
    if fused:
        try:
            prob.mpi(b, 10, seed=0, eps=1e-6, max_outer=1, fused=True)
        except rmb.RmbError as e:
            print(f"bench.py: config 5 fused path unavailable ({e})", file=sys.stderr)
            fused = False
    prob.mpi(b, 10, seed=0, eps=1e-6, max_outer=1, fused=fused)
    sol = prob.mpi(b, 10, seed=1, eps=1e-6, max_outer=1000, fused=fused)
    t = sol.stats.seconds
    if dist:
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt[0])
    st = sol.stats
    share = (rows[1] - rows[0]) * A * n * 4
    # bytes per rank: eval sweeps read one row per owned state, improvements all owned rows
    rank_bytes = st.sweeps * share / A + (st.outer_iters + 1) * share
    line = {"workload": f"config 5 on {world} GPU(s): dense |S|={n} |A|={A} fp32 ({share / 1e9:.1f} GB of P per GPU), "
                        f"gamma={gamma}, MB-MPI m=10 b=n/8={b} to eps=1e-6",
            "status": int(sol.status), "outer_iterations": st.outer_iters, "eval_sweeps": st.sweeps,
            "exchange": "fused in-kernel NVLink" if fused else ("none" if world == 1 else "NCCL all-gather per batch"),
            "time_to_eps_ms": t * 1e3, "backups_per_s": (st.sweeps * n + (st.outer_iters + 1) * n * A) / t,
            "per_gpu_GB_per_s": rank_bytes / t / 1e9}
    if world == 1:
        import oracle
        Vh = sol.V.cpu().numpy()
        oracle.set_threads(os.cpu_count() or 1)
        t0 = time.perf_counter()
        try:
            rT, arg = oracle.bellman_residual_dense_gen(5, n, A, gamma, Vh)
        finally:
            oracle.set_threads(1)
        line["certificate"] = {"bellman_residual_host": rT, "bound_V_minus_Vstar": rT / (1 - gamma),
                               "gpu_final_residual": st.final_residual, "host_seconds": time.perf_counter() - t0,
                               "policy_agrees_frac": float((arg == sol.pi.cpu().numpy()).mean()),
                               "how": "oracle.bellman_residual_dense_gen: every row regenerated on the host "
                                      "from gen/rmb_gen.h (fp32 storage), fp64 sequential sums, all cores"}
    del prob, P, c
    torch.cuda.empty_cache()
    return line


def other_configs(rmb, torch, dev):
    """Secondary lines: BASELINE config 3 (sparse 10^6 x 8 x 32, MB-VI b = n/8)
    and config 4 (2048^2 gridworld, MB-MPI m = 10, b = 65536), one solve each."""
    out = []
    n, A, K = 1_000_000, 8, 32
    rp, col, val, c = rmb.generate_sparse(n, A, K, 1)
    prob = rmb.Problem.csr(n, A, rp, col, val, c, 0.99)
    prob.vi(n // 8, seed=0, eps=1e-6, max_sweeps=3)
    sol = prob.vi(n // 8, seed=0, eps=1e-6, max_sweeps=100_000)
    st = sol.stats
    bps = n * A * K * 8 + n * A * 4 + 16 * n
    peak, _ = peaks()
    out.append({"workload": "config 3: sparse random |S|=1e6 |A|=8 K=32 (ELL fp32), gamma=0.99, MB-VI b=n/8 to eps=1e-6",
                "status": int(sol.status), "sweeps": st.sweeps, "time_to_eps_ms": st.seconds * 1e3,
                "backups_per_s": st.sweeps * n * A / st.seconds,
                "hbm_algorithmic_GB_per_s": st.sweeps * bps / st.seconds / 1e9,
                "frac": st.sweeps * bps / st.seconds / 1e9 / peak,
                "note": "bound by L1TEX wavefronts of the random 8-byte V gathers (one sector each, 2.56e8 per "
                        "sweep), not HBM: profiles/r02"})
    sol = prob.vi(1, seed=0, eps=1e-6, max_sweeps=100_000, asynchronous=True)
    st = sol.stats
    out.append({"workload": "config 3, asynchronous MB-VI (SURVEY 8(f) row 4, R31: no batch barrier, one V buffer)",
                "status": int(sol.status), "sweeps": st.sweeps, "time_to_eps_ms": st.seconds * 1e3,
                "backups_per_s": st.sweeps * n * A / st.seconds,
                "hbm_algorithmic_GB_per_s": st.sweeps * bps / st.seconds / 1e9,
                "frac": st.sweeps * bps / st.seconds / 1e9 / peak})
    del prob, rp, col, val, c
    torch.cuda.empty_cache()
    N = 2048
    n = N * N
    rp, col, val, c = rmb.generate_grid(N)
    prob = rmb.Problem.csr(n, 4, rp, col, val, c, 0.95)
    prob.mpi(65536, 10, seed=0, eps=1e-6, max_outer=2)
    sol = prob.mpi(65536, 10, seed=0, eps=1e-6, max_outer=100_000)
    st = sol.stats
    backups = st.sweeps * n + (st.outer_iters + 1) * n * 4
    # algorithmic bytes: eval n(40 + 4 + 4) + 2 V; improvement the whole ELL + c + V
    algo = st.sweeps * (n * 48 + 16 * n) + (st.outer_iters + 1) * (n * 4 * 40 + n * 4 * 4 + 8 * n)
    out.append({"workload": "config 4: 2048x2048 slip gridworld, gamma=0.95, MB-MPI m=10 b=65536 to eps=1e-6",
                "status": int(sol.status), "outer_iterations": st.outer_iters, "eval_sweeps": st.sweeps,
                "time_to_eps_ms": st.seconds * 1e3, "backups_per_s": backups / st.seconds,
                "hbm_algorithmic_GB_per_s": algo / st.seconds / 1e9, "frac": algo / st.seconds / 1e9 / peak,
                "note": "64 batches per evaluation sweep: per-batch latency (grid barrier ~2.5 us + one V-gather "
                        "round trip) and L2 capacity (two 33.5 MB copies of V) bound it: profiles/r02"})
    sol = prob.mpi(65536, 10, seed=0, eps=1e-6, max_outer=100_000, asynchronous=True)
    st = sol.stats
    backups = st.sweeps * n + (st.outer_iters + 1) * n * 4
    algo = st.sweeps * (n * 48 + 16 * n) + (st.outer_iters + 1) * (n * 4 * 40 + n * 4 * 4 + 8 * n)
    out.append({"workload": "config 4, asynchronous MB-MPI m=10 (SURVEY 8(f) row 4, R31: evaluation sweeps with no "
                            "batch barrier, one V buffer)",
                "status": int(sol.status), "outer_iterations": st.outer_iters, "eval_sweeps": st.sweeps,
                "time_to_eps_ms": st.seconds * 1e3, "backups_per_s": backups / st.seconds,
                "hbm_algorithmic_GB_per_s": algo / st.seconds / 1e9, "frac": algo / st.seconds / 1e9 / peak})
    del prob, rp, col, val, c
    torch.cuda.empty_cache()
    return out


def paper_envs(rmb, torch):
    """Secondary lines: the paper's own environments (gen/envs.py),
    MB-VI to a 1e-6 residual at b = 1 (GS-VI), |S|/10 and |S| (VI): sweeps,
    time-to-eps and time per batch — the latency-bound regime of SURVEY 6."""
    from gen import envs
    out = []
    for name, f in (("FrozenLake 8x8", envs.frozenlake), ("Taxi", envs.taxi),
                    ("2D-Maze N=80", lambda: envs.maze(80)), ("2D-Maze N=100", lambda: envs.maze(100))):
        n, A, rp, col, val, c, _ = f()
        dev = lambda x: torch.from_numpy(x).cuda()
        prob = rmb.Problem.csr(n, A, dev(rp), dev(col), dev(val), dev(c), 0.95)
        prob.vi(n, seed=0, eps=1e-6, max_sweeps=3)
        rows = []
        for b in (1, max(1, n // 10), n):
            sol = prob.vi(b, seed=0, eps=1e-6, max_sweeps=100_000)
            st = sol.stats
            rows.append({"b": b, "sweeps": st.sweeps, "time_to_eps_ms": st.seconds * 1e3,
                         "us_per_batch": st.seconds / max(1, st.batches) * 1e6})
        sol = prob.vi(1, seed=0, eps=1e-6, max_sweeps=100_000, asynchronous=True)  # R31: no batch barrier
        rows.append({"b": "async", "sweeps": sol.stats.sweeps, "time_to_eps_ms": sol.stats.seconds * 1e3,
                     "us_per_batch": sol.stats.seconds / max(1, sol.stats.batches) * 1e6})
        out.append({"env": name, "n": n, "A": A, "nnz": int(len(val)), "gamma": 0.95, "vi": rows})
        prob.close()
    return out


# ------------------------------------------------------------------ GPU arm
def sharded_config3(rmb, torch, dist, comm, world, rank, dev, sweeps=20):
    """BASELINE config 3 on N GPUs: each rank generates and owns
    its rmb_shard_range rows of the sparse 10^6 x 8 x 32 instance (col = global
    ids), V replicated; MB-VI b = n/8 for a fixed number of sweeps (the
    per-batch NCCL all-gather exchange).  Time = max over ranks of the device
    time of the solve (events on the solve's stream, inside the library)."""
    n, A, K = 1_000_000, 8, 32
    rows = rmb.shard_range(n, world, rank)
    rp, col, val, c = rmb.generate_sparse(n, A, K, 1, rows=rows)
    prob = rmb.Problem.csr(n, A, rp, col, val, c, 0.99, row_range=rows, nccl_comm=comm)
    prob.vi(n // 8, seed=0, eps=1e-300, max_sweeps=2)
    sol = prob.vi(n // 8, seed=1, eps=1e-300, max_sweeps=sweeps)
    t = torch.tensor([sol.stats.seconds], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t = float(t[0])
    del prob, rp, col, val, c
    torch.cuda.empty_cache()
    return {"workload": f"config 3 sharded over {world} GPUs: sparse random |S|=1e6 |A|=8 K=32 (ELL fp32), "
                        f"gamma=0.99, MB-VI b=n/8, {sweeps} sweeps", "scaling": "strong",
            "sweeps": sol.stats.sweeps, "ms_per_sweep": t / max(1, sol.stats.sweeps) * 1e3,
            "backups_per_s": sol.stats.sweeps * n * A / t}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--b", type=int, default=1000)
    ap.add_argument("--impl", default="rmb", choices=["rmb", "reference"])
    ap.add_argument("--no-bsweep", action="store_true", help="skip the per-b time-to-eps table")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-other", action="store_true", help="skip the config 3 / 4 secondary lines")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run (the
        # driver's own launch sets WORLD_SIZE and lands below)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if world_env != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch

    import paper_2110_02901_b200 as rmb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    comm = None
    if world == 1:
        P, c = rmb.generate_dense(N_STATES, N_ACTIONS, INST_SEED)
        prob = rmb.Problem.dense(P, c, GAMMA)
        rows = (0, N_STATES)
    else:
        # the sharded path: this rank's rows of the ONE config-2
        # instance, V replicated, per-batch NCCL all-gather of the updates
        rows = rmb.shard_range(N_STATES, world, rank)
        P, c = rmb.generate_dense(N_STATES, N_ACTIONS, INST_SEED, rows=rows)
        uid = [rmb.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = rmb.nccl_comm_init(world, rank, uid[0])
        prob = rmb.Problem.dense(P, c, GAMMA, n=N_STATES, row_range=rows, nccl_comm=comm)
    V = torch.zeros(N_STATES, dtype=torch.float64, device=dev)
    pi = torch.zeros(N_STATES, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > L2 (126 MB)

    # N > 1: the fused path (RMB_FUSED: exchange inside the persistent kernel
    # over NVLink peer memory); should it fail on this node, every rank falls
    # back to the per-batch NCCL all-gather protocol (same results)
    mode = {"fused": world > 1}

    def solve(b, seed=0):
        if mode["fused"]:
            try:
                return prob.vi(b, seed=seed, eps=EPS, max_sweeps=200_000, V=V, pi=pi, v0_zero=True, fused=True)
            except rmb.RmbError as e:
                print(f"bench.py: fused path unavailable ({e}); per-batch all-gather instead", file=sys.stderr)
                mode["fused"] = False
        return prob.vi(b, seed=seed, eps=EPS, max_sweeps=200_000, V=V, pi=pi, v0_zero=True)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
            torch.cuda.synchronize()

    for w in range(args.warmup):
        solve(args.b, seed=w)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sweeps = 0
    kernel_s = 0.0
    launches = 0
    with Clocks(local) as clk:
        barrier()
        ev0.record(stream)
        for s in range(args.steps):
            sol = solve(args.b, seed=100 + s)
            sweeps += sol.stats.sweeps
            kernel_s += sol.stats.seconds
            launches += prob.last_launch_count()
            flush.zero_()  # L2 flush between timed solves (P is > L2 anyway)
        ev1.record(stream)
        barrier()
    t = ev0.elapsed_time(ev1) / 1e3
    tt = torch.tensor([t, sweeps], dtype=torch.float64, device=dev)
    if dist:
        # one instance sharded over the ranks: every rank runs the same sweeps
        # and together they back up every state once per sweep; time = max
        tmax = tt.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        t = float(tmax[0])
    value = sweeps * N_STATES * N_ACTIONS / t

    # roofline of THIS rank's kernels: its rows of P per sweep
    frac_rows = (rows[1] - rows[0]) / N_STATES
    peak, peak_src = peaks()
    traffic = None
    try:  # DRAM bytes per sweep of the solver kernel from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        traffic = tj["dram_bytes_per_sweep"] * sweeps / args.steps  # per launch (= one solve)
    except Exception:
        pass
    bps = algo_bytes_per_sweep(N_STATES, N_ACTIONS, 4, args.b)
    if world > 1:
        bps = int(bps * frac_rows)
    achieved = sweeps * bps / kernel_s / 1e9  # per launch = whole solve kernel (N=1); per rank share (N>1)
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": arm_config(args.b, (f"shard{world} (rows by state, V replicated, " +
                                      ("fused in-kernel NVLink exchange per batch)" if mode["fused"]
                                       else "NCCL all-gather per batch)"))
                             if world > 1 else "dp1", {"sweeps_per_solve": sweeps / args.steps}),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_note": "dram read+write bytes per launch = per-sweep DRAM bytes of the committed "
                                     "ncu --set full capture (profiles/ncu_traffic.json) x sweeps per solve",
                     "achieved_bytes_per_launch": sweeps * bps / args.steps,
                     "peak_source": peak_src, "kernel": "dense_tma_kernel<float,4> (TMA ring path)",
                     "algorithmic_bytes_per_sweep": bps,
                     "peak_note": "MEASURED_PEAKS hbm_gbs is a device-to-device COPY (read+write turnaround); "
                                  "this kernel is a read stream (P) and can exceed it; frac_nominal is vs the "
                                  "8.0 TB/s HBM3e nominal",
                     "peak_nominal": 8000.0, "frac_nominal": achieved / 8000.0},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }

    if rank == 0 and world == 1 and not args.no_bsweep:
        table = []
        for b in (1, 64, 1000, 10_000):
            sol = solve(b, seed=7)
            st = sol.stats
            bb = algo_bytes_per_sweep(N_STATES, N_ACTIONS, 4, b)
            table.append({"b": b, "sweeps": st.sweeps, "batches_per_sweep": -(-N_STATES // b),
                          "time_to_eps_ms": st.seconds * 1e3,
                          "us_per_batch": st.seconds / max(1, st.batches) * 1e6,
                          "backups_per_s": st.sweeps * N_STATES * N_ACTIONS / st.seconds,
                          "GB_per_s": st.sweeps * bb / st.seconds / 1e9})
        result["time_to_eps_vs_b"] = table
    if rank == 0 and world == 1 and not args.no_other:
        result["vi_star_vs_mb_vi"] = vi_star_rows(rmb, torch, prob, V, pi)
        result["selection_and_async"] = f4_rows(rmb, torch, prob, V, pi)

    if rank == 0 and world == 1 and not args.no_e2e:
        # e2e through the C ABI with HOST buffers: H2D of P, c inside the timed region
        Ph = torch.empty(P.shape, dtype=P.dtype, pin_memory=True)
        ch = torch.empty(c.shape, dtype=c.dtype, pin_memory=True)
        Ph.copy_(P)
        ch.copy_(c)
        Vh = np.zeros(N_STATES)
        pih = np.zeros(N_STATES, np.int32)
        del prob
        torch.cuda.empty_cache()
        del P
        torch.cuda.empty_cache()

        def e2e_step(seed):
            p2 = rmb.Problem.dense(Ph, ch, GAMMA)
            sol = p2.vi(args.b, seed=seed, eps=EPS, max_sweeps=200_000, V=Vh, pi=pih, v0_zero=True)
            p2.close()
            return sol.stats.sweeps

        e2e_step(0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sw = 0
        ksteps = max(1, min(args.steps, 3))
        for s in range(ksteps):
            sw += e2e_step(100 + s)
        te = time.perf_counter() - t0
        result["e2e"] = {"value": sw * N_STATES * N_ACTIONS / te, "unit": UNIT,
                         "h2d_bytes_per_step": int(Ph.numel() * 4 + ch.numel() * 4),
                         "d2h_bytes_per_step": int(N_STATES * 8 + N_STATES * 4 + 8 * sw / ksteps),
                         "steps": ksteps, "path": "rmb_create_dense(host P,c) + rmb_vi(host V,pi) + rmb_destroy"}

    if rank == 0 and world == 1 and not args.no_other:
        result["other_configs"] = other_configs(rmb, torch, dev)
    if world > 1 and not args.no_other:
        line = sharded_config3(rmb, torch, dist, comm, world, rank, dev)
        if rank == 0:
            result["other_configs"] = [line]
    if not args.no_other:
        line = config5_line(rmb, torch, dist, comm, world, rank, dev)
        if rank == 0:
            result.setdefault("other_configs", []).append(line)

    if rank == 0 and world == 1 and not args.no_other:
        result["paper_envs"] = paper_envs(rmb, torch)

    if rank == 0 and world == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baselines(args.b)

    if rank == 0:
        print(json.dumps(result), flush=True)
    if dist:
        dist.barrier()
        del prob
        rmb.nccl_comm_destroy(comm)
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
