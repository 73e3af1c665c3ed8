"""CPU, world_size-2 `gloo` test of the multi-GPU exchange protocol.

Each process owns the rows rmb_shard_range() gives it (product host code),
draws every sweep's partition with rmb_partition() (product host code), backs
up its states of each batch against its replica V (oracle arithmetic, one
state at a time), packs (state, value, argmin) into the fixed-capacity record
the library exchanges (cap = min(b, ceil(n/G))), all-gathers the records over
torch.distributed (gloo here, NCCL on GPUs) and commits every rank's updates.
The result must equal the single-process oracle MB-VI bit for bit: the
protocol realises Eq. 12 exactly and is independent of the number of ranks.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
import paper_2110_02901_b200 as rmb

N, A, GAMMA, SEED, EPS = 37, 3, 0.9, 5, 1e-9


K = 6  # successors per (s, a) of the sparse variant


def backup_fn(kind, r0, r1):
    """This rank's backup of a state s (owned rows only: dense rows, or CSR rows
    generated for [r0, r1) with global successor ids)."""
    if kind == "dense":
        P, c = gen.dense(N, A, 11, dtype=np.float64)
        Pl, cl = P[r0:r1], c[r0:r1]
        return lambda s, V: oracle.backup_dense_row(Pl[s - r0], cl[s - r0], GAMMA, V)
    rp, col, val, cl = gen.sparse(N, A, K, 11, dtype=np.float64, rows=(r0, r1))

    def f(s, V):
        q = s - r0
        rows = rp[q * A:(q + 1) * A + 1]
        return oracle.backup_csr_row(N, rows - rows[0], col[rows[0]:rows[-1]], val[rows[0]:rows[-1]], cl[q],
                                     GAMMA, V)
    return f


def sharded_vi(rank, world, b, sweeps, kind="dense"):
    r0, r1 = rmb.shard_range(N, world, rank)
    backup = backup_fn(kind, r0, r1)
    cap = min(b, -(-N // world))
    V = np.zeros(N)
    pi = np.zeros(N, np.int32)
    trace = []
    for k in range(1, sweeps + 1):
        perm = rmb.partition(N, SEED, k)
        r = 0.0
        for lo in range(0, N, b):
            batch = perm[lo:lo + b]
            mine = [int(s) for s in batch if r0 <= s < r1]
            assert len(mine) <= cap
            rec = torch.zeros(1 + 3 * cap, dtype=torch.float64)
            rec[0] = len(mine)
            for q, s in enumerate(mine):
                v, a = backup(s, V)
                rec[1 + q], rec[1 + cap + q], rec[1 + 2 * cap + q] = v, s, a
            recs = [torch.zeros_like(rec) for _ in range(world)]
            dist.all_gather(recs, rec)
            for g in range(world):
                cnt = int(recs[g][0])
                for q in range(cnt):
                    v = float(recs[g][1 + q])
                    s = int(recs[g][1 + cap + q])
                    r = max(r, abs(v - V[s]))
                    V[s] = v
                    if r0 <= s < r1:
                        pi[s] = int(recs[g][1 + 2 * cap + q])
        trace.append(r)
    return V, pi, np.array(trace), (r0, r1)


def _worker(rank, world, port, b, sweeps, out, kind):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        V, pi, tr, (r0, r1) = sharded_vi(rank, world, b, sweeps, kind)
        out[rank] = (V, pi[r0:r1], tr, r0, r1)
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("kind", ["dense", "sparse"])
@pytest.mark.parametrize("b", [1, 4, 10, N])
def test_two_rank_gloo_protocol_equals_oracle(b, kind):
    world, sweeps = 2, 6
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), b, sweeps, out, kind), nprocs=world, join=True)
        res = dict(out)
    if kind == "dense":
        P, c = gen.dense(N, A, 11, dtype=np.float64)
        m = oracle.MDP(N, A, GAMMA, c, P=P)
    else:
        rp, col, val, c = gen.sparse(N, A, K, 11, dtype=np.float64)
        m = oracle.MDP(N, A, GAMMA, c, row_ptr=rp, col=col, val=val)
    ref = oracle.vi(m, b, seed=SEED, eps=1e-300, max_sweeps=sweeps)
    pi = np.zeros(N, np.int32)
    for rank in range(world):
        V, pil, tr, r0, r1 = res[rank]
        assert np.array_equal(V, ref.V)          # every replica is the oracle's V, bit for bit
        assert np.array_equal(tr, ref.trace)     # and so is the residual trace
        pi[r0:r1] = pil
    assert np.array_equal(pi, ref.pi)


def test_shard_ranges_partition_the_states():
    for n in (1, 2, 5, 37, 10_000, 50_000):
        for G in (1, 2, 3, 4, 7, 8):
            spans = [rmb.shard_range(n, G, g) for g in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
                assert e0 == b1 and b0 <= e0
            assert max(e - b for b, e in spans) == -(-n // G)


# ------------------------------------------------- fused exchange (K8f) model
def fused_mpi(rank, world, b, msweeps, outer_iters):
    """The fused multi-rank protocol of the dense kernel (RMB_FUSED) step by
    step on CPU: per batch each rank builds the list of its states (order-free:
    shuffled on purpose), backs them up against its replica, stores (value,
    argmin) at their batch POSITIONS into every rank's exchange arrays (here: a
    position-indexed array all-gathered, each position written by its owner
    only), meets the others (the collective), then patches ALL of the batch from
    its own arrays.  Improvements run on the owned states only, and (residual,
    changed) records are exchanged and reduced.  MB-MPI from V0 = 0, pi_0 =
    greedy(V0)."""
    r0, r1 = rmb.shard_range(N, world, rank)
    P, c = gen.dense(N, A, 11, dtype=np.float64)
    m = oracle.MDP(N, A, GAMMA, c, P=P)
    rng = np.random.default_rng(rank)
    V = np.zeros(N)
    pi = np.zeros(N, np.int32)

    def improve_owned():
        rT, ch = 0.0, 0
        for s in range(r0, r1):
            q, a = oracle.backup_dense_row(P[s], c[s], GAMMA, V)
            rT = max(rT, abs(q - V[s]))
            ch += int(a != pi[s])
            pi[s] = a
        rec = torch.tensor([rT, float(ch)], dtype=torch.float64)
        recs = [torch.zeros_like(rec) for _ in range(world)]
        dist.all_gather(recs, rec)
        return max(float(x[0]) for x in recs), int(sum(float(x[1]) for x in recs))

    improve_owned()  # pi_0 = greedy(V0)
    k, trace, changed = 1, [], []
    for o in range(outer_iters):
        for e in range(msweeps):
            perm = rmb.partition(N, SEED, k)
            k += 1
            r = 0.0
            for lo in range(0, N, b):
                cnt = min(b, N - lo)
                own = [(i, int(perm[lo + i])) for i in range(cnt) if r0 <= perm[lo + i] < r1]
                rng.shuffle(own)  # list order is irrelevant to every state's arithmetic
                xval = torch.zeros(cnt, dtype=torch.float64)
                for i, s in own:
                    xval[i], _ = oracle.backup_dense_row(P[s], c[s], GAMMA, V, pi_a=int(pi[s]))
                parts = [torch.zeros_like(xval) for _ in range(world)]
                dist.all_gather(parts, xval)  # each rank's stores land in every rank's arrays
                mine = parts[0].clone()
                for g in range(1, world):
                    mine += parts[g]  # positions are disjoint across ranks: exact
                for i in range(cnt):
                    s = int(perm[lo + i])
                    r = max(r, abs(float(mine[i]) - V[s]))
                    V[s] = float(mine[i])
            trace.append(r)
        rT, ch = improve_owned()
        trace.append(rT)
        changed.append(ch)
    return V, pi[r0:r1], np.array(trace), np.array(changed), (r0, r1)


def _fused_worker(rank, world, port, b, msweeps, outer, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        V, pil, tr, ch, (r0, r1) = fused_mpi(rank, world, b, msweeps, outer)
        out[rank] = (V, pil, tr, ch, r0, r1)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("b", [1, 7, N])
def test_two_rank_gloo_fused_protocol_mpi_equals_oracle(b):
    world, msweeps, outer = 2, 3, 4
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_fused_worker, args=(world, _free_port(), b, msweeps, outer, out), nprocs=world, join=True)
        res = dict(out)
    P, c = gen.dense(N, A, 11, dtype=np.float64)
    ref = oracle.mpi(oracle.MDP(N, A, GAMMA, c, P=P), b, msweeps, seed=SEED, eps=1e-300, max_outer=outer)
    pi = np.zeros(N, np.int32)
    for rank in range(world):
        V, pil, tr, ch, r0, r1 = res[rank]
        assert np.array_equal(V, ref.V) and np.array_equal(tr, ref.trace)
        assert np.array_equal(ch, ref.changed)
        pi[r0:r1] = pil
    assert np.array_equal(pi, ref.pi)
