"""Multi-GPU protocol overhead at 1 rank (real 1-rank NCCL communicator) on
BASELINE config 2 (dense 10^4 x 16 fp32), next to the persistent single-GPU
solver: ms per sweep of the fused path (RMB_FUSED: in-kernel exchange), the
host-driven protocol (per-batch NCCL all-gather, graph replay and eager), and
8 logical fused ranks sharing the one device."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_02901_b200 as rmb  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29534")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
comm = rmb.nccl_comm_init(1, 0, rmb.nccl_unique_id())
n, A = 10_000, 16
P, c = rmb.generate_dense(n, A, 1)
out = {}


def per_sweep(f):
    f(seed=0, max_sweeps=2)
    s = f(seed=1, max_sweeps=20)
    return s.stats.seconds / s.stats.sweeps * 1e3, s


for b in (1000, 64):
    row = {}
    one = rmb.Problem.dense(P, c, 0.99)
    row["persistent_ms_per_sweep"], ref = per_sweep(lambda **k: one.vi(b, eps=1e-300, **k))
    sh = rmb.Problem.dense(P, c, 0.99, n=n, row_range=(0, n), nccl_comm=comm)
    row["fused_1rank_ms_per_sweep"], fs = per_sweep(lambda **k: sh.vi(b, eps=1e-300, fused=True, **k))
    row["fused_bitwise"] = bool(torch.equal(fs.V, ref.V))
    row["host_protocol_1rank_graph_ms_per_sweep"], _ = per_sweep(lambda **k: sh.vi(b, eps=1e-300, **k))
    sh.close()
    she = rmb.Problem.dense(P, c, 0.99, n=n, row_range=(0, n), nccl_comm=comm, flags=rmb.SHARD_NO_GRAPH)
    row["host_protocol_1rank_eager_ms_per_sweep"], _ = per_sweep(lambda **k: she.vi(b, eps=1e-300, **k))
    she.close()
    hs = [rmb.Problem.dense(P[r0:r1], c[r0:r1], 0.99, n=n, row_range=(r0, r1))
          for r0, r1 in (rmb.shard_range(n, 8, g) for g in range(8))]
    row["fused_8_logical_ranks_one_gpu_ms_per_sweep"], g8 = per_sweep(
        lambda **k: rmb.vi_group(hs, b, eps=1e-300, fused=True, **k))
    row["fused_8_bitwise"] = bool(torch.equal(g8.V, ref.V))
    row["phases_8_logical"] = hs[0].last_phase_times()
    for h in hs:
        h.close()
    one.close()
    out[f"b={b}"] = row
    print(json.dumps({f"b={b}": row}), flush=True)
rmb.nccl_comm_destroy(comm)
dist.destroy_process_group()
