"""Sharded protocol overhead at 1 rank (real 1-rank NCCL communicator) on
BASELINE config 2 (dense 10^4 x 16 fp32, b = 1000), next to the persistent
single-GPU solver: ms per sweep of each."""
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
for b in (1000, 64):
    she = rmb.Problem.dense(P, c, 0.99, n=n, row_range=(0, n), nccl_comm=comm, flags=rmb.SHARD_NO_GRAPH)
    she.vi(b, seed=0, eps=1e-300, max_sweeps=2)
    se = she.vi(b, seed=1, eps=1e-300, max_sweeps=20)
    she.close()
    sh = rmb.Problem.dense(P, c, 0.99, n=n, row_range=(0, n), nccl_comm=comm)
    sh.vi(b, seed=0, eps=1e-300, max_sweeps=2)
    s = sh.vi(b, seed=1, eps=1e-300, max_sweeps=20)
    one = rmb.Problem.dense(P, c, 0.99)
    one.vi(b, seed=0, eps=1e-300, max_sweeps=2)
    r = one.vi(b, seed=1, eps=1e-300, max_sweeps=20)
    out[f"b={b}"] = {"sharded_1rank_ms_per_sweep": s.stats.seconds / s.stats.sweeps * 1e3,
                     "sharded_1rank_eager_ms_per_sweep": se.stats.seconds / se.stats.sweeps * 1e3,
                     "persistent_ms_per_sweep": r.stats.seconds / r.stats.sweeps * 1e3,
                     "sharded_launches": sh.last_launch_count()}
    sh.close()
    one.close()
print(json.dumps(out))
rmb.nccl_comm_destroy(comm)
dist.destroy_process_group()
