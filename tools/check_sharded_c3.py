"""GPU check of bench.sharded_config3 on ONE rank (1-rank NCCL communicator):
the sharded sparse protocol at config-3 size, timed like the N > 1 bench line,
next to the single-handle persistent solver."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2110_02901_b200 as rmb  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
comm = rmb.nccl_comm_init(1, 0, rmb.nccl_unique_id())
line = bench.sharded_config3(rmb, torch, dist, comm, 1, 0, torch.device("cuda", 0))
print(json.dumps(line))
rmb.nccl_comm_destroy(comm)
dist.destroy_process_group()
