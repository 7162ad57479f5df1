"""One-GPU smoke test of bench.py's multi-rank code path: torch.distributed
with the NCCL backend at world size 1, NCCL id broadcast, slab engine with an
attached communicator.  Run: torchrun --nproc-per-node 1 --master-addr
127.0.0.1 --master-port 29511 tools/dist_smoke.py"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_10279_b200 as pk  # noqa: E402
from paper_1712_10279_b200 import distributed as D, synthetic  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
n = 1024
b = D.slab_bounds(n, world)
l0, l1 = synthetic.rgb_disk_rows(n, b[rank], b[rank + 1])
cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", tol_gap=1e-300, tol_feas=1e-300,
                      max_iters=300, check_every=100)
uid = D.share_unique_id(dist, rank)
rep, st = D.solve_vector_rows(l0, l1, pk.triangle_graph(), n, cfg, nranks=world, rank=rank,
                              unique_id=uid)
t = torch.tensor([rep.transport_value], device="cuda")
dist.all_reduce(t)
print("rank", rank, "iterations", rep.iterations, "value", rep.transport_value, float(t[0]))
dist.barrier()
dist.destroy_process_group()
