"""Debug helper (GPU box): int64 distributed equi-join counts, fused vs NCCL shuffle vs 1 GPU.
torchrun --nproc-per-node 2 tools/dbg_dist.py"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_1904_11201_b200 as gj  # noqa: E402
from test_gpu_dist import _i64_inputs  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
ctx = gj.Context(rank)
comm = gj.Comm(rank, world)
R4all, S4all = _i64_inputs()
if rank == 0:
    import oracle
    print("oracle", oracle.hash_equi(R4all, S4all)[0], flush=True)
    print("single", gj.join_count(ctx, gj.Rel(torch.from_numpy(R4all).cuda()), gj.Rel(torch.from_numpy(S4all).cuda())),
          flush=True)
for variant in ["r0empty", "even"]:
    if variant == "r0empty":
        r0, r1 = (0, 0) if rank == 0 else ((rank - 1) * len(R4all) // (world - 1), rank * len(R4all) // (world - 1))
    else:
        r0, r1 = rank * len(R4all) // world, (rank + 1) * len(R4all) // world
    s0, s1 = (rank * len(S4all)) // world, ((rank + 1) * len(S4all)) // world
    for dt in [np.int64, np.int32]:
        Rk = torch.from_numpy((R4all[r0:r1] >> (35 if dt == np.int32 else 0)).astype(dt)).cuda()
        Sk = torch.from_numpy((S4all[s0:s1] >> (35 if dt == np.int32 else 0)).astype(dt)).cuda()
        R4 = gj.Rel(Rk, None, r0)
        S4 = gj.Rel(Sk, None, s0)
        for sh in ["fused", "nccl"]:
            if sh == "nccl":
                os.environ["GJ_SHUFFLE"] = "nccl"
            else:
                os.environ.pop("GJ_SHUFFLE", None)
            nl, ng = gj.join_dist_count(ctx, comm, R4, S4)
            print(f"rank {rank} {variant} {dt.__name__} {sh}: local {nl} global {ng}", flush=True)
comm.close()
ctx.close()
dist.destroy_process_group()
