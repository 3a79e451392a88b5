"""NCCL exchange microbenchmark (torchrun, 2+ GPUs): all_to_all_single and batched
send/recv of ~1 GiB per rank, with and without a self-send slot.  Prints GB/s
per direction per rank (max over ranks of device time)."""
import os
import time

import torch
import torch.distributed as dist


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return ms.item()


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    n = 1 << 28  # int32 elements per rank = 1 GiB
    x = torch.randint(0, 100, (n,), dtype=torch.int32, device="cuda")
    y = torch.empty_like(x)
    ms = timed(lambda: dist.all_to_all_single(y, x))
    sent = n * 4 * (world - 1) / world
    if rank == 0:
        print(f"all_to_all_single 1GiB/rank: {ms:.3f} ms  {sent / ms / 1e6:.1f} GB/s off-rank per direction")
    chunk = n // world

    def p2p(self_send):
        ops = []
        for p in range(world):
            if p == rank and not self_send:
                y[p * chunk:(p + 1) * chunk].copy_(x[p * chunk:(p + 1) * chunk])
                continue
            ops.append(dist.P2POp(dist.isend, x[p * chunk:(p + 1) * chunk], p))
            ops.append(dist.P2POp(dist.irecv, y[p * chunk:(p + 1) * chunk], p))
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    for ss in (True, False):
        ms = timed(lambda: p2p(ss))
        if rank == 0:
            print(f"batch send/recv self_send={ss}: {ms:.3f} ms  {sent / ms / 1e6:.1f} GB/s")

    # the join shuffle's shape: 4 messages per peer (R keys, R rids, S keys, S rids)
    def p2p_split(parts):
        ops = []
        sub = chunk // parts
        for p in range(world):
            if p == rank:
                continue
            for q in range(parts):
                a = p * chunk + q * sub
                ops.append(dist.P2POp(dist.isend, x[a:a + sub], p))
                ops.append(dist.P2POp(dist.irecv, y[a:a + sub], p))
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    for parts in (1, 4, 16):
        ms = timed(lambda: p2p_split(parts))
        if rank == 0:
            print(f"batch send/recv {parts} msgs/peer: {ms:.3f} ms  {sent / ms / 1e6:.1f} GB/s")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
