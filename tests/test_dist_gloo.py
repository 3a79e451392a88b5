"""Multi-process host logic on CPU (gloo, world_size 2, 127.0.0.1).

* every rank computes its receive plan from the all-gathered run-count matrix through
  gj_dist_plan -- the same host function join_dist_count* runs -- and the scatter
  it drives is simulated tuple by tuple: every receive slot is written exactly once,
  in digit-major / sender-rank / input order (see also test_dist_plan.py);
* the communicator-id broadcast used by paper_1904_11201_b200.Comm (object
  broadcast over the process group) delivers identical bytes to every rank;
* the oracle-side shard bookkeeping (global rids = rid_base + local row) composes:
  the union of per-shard hash joins of hash-partitioned shards equals the full join
  (the invariant the NCCL shuffle relies on), computed with the CPU oracle only.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _simulate(M, adjs, me, seg, need, lbits):
    """The shuffle scatter driven by the plans: sender q's tuples in its own
    (destination, digit, input) order get position pos; tuple (p, d, j) lands at
    index pos + adj_q[p, d] (mod 2^32) of rank p's buffer.  Checks every slot of
    rank `me`'s buffer is written once, in (digit, sender, input) order, and that
    seg / need describe it."""
    G, L = M.shape[0], 1 << lbits
    buf = {}
    for q in range(G):
        pos = 0
        for p in range(G):
            for d in range(L):
                for j in range(int(M[q, p, d])):
                    if p == me:
                        idx = (pos + int(adjs[q][p, d])) % (1 << 32)
                        if idx in buf:
                            return False
                        buf[idx] = (d, q, j)
                    pos += 1
    n = int(M[:, me, :].sum())
    if sorted(buf) != list(range(n)) or int(need[me]) != n:
        return False
    if [buf[i] for i in range(n)] != sorted(buf.values()):
        return False
    starts = [int(M[:, me, :d].sum()) for d in range(L + 1)]
    return list(map(int, seg)) == starts and all(int(need[p]) == int(M[:, p, :].sum()) for p in range(G))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import torch
        import paper_1904_11201_b200 as gj
        import oracle
        import gen

        lbits, L = 2, 4
        rng = np.random.default_rng(100 + rank)
        row = torch.tensor(rng.integers(0, 50, world * L), dtype=torch.int64)  # my sends [p, d]
        rows = [torch.zeros(world * L, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(rows, row)
        M = np.stack([r.numpy() for r in rows]).reshape(world, world, L).astype(np.uint64)
        adj, seg, need = gj.dist_plan(M, rank, lbits)
        adjs = [None] * world
        dist.all_gather_object(adjs, adj)
        ok_plan = _simulate(M, adjs, rank, seg, need, lbits)
        blob = [os.urandom(gj.COMM_ID_BYTES) if rank == 0 else None]
        dist.broadcast_object_list(blob, src=0)
        gathered = [None] * world
        dist.all_gather_object(gathered, blob[0])
        ok_id = all(g == gathered[0] for g in gathered) and len(gathered[0]) == gj.COMM_ID_BYTES

        # shard bookkeeping with the oracle: rank owns keys with hash bucket == rank
        n = 4000
        R = gen.uniform_keys(n * world, 3000, 7, 0)
        S = gen.uniform_keys(n * world, 3000, 7, 1)
        owner_R = (R.astype(np.int64) * 2654435761) % world
        owner_S = (S.astype(np.int64) * 2654435761) % world
        rR = np.nonzero(owner_R == rank)[0]
        rS = np.nonzero(owner_S == rank)[0]
        c, p = oracle.hash_equi(R[rR], S[rS])
        mine = np.stack([rR[p[:, 0]], rS[p[:, 1]]], 1)
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        union = np.concatenate(allp)
        union = union[np.lexsort((union[:, 1], union[:, 0]))].astype(np.uint32)
        ok_union = np.array_equal(union, oracle.hash_equi(R, S)[1])
        q.put((rank, ok_plan, ok_id, ok_union))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_host_logic():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_plan, ok_id, ok_union in res:
        assert ok_plan, f"rank {rank}: receive plan mismatch"
        assert ok_id, f"rank {rank}: comm id broadcast mismatch"
        assert ok_union, f"rank {rank}: sharded joins do not compose to the full join"
