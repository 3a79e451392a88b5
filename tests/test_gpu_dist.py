"""Multi-GPU parity (NCCL, one process per GPU): join_dist_* / theta_join_dist_*
vs the CPU oracle on the union of all ranks' outputs.  Skips below 2 GPUs."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


C5_FLAGS = (7, 1, 2)  # RANGE|BLOOM|TWO_SIDED, RANGE only, BLOOM only


def _c5_inputs():
    """gen.c5 over a 2^16-row domain: R = 2*perm(i) unique, S 10% members else odd keys."""
    import gen
    return gen.c5(1 << 16, 1 << 18, seed=21, b=16)


def _i64_inputs():
    """int64 keys spread over +-2^56 (upper hash bits exercised), duplicates on both sides."""
    import gen
    R = gen.uniform_keys(60_000, 40_000, 12, 0, dtype=np.int64) * np.int64(1 << 35) - np.int64(1 << 56)
    S = gen.uniform_keys(250_000, 50_000, 12, 1, dtype=np.int64) * np.int64(1 << 35) - np.int64(1 << 56)
    return R, S


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        import gen
        import paper_1904_11201_b200 as gj
        ctx = gj.Context(rank)
        comm = gj.Comm(rank, world)
        out = {}
        # equi: PK-FK Zipf, block-sharded; rid_base = global row offset
        b = 18
        q_tab = gen.zipf_table(1 << b)
        Rall, Sall, m = gen.zipf_pkfk(b, 1 << 20, q_tab, seed=5)
        nr, ns = len(Rall) // world, len(Sall) // world
        Rk = torch.from_numpy(Rall[rank * nr:(rank + 1) * nr]).cuda()
        Sk = torch.from_numpy(Sall[rank * ns:(rank + 1) * ns]).cuda()
        R = gj.Rel(Rk, None, rank * nr)
        S = gj.Rel(Sk, None, rank * ns)
        nl, ng = gj.join_dist_count(ctx, comm, R, S)
        pairs = gj.join_dist_materialize(ctx, comm, R, S, nl).cpu().numpy().view(np.uint32)
        out["equi"] = (nl, ng, pairs)
        # duplicates on both sides, uneven shards
        R2all = gen.uniform_keys(30_001, 2000, 3, 0)
        S2all = gen.uniform_keys(40_003, 2000, 3, 1)
        r0, r1 = (rank * len(R2all)) // world, ((rank + 1) * len(R2all)) // world
        s0, s1 = (rank * len(S2all)) // world, ((rank + 1) * len(S2all)) // world
        R2 = gj.Rel(torch.from_numpy(R2all[r0:r1]).cuda(), None, r0)
        S2 = gj.Rel(torch.from_numpy(S2all[s0:s1]).cuda(), None, s0)
        nl, ng = gj.join_dist_count(ctx, comm, R2, S2)
        out["dup"] = (nl, ng, gj.join_dist_materialize(ctx, comm, R2, S2, nl).cpu().numpy().view(np.uint32))
        # a single-GPU join on the same ctx between the dist count and materialize must
        # not leak into the dist output (the dist cache checks the ctx's fill epoch)
        nl, ng = gj.join_dist_count(ctx, comm, R2, S2)
        tiny = torch.arange(100, dtype=torch.int32, device="cuda")
        assert gj.join_count(ctx, tiny, tiny) == 100
        out["dup_epoch"] = (nl, ng, gj.join_dist_materialize(ctx, comm, R2, S2, nl).cpu().numpy().view(np.uint32))
        # shards that are views at element offsets (not 16-byte aligned): R2[1:], S2[3:]
        # of the same global rows, through the fused NVLink shuffle's bulk copies
        bigR = torch.from_numpy(R2all[max(r0 - 1, 0):r1]).cuda()
        bigS = torch.from_numpy(S2all[max(s0 - 3, 0):s1]).cuda()
        R2u = gj.Rel(bigR[r0 - max(r0 - 1, 0):], None, r0)
        S2u = gj.Rel(bigS[s0 - max(s0 - 3, 0):], None, s0)
        nl, ng = gj.join_dist_count(ctx, comm, R2u, S2u)
        out["dup_unaligned"] = (nl, ng, gj.join_dist_materialize(ctx, comm, R2u, S2u, nl).cpu().numpy().view(np.uint32))
        # local radix digits folded into the NVLink shuffle (receivers lay out digit-major):
        # (a) 3 radix bits in all, so the shuffle's local digit alone forms the partitions
        ctx.set_option("shuffle_bits", 8)
        ctx.set_option("part_bits", 3)
        nl, ng = gj.join_dist_count(ctx, comm, R2, S2)
        out["dup_pb3"] = (nl, ng, gj.join_dist_materialize(ctx, comm, R2, S2, nl).cpu().numpy().view(np.uint32))
        ctx.set_option("part_bits", -1)
        # (b) 6 folded bits + the remaining radix bits of the local join on top
        ctx.set_option("shuffle_bits", 6)
        nl, ng = gj.join_dist_count(ctx, comm, R, S)
        out["equi_sb6"] = (nl, ng, gj.join_dist_materialize(ctx, comm, R, S, nl).cpu().numpy().view(np.uint32))
        ctx.set_option("shuffle_bits", 0)
        # int64 keys (configs[4] shape, C5 recipe), rank 0 holds no R rows; larger than the
        # calls above, so the receive buffers grow and the IPC handles are re-exchanged
        R4all, S4all = _i64_inputs()
        r0, r1 = (0, 0) if rank == 0 else ((rank - 1) * len(R4all) // (world - 1), rank * len(R4all) // (world - 1))
        s0, s1 = (rank * len(S4all)) // world, ((rank + 1) * len(S4all)) // world
        R4 = gj.Rel(torch.from_numpy(R4all[r0:r1]).cuda(), None, r0)
        S4 = gj.Rel(torch.from_numpy(S4all[s0:s1]).cuda(), None, s0)
        nl, ng = gj.join_dist_count(ctx, comm, R4, S4)
        out["i64"] = (nl, ng, gj.join_dist_materialize(ctx, comm, R4, S4, nl).cpu().numpy().view(np.uint32))
        # configs[4] shape (int64, 10% S members), pre-filtered join: range by all-reduce,
        # R shuffled first, per-owner Bloom filters all-gathered, S filtered at the source
        R5all, S5all, _ = _c5_inputs()
        a0, a1 = (rank * len(R5all)) // world, ((rank + 1) * len(R5all)) // world
        c0, c1 = (rank * len(S5all)) // world, ((rank + 1) * len(S5all)) // world
        R5 = gj.Rel(torch.from_numpy(R5all[a0:a1]).cuda(), None, a0)
        S5 = gj.Rel(torch.from_numpy(S5all[c0:c1]).cuda(), None, c0)
        for flags in (7, 3, 1):  # standalone sharded pre-filter: this rank's own survivors
            kR, rR, kS, rS = gj.prefilter_dist(ctx, comm, R5, S5, flags)
            out[f"pfd{flags}"] = (rR.cpu().numpy().view(np.uint32), rS.cpu().numpy().view(np.uint32),
                                  kR.cpu().numpy(), kS.cpu().numpy(), (a0, a1, c0, c1))
        for flags in C5_FLAGS:
            nl, ng, kept = gj.join_dist_count_filtered(ctx, comm, R5, S5, flags, 8.0)
            out[f"c5pf{flags}"] = (nl, ng, gj.join_dist_materialize(ctx, comm, R5, S5, nl).cpu().numpy().view(
                np.uint32))
            out[f"kept{flags}"] = kept
        # theta band: R replicated, S sharded
        R3all = gen.uniform_keys(5000, 1 << 20, 8, 0)
        S3all = gen.uniform_keys(20_000, 1 << 20, 8, 1)
        a0, a1 = (rank * 5000) // world, ((rank + 1) * 5000) // world
        c0, c1 = (rank * 20_000) // world, ((rank + 1) * 20_000) // world
        R3 = gj.Rel(torch.from_numpy(R3all[a0:a1]).cuda(), None, a0)
        S3 = gj.Rel(torch.from_numpy(S3all[c0:c1]).cuda(), None, c0)
        nl, ng = gj.theta_join_dist_count(ctx, comm, R3, S3, "band", 40)
        out["band"] = (nl, ng, gj.theta_join_dist_materialize(ctx, comm, R3, S3, "band", 40, nl).cpu().numpy().view(
            np.uint32))
        # 1-Bucket grid (NEXT f3): r x (G/r) ranks, R block per grid row, S block per grid column
        for rows in sorted({world, 2}):
            ctx.set_option("theta_grid_rows", rows)
            nl, ng = gj.theta_join_dist_count(ctx, comm, R3, S3, "band", 40)
            out[f"band_grid{rows}"] = (nl, ng, gj.theta_join_dist_materialize(ctx, comm, R3, S3, "band", 40, nl)
                                       .cpu().numpy().view(np.uint32))
            g0, g1 = (rank * 2000) // world, ((rank + 1) * 2000) // world
            h0, h1 = (rank * 3000) // world, ((rank + 1) * 3000) // world
            R6 = gj.Rel(torch.from_numpy(R3all[:2000][g0:g1]).cuda(), None, g0)
            S6 = gj.Rel(torch.from_numpy(S3all[:3000][h0:h1]).cuda(), None, h0)
            nl, ng = gj.theta_join_dist_count(ctx, comm, R6, S6, "ge", 0)
            out[f"ge_grid{rows}"] = (nl, ng, gj.theta_join_dist_materialize(ctx, comm, R6, S6, "ge", 0, nl)
                                     .cpu().numpy().view(np.uint32))
        ctx.set_option("theta_grid_rows", 0)
        # GJ_OPT_CHECK_ARGS: a rank passing a different eps makes EVERY rank fail with
        # GJ_EINVAL (instead of a silently wrong union); equal arguments pass
        ctx.set_option("check_args", 1)
        nl, ng = gj.theta_join_dist_count(ctx, comm, R3, S3, "band", 40)
        try:
            gj.theta_join_dist_count(ctx, comm, R3, S3, "band", 40 + rank)
            out["argcheck"] = "no error"
        except gj.GJError as e:
            out["argcheck"] = e.status
        ctx.set_option("check_args", 0)
        q.put((rank, out))
        comm.close()
        ctx.close()
    finally:
        dist.destroy_process_group()


def _canon(p):
    p = np.asarray(p, dtype=np.uint32).reshape(-1, 2)
    return p[np.lexsort((p[:, 1], p[:, 0]))]


@pytest.mark.timeout(400)
@pytest.mark.parametrize("world", [2, 4])
def test_dist_joins_match_oracle(world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import gen
    import oracle
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, o = q.get(timeout=300)
            res[r] = o
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.exitcode is None:
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    b = 18
    Rall, Sall, m = gen.zipf_pkfk(b, 1 << 20, gen.zipf_table(1 << b), seed=5)
    R2all, S2all = gen.uniform_keys(30_001, 2000, 3, 0), gen.uniform_keys(40_003, 2000, 3, 1)
    R3all, S3all = gen.uniform_keys(5000, 1 << 20, 8, 0), gen.uniform_keys(20_000, 1 << 20, 8, 1)
    R4all, S4all = _i64_inputs()
    dup = oracle.hash_equi(R2all, S2all)
    pk = oracle.pkfk_closed_form(m)
    expect = {"equi": pk, "equi_sb6": pk, "dup": dup, "dup_pb3": dup, "dup_epoch": dup, "dup_unaligned": dup,
              "i64": oracle.hash_equi(R4all, S4all), "band": oracle.band_materialize(R3all, S3all, 40)}
    for rows in sorted({world, 2}):
        expect[f"band_grid{rows}"] = expect["band"]
        expect[f"ge_grid{rows}"] = oracle.nlj(R3all[:2000], S3all[:3000], "ge")
    R5all, S5all, m5 = _c5_inputs()
    import paper_1904_11201_b200 as gj
    pk5 = oracle.pkfk_closed_form(m5)
    members = int((m5 >= 0).sum())
    lo, hi = max(R5all.min(), S5all.min()), min(R5all.max(), S5all.max())
    in_range = (int(((R5all >= lo) & (R5all <= hi)).sum()), int(((S5all >= lo) & (S5all <= hi)).sum()))
    for flags in C5_FLAGS:
        expect[f"c5pf{flags}"] = pk5
        kept_R = sum(res[r][f"kept{flags}"][0] for r in range(world))
        kept_S = sum(res[r][f"kept{flags}"][1] for r in range(world))
        assert members <= kept_S <= len(S5all), flags  # no false negatives
        if flags == gj.RANGE:
            assert (kept_R, kept_S) == in_range, flags
        if flags & gj.BLOOM:  # 8 bits/key: ~2-3% false positives among the 90% non-members
            assert kept_S < members + 0.08 * len(S5all), (flags, kept_S)
        if flags & gj.TWO_SIDED:
            assert kept_R < len(R5all), flags
    assert all(res[r]["argcheck"] == 1 for r in range(world)), [res[r]["argcheck"] for r in range(world)]
    # prefilter_dist: each rank's survivors are its own rows, in order, with their keys;
    # no false negatives (the exact semi-joins survive); the union joins to J(R, S)
    semR = set(np.nonzero(oracle.semijoin_exact(R5all, S5all))[0].tolist())
    semS = set(np.nonzero(oracle.semijoin_exact(S5all, R5all))[0].tolist())
    for flags in (7, 3, 1):
        allR, allS = [], []
        for r in range(world):
            rR, rS, kR, kS, (a0, a1, c0, c1) = res[r][f"pfd{flags}"]
            assert np.all((rR >= a0) & (rR < a1)) and np.all((rS >= c0) & (rS < c1)), flags
            assert np.all(np.diff(rR.astype(np.int64)) > 0) and np.all(np.diff(rS.astype(np.int64)) > 0), flags
            assert np.array_equal(kR, R5all[rR]) and np.array_equal(kS, S5all[rS]), flags
            allR.append(rR)
            allS.append(rS)
        allR, allS = np.concatenate(allR), np.concatenate(allS)
        assert semS <= set(allS.tolist()), flags
        if flags & gj.TWO_SIDED:
            assert semR <= set(allR.tolist()) and len(allR) < len(R5all), flags
        c, p = oracle.hash_equi(R5all[allR], S5all[allS])
        p = np.stack([allR[p[:, 0]], allS[p[:, 1]]], 1).astype(np.uint32)
        assert np.array_equal(_canon(p), pk5[1]), flags
    for name, (cnt, pairs) in expect.items():
        locals_ = [res[r][name] for r in range(world)]
        assert all(l[1] == cnt for l in locals_), name  # n_global
        assert sum(l[0] for l in locals_) == cnt, name  # n_local adds up
        union = _canon(np.concatenate([l[2] for l in locals_]))
        assert np.array_equal(union, pairs), name
