#!/usr/bin/env python
"""Benchmark of the GPU join hot path (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c1|c2|c3|c4|c5] [--impl ours|reference]

Default workload (N=1): BASELINE.json configs[1] -- equi hash join of 2^27 x 2^27
8-byte tuples (int32 key + int32 payload; payload never read), PK-FK "unique-ish"
keys.  One step = the whole exact join: radix partition R and S,
build/probe count, exclusive scan, D2H of |J|, build/probe write of all |J| pairs.
Inputs are generated in HBM by the seeded generator twin before timing (1 GiB of
keys > the 126 MB L2, so no L2 flush is needed between steps).

`value` = input tuples/s = (n_R + n_S) * K / T (device time, CUDA events on the
ctx stream, max over ranks).  `e2e` = the same metric through the host-buffer C-ABI
entry `join_host` (pinned H2D of both key columns + D2H of all pairs inside the
timed region).  `roofline` = the dominant kernel's algorithmic bytes per launch /
its mean launch time (CUDA events around every launch on the ctx stream, in a
second, profiled pass of the same K steps) vs MEASURED_PEAKS.json hbm_gbs.
`cpu_baseline` = the CPU oracle timed on a bounded sample of the same workload on this
host: O7 (O2's unordered_multimap hash join sliced by key hash over all host threads)
as the value, O2 on one thread beside it.

--impl reference: this tier has no runnable reference implementation; the
reference arm is the oracle itself, timed the same way on the host cores.

N > 1 (torchrun): weak scaling -- every rank holds a same-size shard of one global
join.  Equi (c2): join_dist_count/materialize = a hash shuffle by the top log2(N)
hash bits fused into the first radix scatter (NVLink peer stores),
then the local partitioned hash join.  Band (c4): R all-gathered over NCCL, local
NLJ against the rank's S shard.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

S_BITS_C4 = 24  # set from --c4-s-bits
C5_BITS = 28  # set from --c5-bits
C3_WEAK = False  # set from --c3-weak
C2_SPARSE = False  # set from --c2-sparse
C4_SKEW = False  # set from --c4-skew
METRIC = "join input & output tuples/s at 1/2/4/8 B200; % of HBM/INT roofline"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clock and clock-event reasons via NVML during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
            "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, v in names.items():
                    if r & v and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ workloads

def make_workload(name, device, rank=0, world=1):
    """Synthetic relations in HBM.  With world > 1 every rank holds a block shard
    of a problem `world` times larger (weak scaling); rid_base = global row offset."""
    import torch
    import gen
    import gen.device as gd
    seed = gen.BASE_SEED
    g = max(world.bit_length() - 1, 0)
    if name == "c2":
        n = 1 << 27  # per GPU
        if C2_SPARSE:  # R = 2^27 x N distinct keys drawn from a permutation of [0, 2^31)
            b = 31
            R = gd.perm_range(n, b, seed, offset=rank * n, device=device)
            S = gd.pkfk_S(n, b, seed, offset=rank * n, device=device, domain=n * world)
        else:  # R = a permutation of [0, 2^(27 + log2 N)) (dense keys)
            b = 27 + g
            R = gd.perm_range(n, b, seed, offset=rank * n, device=device)
            S = gd.pkfk_S(n, b, seed, offset=rank * n, device=device)
        desc = ("configs[1]: equi hash join 2^27 x 2^27 8-byte tuples (int32 key+payload, payload not read), "
                "PK-FK unique R keys" + (" drawn from [0, 2^31) (--c2-sparse)" if C2_SPARSE else ""))
        if world > 1:
            desc += f"; weak scaling: {world} ranks x (2^27 x 2^27) block shards, NCCL hash shuffle + local join"
        return dict(kind="equi", R=R, S=S, desc=desc, rid_base_R=rank * n, rid_base=rank * n, n_out_expected=n)
    if name == "c3":
        # configs[2]: R unique over 2^b ranks (perm_b), S = Zipf(1) FK draws over R's ranks
        # (reading R11).  Strong (default): the full 2^28 x 2^30 on every N
        # (rank r holds a 1/N block shard).  Weak (--c3-weak): 2^25 x 2^27 per GPU, so
        # N = 8 is configs[2]'s total (SURVEY reading 17).
        if C3_WEAK:
            nr, ns, b = 1 << 25, 1 << 27, 25 + g
        else:
            b = 28
            nr, ns = (1 << 28) // world, (1 << 30) // world
        R = gd.perm_range(nr, b, seed, offset=rank * nr, device=device)
        S = gd.zipf_S(ns, b, gd.zipf_table_device(1 << b, device=device), seed, offset=rank * ns, device=device)
        desc = (f"configs[2]: Zipf(s=1) skewed equi join, R unique over 2^{b} ranks, S Zipf FK; "
                + (f"weak: 2^25 x 2^27 per GPU x {world}" if C3_WEAK else
                   f"strong: 2^28 x 2^30 total over {world} GPU(s)"))
        return dict(kind="equi", R=R, S=S, desc=desc, rid_base_R=rank * nr, rid_base=rank * ns,
                    n_out_expected=ns)
    if name == "c1":
        R = gd.uniform(10_000, 10_000, seed, 0, device=device)
        S = gd.uniform(10_000, 10_000, seed, 1, device=device)
        return dict(kind="equi", R=R, S=S, desc="configs[0]: R=S=10^4 uniform keys in [0,10^4), equi hash join")
    if name == "c4":
        nr = (1 << 20) // world  # R (2^20) is block-sharded and replicated by the join
        ns = 1 << S_BITS_C4      # per GPU (2^24 = configs[3]; smaller only for ncu captures)
        if C4_SKEW:
            # skewed keys: cluster z ~ Zipf(1) over 4096 clusters (permuted ids) spaced
            # 2^18 apart in [0, 2^30), key = 2^18 z + uniform [0, 2^15); eps = 16 keeps
            # the output near 3.7e8 pairs.  The hot cluster (11% of each side) packs
            # ~235K S rows into one 4096-wide bucket: equal-width buckets (reading R15)
            # stop pruning there.
            zt = gd.zipf_table_device(1 << 12, device=device)
            R = gd.zipf_S(nr, 12, zt, seed, offset=rank * nr, device=device) * (1 << 18) + \
                gd.uniform(nr, 1 << 15, seed, 2, offset=rank * nr, device=device)
            S = gd.zipf_S(ns, 12, zt, seed + 1, offset=rank * ns, device=device) * (1 << 18) + \
                gd.uniform(ns, 1 << 15, seed, 3, offset=rank * ns, device=device)
            eps = 16
            desc = (f"configs[3] shape, skewed (--c4-skew): band join |R.a-S.b|<=16, 2^20 x 2^{S_BITS_C4} int32 "
                    "keys in Zipf(1)-weighted clusters (4096 clusters 2^18 apart, 2^15 wide), count+scan+write")
        else:
            R = gd.uniform(nr, 1 << 30, seed, 0, offset=rank * nr, device=device)
            S = gd.uniform(ns, 1 << 30, seed, 1, offset=rank * ns, device=device)
            eps = gen.C4_EPS
            desc = (f"configs[3]: band join |R.a-S.b|<=53687, 2^20 x 2^{S_BITS_C4} uniform int32 in [0,2^30), "
                    "count+scan+write; region matrix (PAPER.md §4.2 Alg.3) unless --opt theta_regions=0")
        if world > 1:
            desc += f"; weak scaling: R (2^20) all-gathered, {world} x 2^24 S shards"
        return dict(kind="band", R=R, S=S, eps=eps, desc=desc, rid_base_R=rank * nr, rid_base=rank * ns)
    if name == "c5":
        nr, ns = 1 << C5_BITS, 1 << (C5_BITS + 1)  # per GPU; 2^28 x 2^29 at N=8 = 2^31 x 2^32 = configs[4]
        b = C5_BITS + g
        R = gd.c5_R(nr, seed, offset=rank * nr, device=device, b=b)
        S = gd.c5_S(ns, seed, offset=rank * ns, device=device, b=b)
        desc = (f"configs[4] shape: pre-filtered (range + Bloom 8 bits/key, two-sided) equi join, int64 keys, "
                f"per GPU 2^{C5_BITS} x 2^{C5_BITS + 1} rows of a 2^{b}-row domain (N=8 with 2^28 per GPU = "
                f"2^31 x 2^32 = configs[4]); 10% of S are members")
        if world > 1:
            desc += "; distributed: range all-reduce, R shuffle, per-owner Bloom all-gather, filtered S shuffle"
        return dict(kind="pf_equi", R=R, S=S, desc=desc, rid_base_R=rank * nr, rid_base=rank * ns)
    raise SystemExit(f"unknown workload {name}")


def nvlink_peak(world):
    """Measured per-GPU NVLink egress of SM peer stores in an all-to-all with world-1
    peers (profiles/r02_nvlink.json, tools/mb_nvlink.cu), or (None, reason)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_nvlink.json")) as f:
            t = json.load(f)
        v = t.get(str(world - 1)) or t.get(str(max(int(k) for k in t if k.isdigit())))
        return float(v), "profiles/r02_nvlink.json (tools/mb_nvlink.cu, SM peer stores, all-to-all)"
    except Exception:
        return None, "not measured"


def ncu_traffic(workload, tag):
    """(dram bytes read+written per launch, source file) from the newest committed
    profiles/rNN_traffic.json that has this workload and kernel tag, else (None, None)."""
    import glob
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")), reverse=True):
        t = json.load(open(f)).get(workload, {}).get(tag)
        if t:
            return round(t["dram_bytes_per_launch"]), f"profiles/{os.path.basename(f)} ({t['report']})"
    return None, None


def join_bytes(nR, nS, nout, passes, wk, rid_implicit):
    """Algorithmic bytes of the partitioned hash join, per tag:
    (total bytes per step, launches per step).  wk = key bytes; rid_implicit = the
    first radix pass reads keys only (rids are row positions)."""
    n = nR + nS
    first = wk + (wk + 4) if rid_implicit else 2 * (wk + 4)
    scatter_total = n * first + (passes - 1) * n * 2 * (wk + 4)
    nb, npb = min(nR, nS), max(nR, nS)
    return {
        # multi-GPU shuffle pass: key (+ rid unless implicit) in, key + rid out (to the
        # owner's buffer, local HBM or a peer's over NVLink)
        "shuffle_scatter": (n * (wk + (wk + 4) if rid_implicit else 2 * (wk + 4)), 2),
        "part_hist": (wk * n * passes, 2 * passes),
        "part_scatter": (scatter_total, 2 * passes),
        # count: build + probe keys in, one uint16 match index per probe row out
        "hj_count": (wk * n + 2 * npb, 1),
        # write: build + probe rids and the staged index in, 8-byte pairs out
        "hj_write": (4 * nb + 4 * npb + 2 * npb + 8 * nout, 1),
    }


def algorithmic_bytes(w, info):
    """Algorithmic HBM bytes per launch of each kernel tag."""
    nR, nS = w["R"].numel(), w["S"].numel()
    nout = info["n_out"]
    if w["kind"] == "equi":
        ab = join_bytes(nR, nS, nout, info["passes"], w["R"].element_size(), info["world"] == 1)
        if info["world"] > 1:  # the shuffle reads the implicit-rid input; the local passes carry rids
            ab["shuffle_scatter"] = ((nR + nS) * (w["R"].element_size() + (w["R"].element_size() + 4)), 2)
            ab["part_scatter"] = ((nR + nS) * 2 * (w["R"].element_size() + 4) * info["passes"], 2 * info["passes"])
        return ab
    if w["kind"] == "pf_equi":
        # a probed row costs its 8 B key + one 32 B DRAM sector of the
        # filter (its 8-byte block; + 1 flag bit); the write pass reads the flags and
        # each survivor's key (8 B) and writes key + rid (12 B); then the hash join on
        # the survivors with 8-byte keys.  (N=1 row counts: R and S each compacted once.)
        kR, kS = w["kept"]
        pf = info["pf_launches"]
        ab = join_bytes(kR, kS, nout, info["passes"], 8, False)
        ab["pf_count"] = (40 * (nR + nS) + (nR + nS) // 8, pf)
        ab["pf_write"] = ((nR + nS) // 8 + 20 * (kR + kS), pf)
        # a filter insert reads its 8 B key once (multi-slice filters: after a slice
        # partition of the keys, counted with part_scatter) and updates one 32 B sector
        ab["bloom_build"] = (40 * (nR + kS), info["bloom_launches"])
        return ab
    # band: NLJ is ALU-bound; bytes are tiny
    return {"nlj_count": (4 * (nR + nS), 1), "nlj_write": (4 * (nR + nS) + 8 * nout, 1)}


def run_ours(args, world, rank, local):
    import torch
    import paper_1904_11201_b200 as gj

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    w = make_workload(args.workload, dev, rank, world)
    stream = torch.cuda.current_stream(dev)
    ctx = gj.Context(local, stream)
    for o in args.opt:
        k, v = o.split("=")
        ctx.set_option(k, int(v))
    nR, nS = w["R"].numel(), w["S"].numel()
    R = gj.Rel(w["R"], None, w.get("rid_base_R", w.get("rid_base", 0)))
    S = gj.Rel(w["S"], None, w.get("rid_base", 0))
    comm = gj.Comm(rank, world) if world > 1 else None

    if w["kind"] == "equi":
        if comm is None:
            n = n_global = gj.join_count(ctx, R, S)
        else:
            n, n_global = gj.join_dist_count(ctx, comm, R, S)
        out = torch.empty((max(int(n * 1.2) + 1024, 1), 2), dtype=torch.int32, device=dev)

        def step():
            if comm is None and not args.two_call_step:  # count -> scan -> write in one C-ABI call
                m = gj.join_count_materialize(ctx, R, S, out).shape[0]
            elif comm is None:
                m = gj.join_count(ctx, R, S)
                gj.join_materialize(ctx, R, S, m, out=out)
            else:
                m, _ = gj.join_dist_count(ctx, comm, R, S)
                gj.join_dist_materialize(ctx, comm, R, S, m, out=out)
            return m
    elif w["kind"] == "pf_equi":
        PF = gj.RANGE | gj.BLOOM | gj.TWO_SIDED

        def pf_step_count():
            if comm is None:  # one GPU: prefilter() survivors (with rid maps) -> join
                kR, rR, kS, rS = gj.prefilter(ctx, R, S, PF, "eq", 0, 8.0)
                R2, S2 = gj.Rel(kR, rR), gj.Rel(kS, rS)
                return gj.join_count(ctx, R2, S2), (R2, S2), (kR.numel(), kS.numel())
            m, _, kept = gj.join_dist_count_filtered(ctx, comm, R, S, PF, 8.0)
            return m, (R, S), kept

        n, _, kept0 = pf_step_count()
        n_global = n if comm is None else gj.join_dist_count_filtered(ctx, comm, R, S, PF, 8.0)[1]
        w["kept"] = kept0
        out = torch.empty((max(int(n * 1.2) + 1024, 1), 2), dtype=torch.int32, device=dev)

        def step():
            if comm is None and not args.two_call_step:
                kR, rR, kS, rS = gj.prefilter(ctx, R, S, PF, "eq", 0, 8.0)
                return gj.join_count_materialize(ctx, gj.Rel(kR, rR), gj.Rel(kS, rS), out).shape[0]
            m, (R2, S2), _ = pf_step_count()
            if comm is None:
                gj.join_materialize(ctx, R2, S2, m, out=out)
            else:
                gj.join_dist_materialize(ctx, comm, R2, S2, m, out=out)
            return m
    else:
        eps = w["eps"]
        if comm is None:
            n = n_global = gj.theta_join_count(ctx, R, S, "band", eps)
        else:
            n, n_global = gj.theta_join_dist_count(ctx, comm, R, S, "band", eps)
        out = torch.empty((max(n, 1), 2), dtype=torch.int32, device=dev)

        def step():
            if comm is None:
                m = gj.theta_join_count(ctx, R, S, "band", eps)
                gj.theta_join_materialize(ctx, R, S, "band", eps, m, out=out)
            else:
                m, _ = gj.theta_join_dist_count(ctx, comm, R, S, "band", eps)
                gj.theta_join_dist_materialize(ctx, comm, R, S, "band", eps, m, out=out)
            return m

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, device time by CUDA events on the ctx stream
    sampler = ClockSampler(local)
    ctx.reset_stats()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        e0.record(stream)
        for _ in range(args.steps):
            m = step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms = e0.elapsed_time(e1)
    launches = ctx.launches()
    assert m == n
    ms_max = max_over_ranks(ms, world)

    # receive balance of the hash shuffle (N > 1) and the hash-join unit plan: the
    # tuples every rank's local join processed, max / mean over ranks
    recv = None
    if w["kind"] in ("equi", "pf_equi"):
        lr, ls = ctx.join_local_sizes()
        _, pbits, units = ctx.join_stats()
        recv = {"local_R": lr, "local_S": ls, "partitions": 1 << pbits, "units": units}
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([lr, ls], dtype=torch.float64, device=dev)
            allt = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(allt, t)
            a = torch.stack(allt).cpu()
            recv["recv_R_per_rank"] = [int(x) for x in a[:, 0]]
            recv["recv_S_per_rank"] = [int(x) for x in a[:, 1]]
            recv["imbalance_R"] = round(float(a[:, 0].max() / a[:, 0].mean()), 4)
            recv["imbalance_S"] = round(float(a[:, 1].max() / a[:, 1].mean()), 4)
    # ---- profiled pass (per-kernel CUDA events on the ctx stream)
    ctx.set_option("profile", 1)
    ctx.reset_stats()
    for _ in range(args.steps):
        step()
    ktimes = ctx.kernel_times()
    # 1 GPU: S's radix passes overlap R's on a second stream (GJ_OPT_OVERLAP_PARTITIONS),
    # which stretches each kernel's event-timed duration; a second profiled pass with
    # the relations one after the other gives the kernels' standalone times
    ktimes_serial = None
    if world == 1 and w["kind"] in ("equi", "pf_equi"):
        ctx.set_option("overlap_partitions", 0)
        ctx.reset_stats()
        for _ in range(args.steps):
            step()
        ktimes_serial = ctx.kernel_times()
        ctx.set_option("overlap_partitions", 1)
    ctx.set_option("profile", 0)

    info = {"n_out": n, "world": world}
    # local radix passes per relation actually run (the multi-GPU shuffle is "shuffle_scatter")
    info["passes"] = max(1, round(ktimes.get("part_scatter", (0, 0))[1] / args.steps / 2))
    info["pf_launches"] = max(1, round(ktimes.get("pf_count", (0, 0))[1] / args.steps))
    info["bloom_launches"] = max(1, round(ktimes.get("bloom_build", (0, 0))[1] / args.steps))
    ab = algorithmic_bytes(w, info)
    hbm, peak_src = peaks()
    per_kernel = {}
    for tag, (tms, cnt) in ktimes.items():
        rec = {"ms_per_launch": tms / cnt, "launches_per_step": cnt / args.steps,
               "share": tms / sum(v[0] for v in ktimes.values())}
        if tag in ab:
            total_bytes, per_step = ab[tag]
            per_launch = total_bytes / per_step
            rec["alg_bytes_per_launch"] = per_launch
            rec["achieved_gbs"] = per_launch / (tms / cnt * 1e-3) / 1e9
        per_kernel[tag] = rec
    dom = max(ktimes.items(), key=lambda kv: kv[1][0])[0]
    # measured DRAM bytes per launch of the dominant kernel: committed ncu --set full
    # capture of the same single-GPU workload (profiles/rNN_traffic.json)
    traffic, tsrc = ncu_traffic(args.workload, dom) if world == 1 else (None, None)
    if w["kind"] in ("equi", "pf_equi"):
        d = per_kernel[dom]
        roof = {"kernel": dom, "bound": "hbm", "achieved": round(d.get("achieved_gbs", 0.0), 1), "peak": hbm,
                "unit": "GB/s", "frac": round(d.get("achieved_gbs", 0.0) / hbm, 4), "traffic": traffic,
                "alg_bytes_per_launch": d.get("alg_bytes_per_launch"), "traffic_source": tsrc,
                "peak_source": peak_src}
        if ktimes_serial and dom in ktimes_serial and d.get("alg_bytes_per_launch"):
            tms, cnt = ktimes_serial[dom]
            a_s = d["alg_bytes_per_launch"] / (tms / cnt * 1e-3) / 1e9
            roof["standalone"] = {
                "achieved": round(a_s, 1), "frac": round(a_s / hbm, 4), "ms_per_launch": round(tms / cnt, 4),
                "note": "same kernel timed with R and S partitioned one after the other (no concurrent "
                        "kernel sharing the GPU); frac above is measured in the timed configuration, where "
                        "S's passes overlap R's on a second stream"}
        if "shuffle_scatter" in per_kernel:
            # the NVLink shuffle: (G-1)/G of every shuffled tuple (key + rid) crosses
            # NVLink as SM peer stores; vs the measured peer-store egress of
            # tools/mb_nvlink.cu (profiles/r02_nvlink.json)
            k = per_kernel["shuffle_scatter"]
            tup = (nR + nS) / 2  # per launch (one relation per launch; R and S are equal-sized here)
            wire = tup * (world - 1) / world * (w["R"].element_size() + 4)
            pk, psrc = nvlink_peak(world)
            nv = {"kernel": "shuffle_scatter", "bound": "nvlink", "achieved": round(
                wire / (k["ms_per_launch"] * 1e-3) / 1e9, 1), "peak": pk, "unit": "GB/s",
                "frac": round(wire / (k["ms_per_launch"] * 1e-3) / 1e9 / pk, 4) if pk else None,
                "traffic": None, "alg_bytes_per_launch": wire, "peak_source": psrc}
            if dom == "shuffle_scatter":  # the dominant kernel is NVLink-bound: that is its roofline
                roof = nv | {"hbm_view": roof}
            else:
                roof["nvlink"] = nv
    else:
        # The NLJ compares the pairs of the cells the region matrix keeps (all n_R x n_S
        # with theta_regions=0): INT ALU roofline, 1.5 ALU-pipe instr per pair-compare
        # (band: + 1 FMA-pipe IMAD), DESIGN.md §5.  The write pass also stores 8 B per
        # pair: its bound is whichever of the two floors is higher (the band's write
        # pass, mostly Green cross products, is HBM-bound).
        pairs, cross = ctx.theta_stats()
        d = per_kernel[dom]
        sm = sampler.summary().get("sm_mhz") or 1965
        alu_peak = 148 * 64 * sm * 1e6 / 1.5 / 1e12  # T pair-compares/s the ALU pipe allows
        t = d["ms_per_launch"] * 1e-3
        t_alu = pairs / (alu_peak * 1e12)
        t_hbm = (8 * info["n_out"] / (hbm * 1e9)) if dom in ("nlj_write", "band_write", "cross_rect") else 0.0
        if t_hbm > t_alu:
            ach = 8 * info["n_out"] / t / 1e9
            roof = {"kernel": dom, "bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(ach / hbm, 4), "traffic": traffic, "alg_bytes_per_launch": 8 * info["n_out"],
                    "traffic_source": tsrc, "peak_source": peak_src}
        else:
            ach = pairs / t / 1e12
            roof = {"kernel": dom, "bound": "alu", "achieved": round(ach, 3), "peak": round(alu_peak, 3),
                    "unit": "Tpair/s", "frac": round(ach / alu_peak, 4), "traffic": traffic,
                    "alg_bytes_per_launch": d.get("alg_bytes_per_launch"), "traffic_source": tsrc,
                    "peak_source": "148 SM x 64 ALU-pipe instr/clk (measured 62.7-63.5 by tools/mb_ops.cu, profiles/r02_mb_ops.txt) x median SM clock / 1.5 ALU instr per pair"}
        roof["nlj_pairs_per_launch"] = pairs
        roof["cross_pairs"] = cross
        roof["pairs_all"] = nR * world * nS

    # ---- e2e: host buffers in, host pairs out, through the public API
    e2e = None
    if w["kind"] in ("equi", "pf_equi"):
        hR = w["R"].cpu().pin_memory()
        hS = w["S"].cpu().pin_memory()
        hout = torch.empty((max(n, 1), 2), dtype=torch.int32).pin_memory()
        k_e2e = max(1, min(args.steps, args.e2e_steps))
        batch_api = False
        if w["kind"] == "pf_equi":
            dR, dS = torch.empty_like(w["R"]), torch.empty_like(w["S"])
            eR, eS = gj.Rel(dR, None, R.rid_base), gj.Rel(dS, None, S.rid_base)

            def e2e_step():
                dR.copy_(hR, non_blocking=True)
                dS.copy_(hS, non_blocking=True)
                if comm is None:
                    kR, rR, kS, rS = gj.prefilter(ctx, eR, eS, PF, "eq", 0, 8.0)
                    R2, S2 = gj.Rel(kR, rR), gj.Rel(kS, rS)
                    m = gj.join_count(ctx, R2, S2)
                    res = gj.join_materialize(ctx, R2, S2, m, out=out)
                else:
                    m, _, _ = gj.join_dist_count_filtered(ctx, comm, eR, eS, PF, 8.0)
                    res = gj.join_dist_materialize(ctx, comm, eR, eS, m, out=out)
                hout[:m].copy_(res)
                return m
            note = ("per rank: pinned H2D of its shards -> prefilter + join (count/scan/write) through the public "
                    "API -> D2H of its pairs")
        elif comm is None:
            hout2 = torch.empty_like(hout).pin_memory()
            batch_api = True

            def e2e_run(k):  # one C-ABI call streams k joins; host outputs alternate
                ns = gj.join_host_batch(ctx, [(hR, hS, hout if b % 2 == 0 else hout2) for b in range(k)])
                return ns[-1]
            note = ("join_host_batch(): k independent joins from pinned host keys in one C-ABI call -- per join "
                    "H2D -> count/scan/write -> D2H of all pairs; consecutive joins overlap their PCIe transfers "
                    "on two streams")
        else:
            dR, dS = torch.empty_like(w["R"]), torch.empty_like(w["S"])
            eR, eS = gj.Rel(dR, None, R.rid_base), gj.Rel(dS, None, S.rid_base)

            def e2e_step():
                dR.copy_(hR, non_blocking=True)
                dS.copy_(hS, non_blocking=True)
                m, _ = gj.join_dist_count(ctx, comm, eR, eS)
                res = gj.join_dist_materialize(ctx, comm, eR, eS, m, out=out)
                hout[:m].copy_(res)
                return m
            note = "per rank: pinned H2D of its shards -> join_dist_count/materialize (hash shuffle over NVLink peer stores) -> D2H of its pairs"
        if not batch_api:
            e2e_step()
        else:
            e2e_run(2)
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        if batch_api:
            got = e2e_run(k_e2e)
        else:
            for _ in range(k_e2e):
                got = e2e_step()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        assert got == n
        e2e_s = max_over_ranks(t1 - t0, world)
        e2e = {"value": (nR + nS) * k_e2e * world / e2e_s, "unit": "input tuples/s",
               "h2d_bytes_per_step": hR.numel() * hR.element_size() + hS.numel() * hS.element_size(),
               "d2h_bytes_per_step": n * 8, "steps": k_e2e, "note": note + "; wall clock, max over ranks"}
    if comm is not None:
        comm.close()

    return dict(ms=ms_max, n=n_global, nR=nR, nS=nS, launches=launches, roof=roof, per_kernel=per_kernel, e2e=e2e,
                clocks=sampler.summary(), desc=w["desc"], kind=w["kind"], kept=w.get("kept"),
                dtype="i64" if w["R"].dtype == torch.int64 else "i32", recv=recv)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(args, single=True):
    """The oracle timed on this host's cores on a bounded sample of the workload.
    Equi workloads: O7 (O2 sliced by key hash over all host threads) is the value;
    O2 on one thread is reported beside it (single=True).  Band (c4): O3 on 1 thread."""
    import numpy as np  # noqa: F401
    import gen
    import oracle
    T = os.cpu_count() or 1
    if args.workload == "c4":
        R, S = gen.c4(nR=1 << 11, nS=1 << 24)
        t0 = time.perf_counter()
        c = oracle.theta_count_sorted(R, S, "band", gen.C4_EPS)  # noqa: F841
        dt = time.perf_counter() - t0
        return {"value": (len(R) + len(S)) / dt, "unit": "input tuples/s", "cores": 1, "kind": "oracle",
                "sample": "O3 sort+binary-search band count, R 2^11 x S 2^24 slice of configs[3]", "seconds": dt,
                "cpu": cpu_model()}
    b = args.cpu_sample_bits
    if args.workload == "c5":
        b -= 2
        R, S, m = gen.c5(1 << b, 1 << (b + 1), b=b)
        expect = int((m >= 0).sum())
        what = f"configs[4] shape int64 2^{b} x 2^{b + 1} over a 2^{b}-row domain (exact join, no pre-filter)"
    elif args.workload == "c3":
        b -= 2
        R, S, m = gen.zipf_pkfk(b, 1 << (b + 2), gen.zipf_table(1 << b))
        expect = len(S)
        what = f"configs[2] shape: R 2^{b} unique, S 2^{b + 2} Zipf(1) FK"
    else:
        R, S, m = gen.pkfk(b, 1 << b)
        expect = len(S)
        what = f"PK-FK 2^{b} x 2^{b} (configs[1] shape, scaled)"
    t0 = time.perf_counter()
    c, _ = oracle.hash_equi_sliced(R, S, T)
    dt = time.perf_counter() - t0
    assert c == expect
    out = {"value": (len(R) + len(S)) / dt, "unit": "input tuples/s", "cores": T, "kind": "oracle",
           "sample": f"O7 = O2 (std::unordered_multimap build/probe + sort) sliced by key hash over {T} host "
                     f"threads, {what}", "seconds": round(dt, 3), "cpu": cpu_model()}
    if single:
        t0 = time.perf_counter()
        c1, _ = oracle.hash_equi(R, S)
        d1 = time.perf_counter() - t0
        assert c1 == expect
        out["single_thread"] = {"value": (len(R) + len(S)) / d1, "cores": 1, "kind": "oracle O2",
                                "seconds": round(d1, 3)}
    return out


def main():
    # Exactly one JSON line goes to stdout: C-level chatter (e.g. NCCL's version
    # banner) is redirected to stderr and the JSON is written to the saved fd.
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    global print
    _print = print

    def print(*a, **k):  # noqa: A001 - route this module's JSON line to the real stdout
        with os.fdopen(os.dup(json_fd), "w") as f:
            _print(*a, **k, file=f)

    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--c3-weak", action="store_true", help="c3: 2^25 x 2^27 per GPU (weak) instead of 2^28 x 2^30 total")
    ap.add_argument("--c4-skew", action="store_true", help="c4: Zipf-clustered keys, eps = 16 (a perf point)")
    ap.add_argument("--c2-sparse", action="store_true",
                    help="c2: R keys drawn from a permutation of [0, 2^31) instead of [0, 2^(27+log2 N))")
    ap.add_argument("--two-call-step", action="store_true",
                    help="1-GPU equi step as join_count + join_materialize (two C-ABI calls) instead of "
                         "join_count_materialize (A/B of the host round trip between count and write)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-sample-bits", type=int, default=23)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--c4-s-bits", type=int, default=24, help="log2 |S| per GPU for c4 (24 = configs[3]; ncu only)")
    ap.add_argument("--c5-bits", type=int, default=28, help="log2 |R| per GPU for c5 (|S| = 2|R|; 28 at N=8 = configs[4])")
    ap.add_argument("--opt", action="append", default=[], help="ctx option name=value (tuning sweeps)")
    args = ap.parse_args()
    global S_BITS_C4, C5_BITS, C3_WEAK, C2_SPARSE, C4_SKEW
    S_BITS_C4 = args.c4_s_bits
    C5_BITS = args.c5_bits
    C3_WEAK = args.c3_weak
    C2_SPARSE = args.c2_sparse
    C4_SKEW = args.c4_skew
    world, rank, local = dist_setup(args)

    if args.impl == "reference":
        if rank != 0:
            return
        res = []
        # Warm-up is untimed; one bounded oracle step warms the page cache and
        # the host allocator, further ones would only lengthen the run.
        for _ in range(min(max(args.warmup, 0), 1)):
            cpu_baseline(args, single=False)
        for _ in range(args.steps):
            res.append(cpu_baseline(args, single=False))
        v = statistics.median(r["value"] for r in res)
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "input tuples/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * statistics.median(float(r["seconds"]) for r in res),
                "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "i64" if args.workload == "c5" else "i32", "data": "synthetic",
                "config": {"workload": res[0]["sample"]},
                "cpu_baseline": {k: res[0][k] for k in ("kind", "cores", "sample", "cpu")} | {"value": v,
                                                                                       "unit": "input tuples/s"},
                "e2e": {"value": v, "unit": "input tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    r = run_ours(args, world, rank, local)
    if rank != 0:
        return
    T = r["ms"] * 1e-3
    value = (r["nR"] + r["nS"]) * args.steps * world / T
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "input tuples/s",
        "output_tuples_per_s": r["n"] * args.steps / T,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": r["ms"] / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": r["dtype"],
        "data": "synthetic",
        "config": {"workload": r["desc"], "n_R_per_gpu": r["nR"], "n_S_per_gpu": r["nS"], "n_out": r["n"],
                   "l2": "inputs (>=64 MiB of keys, 1 GiB for configs[1]) exceed/stream past the 126 MB L2; no flush",
                   "parallelism": ("1 GPU" if world == 1 else
                                   f"{world} ranks, hash shuffle over NVLink peer stores (equi) / "
                                   "R all-gather (theta)")} | ({"kept_R_S_rank0": list(r["kept"])} if r.get("kept") else {})
                  | ({"options": args.opt} if args.opt else {}),
        "roofline": r["roof"],
        "kernels": r["per_kernel"],
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
        "e2e": r["e2e"],
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(args)
    print(json.dumps(line))


if __name__ == "__main__":
    main()
