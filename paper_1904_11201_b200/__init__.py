"""paper_1904_11201_b200 -- B200-native GPU join hot path of arXiv 1904.11201.

Thin ctypes binding over ``libgjoin.so`` (C ABI declared in ``include/gjoin.h``).
This module only marshals arguments: every step of the join (partitioning, hash
build/probe, nested-loop theta compare, scans, pre-filter, materialisation) runs
in the library's CUDA kernels.  torch supplies device memory, streams and process
groups.  There is NO CPU fallback: importing fails loudly if the library is
missing, and every call needs CUDA tensors.

Names follow the C ABI:

    ctx = Context(device=0)                       # gj_ctx_create
    n   = join_count(ctx, R, S)                   # |J(R, S, =)|
    out = join_materialize(ctx, R, S, n)          # (n, 2) int32 view of uint32 (rid_R, rid_S)
    n   = theta_join_count(ctx, R, S, "band", eps)
    out = theta_join_materialize(ctx, R, S, "band", eps, n)
    (Rk, Rr, Sk, Sr) = prefilter(ctx, R, S, flags=RANGE|BLOOM|TWO_SIDED)
    n   = join_host(ctx, keyR_host, keyS_host, out_host)   # host buffers, e2e

``R``/``S`` are :class:`Rel` (key tensor, optional rid tensor, rid_base) or bare key
tensors (rid = row position).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgjoin.so")

OPS = {"eq": 0, "ne": 1, "lt": 2, "le": 3, "gt": 4, "ge": 5, "band": 6}
RANGE, BLOOM, TWO_SIDED, EXACT = 1, 2, 4, 8
OPT = {"part_bits": 1, "build_chunk": 2, "probe_chunk": 3, "profile": 4, "nlj_split": 5,
       "force_slow_band": 6, "build_side": 7, "shuffle_bits": 8, "theta_regions": 9,
       "theta_grid_rows": 10, "shuffle_ctas": 11, "check_args": 12,
       "overlap_partitions": 13, "fib_slots": 14}
STATUS = {0: "GJ_OK", 1: "GJ_EINVAL", 2: "GJ_ENOMEM", 3: "GJ_ERANGE", 4: "GJ_ESTATE", 5: "GJ_ECUDA",
          6: "GJ_ENCCL"}
I32, I64 = 0, 1


class GJError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Rel(ctypes.Structure):
    _fields_ = [("key", ctypes.c_void_p), ("rid", ctypes.c_void_p), ("n", ctypes.c_uint64),
                ("key_type", ctypes.c_int32), ("rid_base", ctypes.c_uint32)]


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a); "
                          "there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    vp, u64, i32, u32, i64 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32, ctypes.c_int64
    pu64 = ctypes.POINTER(ctypes.c_uint64)
    L.gj_ctx_create.argtypes = [ctypes.POINTER(vp), i32, vp]
    L.gj_ctx_destroy.argtypes = [vp]
    L.gj_ctx_destroy.restype = None
    L.gj_ctx_set_stream.argtypes = [vp, vp]
    L.gj_ctx_set_allocator.argtypes = [vp, ALLOC_FN, FREE_FN, vp]
    L.gj_ctx_set_option.argtypes = [vp, i32, i64]
    L.gj_last_error.restype = ctypes.c_char_p
    L.gj_theta_stats.argtypes = [vp, ctypes.POINTER(u64), ctypes.POINTER(u64)]
    L.gj_theta_stats.restype = i32
    L.gj_join_stats.argtypes = [vp, ctypes.POINTER(u64), ctypes.POINTER(u32), ctypes.POINTER(u32)]
    L.gj_join_stats.restype = i32
    L.gj_join_local_sizes.argtypes = [vp, ctypes.POINTER(u64), ctypes.POINTER(u64)]
    L.gj_join_local_sizes.restype = i32
    L.gj_gather_payloads.argtypes = [vp, vp, u64, vp, u32, u32, vp, u32, u32, vp, vp]
    L.gj_gather_payloads.restype = i32
    L.gj_ctx_launch_count.argtypes = [vp]
    L.gj_ctx_launch_count.restype = u64
    L.gj_ctx_reset_stats.argtypes = [vp]
    L.gj_ctx_reset_stats.restype = None
    L.gj_ctx_kernel_times.argtypes = [vp, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_double),
                                      pu64, i32]
    L.gj_ctx_kernel_times.restype = i32
    L.join_count.argtypes = [vp, _Rel, _Rel, pu64]
    L.join_materialize.argtypes = [vp, _Rel, _Rel, vp, u64, pu64]
    L.join_count_materialize.argtypes = [vp, _Rel, _Rel, vp, u64, pu64]
    L.theta_join_count.argtypes = [vp, _Rel, _Rel, i32, u64, pu64]
    L.theta_join_materialize.argtypes = [vp, _Rel, _Rel, i32, u64, vp, u64, pu64]
    L.prefilter.argtypes = [vp, _Rel, _Rel, u32, i32, u64, ctypes.c_double, vp, vp, pu64, vp, vp, pu64]
    L.join_host.argtypes = [vp, vp, u64, vp, u64, i32, vp, u64, pu64]
    L.join_host_batch.argtypes = [vp, i32, vp, vp, vp, vp, i32, vp, vp, pu64]
    L.gj_comm_unique_id.argtypes = [vp]
    L.gj_comm_init.argtypes = [ctypes.POINTER(vp), vp, i32, i32]
    L.gj_comm_destroy.argtypes = [vp]
    L.gj_comm_destroy.restype = None
    L.join_dist_count.argtypes = [vp, vp, _Rel, _Rel, pu64, pu64]
    L.join_dist_count_filtered.argtypes = [vp, vp, _Rel, _Rel, u32, ctypes.c_double, pu64, pu64, pu64]
    L.join_dist_materialize.argtypes = [vp, vp, _Rel, _Rel, vp, u64, pu64]
    L.prefilter_dist.argtypes = [vp, vp, _Rel, _Rel, u32, i32, u64, ctypes.c_double, vp, vp, pu64, vp, vp, pu64]
    L.theta_join_dist_count.argtypes = [vp, vp, _Rel, _Rel, i32, u64, pu64, pu64]
    L.theta_join_dist_materialize.argtypes = [vp, vp, _Rel, _Rel, i32, u64, vp, u64, pu64]
    L.gj_region_classify.argtypes = [i32, u32, u64, ctypes.c_int64, vp]
    L.gj_region_classify.restype = i32
    L.gj_dist_plan.argtypes = [pu64, i32, i32, i32, ctypes.POINTER(u32), ctypes.POINTER(u32), pu64]
    for f in ("gj_ctx_create", "gj_ctx_set_stream", "gj_ctx_set_allocator", "gj_ctx_set_option", "join_count", "join_materialize",
              "join_count_materialize", "theta_join_count", "theta_join_materialize", "prefilter", "join_host", "join_host_batch",
              "gj_comm_unique_id",
              "gj_comm_init", "join_dist_count", "join_dist_count_filtered", "join_dist_materialize", "prefilter_dist",
              "theta_join_dist_count", "theta_join_dist_materialize", "gj_dist_plan"):
        getattr(L, f).restype = i32
    return L


lib = _load()

# C-ABI symbols declared in include/gjoin.h (checked by tests/test_abi.py)
ABI_SYMBOLS = ("gj_ctx_create", "gj_ctx_destroy", "gj_ctx_set_stream", "gj_ctx_set_allocator", "gj_last_error", "gj_ctx_set_option",
               "gj_ctx_launch_count", "gj_ctx_reset_stats", "gj_ctx_kernel_times", "gj_theta_stats", "gj_join_stats",
               "gj_join_local_sizes", "gj_gather_payloads", "join_count",
               "join_materialize", "join_count_materialize", "theta_join_count", "theta_join_materialize",
               "prefilter", "join_host", "join_host_batch",
               "gj_comm_unique_id", "gj_comm_init", "gj_comm_destroy", "join_dist_count", "join_dist_count_filtered",
               "join_dist_materialize", "prefilter_dist", "theta_join_dist_count", "theta_join_dist_materialize",
               "gj_dist_plan",
               "gj_region_classify")
COMM_ID_BYTES = 128


def _check(status: int):
    if status != 0:
        raise GJError(status, lib.gj_last_error().decode(errors="replace"))


@dataclass
class Rel:
    """One relation's key column (+ optional rid map) on the GPU."""
    key: torch.Tensor
    rid: Optional[torch.Tensor] = None
    rid_base: int = 0

    def c(self) -> _Rel:
        k = self.key
        if not k.is_cuda:
            raise ValueError("Rel.key must be a CUDA tensor (no CPU fallback)")
        if k.dtype not in (torch.int32, torch.int64) or not k.is_contiguous():
            raise ValueError("Rel.key must be a contiguous int32/int64 CUDA tensor")
        rid = None
        if self.rid is not None:
            if not self.rid.is_cuda or self.rid.dtype not in (torch.int32, torch.uint32) or \
                    not self.rid.is_contiguous() or self.rid.numel() != k.numel():
                raise ValueError("Rel.rid must be a contiguous 32-bit CUDA tensor of key's length")
            rid = self.rid.data_ptr()
        return _Rel(k.data_ptr() if k.numel() else None, rid, k.numel(),
                    I32 if k.dtype == torch.int32 else I64, self.rid_base)


def _rel(x) -> _Rel:
    return x.c() if isinstance(x, Rel) else Rel(x).c()


class Context:
    """gj_ctx bound to a device and (by default) torch's current stream there.

    torch_allocator=True backs the library's scratch workspace with torch's caching
    allocator (gj_ctx_set_allocator): the join's partition buffers then show up in,
    and are recycled by, torch.cuda's memory pool."""

    def __init__(self, device: int = 0, stream: Optional[torch.cuda.Stream] = None, torch_allocator: bool = False,
                 **options):
        torch.cuda.set_device(device)
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = ctypes.c_void_p()
        _check(lib.gj_ctx_create(ctypes.byref(h), device, ctypes.c_void_p(self.stream.cuda_stream)))
        self.h = h
        self._alloc_cbs = None
        if torch_allocator:
            self.use_torch_allocator()
        for k, v in options.items():
            self.set_option(k, v)

    def use_torch_allocator(self):
        dev = self.device

        def _alloc(nbytes, stream, _user):
            try:
                return torch.cuda.caching_allocator_alloc(int(nbytes), dev, int(stream or 0))
            except Exception:
                return None

        def _free(ptr, _nbytes, _stream, _user):
            torch.cuda.caching_allocator_delete(int(ptr))

        self._alloc_cbs = (ALLOC_FN(_alloc), FREE_FN(_free))  # keep the callbacks alive
        _check(lib.gj_ctx_set_allocator(self.h, self._alloc_cbs[0], self._alloc_cbs[1], None))

    def set_option(self, name: str, value: int):
        _check(lib.gj_ctx_set_option(self.h, OPT[name], int(value)))

    def set_stream(self, stream: torch.cuda.Stream):
        self.stream = stream
        _check(lib.gj_ctx_set_stream(self.h, ctypes.c_void_p(stream.cuda_stream)))

    def launches(self) -> int:
        return int(lib.gj_ctx_launch_count(self.h))

    def reset_stats(self):
        lib.gj_ctx_reset_stats(self.h)

    def join_stats(self) -> tuple:
        """(Eq.8 result-size bound, partition bits B, hash-join units) of the last equi count."""
        e, b, u = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_uint32()
        _check(lib.gj_join_stats(self.h, ctypes.byref(e), ctypes.byref(b), ctypes.byref(u)))
        return int(e.value), int(b.value), int(u.value)

    def join_local_sizes(self) -> tuple:
        """(n_R, n_S) the last equi count's local join processed (received shards at N > 1)."""
        a, b = ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib.gj_join_local_sizes(self.h, ctypes.byref(a), ctypes.byref(b)))
        return int(a.value), int(b.value)

    def theta_stats(self) -> tuple:
        """(pairs the NLJ compared, pairs written as Green cross products) of the last theta count."""
        a, b = ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib.gj_theta_stats(self.h, ctypes.byref(a), ctypes.byref(b)))
        return int(a.value), int(b.value)

    def kernel_times(self) -> dict:
        """{tag: (total_ms, launches)} of kernels since the last reset (needs profile=1)."""
        n = 64
        names = (ctypes.c_char_p * n)()
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_uint64 * n)()
        k = lib.gj_ctx_kernel_times(self.h, names, ms, cnt, n)
        if k < 0:
            raise GJError(5, lib.gj_last_error().decode())
        return {names[i].decode(): (ms[i], int(cnt[i])) for i in range(min(k, n))}

    def close(self):
        if getattr(self, "h", None):
            lib.gj_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def join_count(ctx: Context, R, S) -> int:
    n = ctypes.c_uint64()
    _check(lib.join_count(ctx.h, _rel(R), _rel(S), ctypes.byref(n)))
    return n.value


def _out(n: int, out: Optional[torch.Tensor], device) -> torch.Tensor:
    if out is None:
        return torch.empty((max(n, 1), 2), dtype=torch.int32, device=device)
    if not out.is_cuda or out.dtype not in (torch.int32, torch.uint32) or not out.is_contiguous():
        raise ValueError("out must be a contiguous 32-bit CUDA tensor of shape (capacity, 2)")
    return out


def join_materialize(ctx: Context, R, S, n: Optional[int] = None, out: Optional[torch.Tensor] = None):
    """Writes |J| (rid_R, rid_S) pairs; returns the (|J|, 2) int32 view (uint32 values)."""
    if n is None and out is None:
        n = join_count(ctx, R, S)
    key = (R.key if isinstance(R, Rel) else R)
    buf = _out(n or 0, out, key.device)
    w = ctypes.c_uint64()
    _check(lib.join_materialize(ctx.h, _rel(R), _rel(S), ctypes.c_void_p(buf.data_ptr()), buf.shape[0],
                                ctypes.byref(w)))
    return buf[: w.value]


def join_count_materialize(ctx: Context, R, S, out: torch.Tensor):
    """Count and write in one C-ABI call (the write launched right after the count's
    host read-back); out = a (capacity, 2) 32-bit CUDA tensor.  Returns the (|J|, 2)
    view; raises GJ_ERANGE if capacity < |J|."""
    buf = _out(0, out, None)
    w = ctypes.c_uint64()
    _check(lib.join_count_materialize(ctx.h, _rel(R), _rel(S), ctypes.c_void_p(buf.data_ptr()), buf.shape[0],
                                      ctypes.byref(w)))
    return buf[: w.value]


def theta_join_count(ctx: Context, R, S, op: str, eps: int = 0) -> int:
    n = ctypes.c_uint64()
    _check(lib.theta_join_count(ctx.h, _rel(R), _rel(S), OPS[op], int(eps), ctypes.byref(n)))
    return n.value


def theta_join_materialize(ctx: Context, R, S, op: str, eps: int = 0, n: Optional[int] = None,
                           out: Optional[torch.Tensor] = None):
    if n is None and out is None:
        n = theta_join_count(ctx, R, S, op, eps)
    key = (R.key if isinstance(R, Rel) else R)
    buf = _out(n or 0, out, key.device)
    w = ctypes.c_uint64()
    _check(lib.theta_join_materialize(ctx.h, _rel(R), _rel(S), OPS[op], int(eps),
                                      ctypes.c_void_p(buf.data_ptr()), buf.shape[0], ctypes.byref(w)))
    return buf[: w.value]


def prefilter(ctx: Context, R, S, flags: int = RANGE | BLOOM | TWO_SIDED, op: str = "eq", eps: int = 0,
              bloom_bits_per_key: float = 8.0):
    """Returns (R_keys, R_rids, S_keys, S_rids) of the surviving tuples (CUDA tensors)."""
    rR, rS = _rel(R), _rel(S)
    kR = (R.key if isinstance(R, Rel) else R)
    kS = (S.key if isinstance(S, Rel) else S)
    okR, orR = torch.empty_like(kR), torch.empty(kR.numel(), dtype=torch.int32, device=kR.device)
    okS, orS = torch.empty_like(kS), torch.empty(kS.numel(), dtype=torch.int32, device=kS.device)
    nR, nS = ctypes.c_uint64(), ctypes.c_uint64()
    _check(lib.prefilter(ctx.h, rR, rS, flags, OPS[op], int(eps), float(bloom_bits_per_key),
                         ctypes.c_void_p(okR.data_ptr()), ctypes.c_void_p(orR.data_ptr()), ctypes.byref(nR),
                         ctypes.c_void_p(okS.data_ptr()), ctypes.c_void_p(orS.data_ptr()), ctypes.byref(nS)))
    return okR[: nR.value], orR[: nR.value], okS[: nS.value], orS[: nS.value]


def gather_payloads(ctx: Context, pairs: torch.Tensor, payload_R: Optional[torch.Tensor] = None,
                    payload_S: Optional[torch.Tensor] = None, rid_base_R: int = 0, rid_base_S: int = 0):
    """Late materialisation: rows pairs[:, 0] - rid_base_R of payload_R and
    pairs[:, 1] - rid_base_S of payload_S (CUDA tensors, rows along dim 0, row bytes a
    multiple of 4).  Returns (out_R, out_S) (None for a side not given)."""
    n = pairs.shape[0]
    outs = []
    args = []
    for pay in (payload_R, payload_S):
        if pay is None:
            outs.append(None)
            args += [None, 0]
            continue
        if not pay.is_cuda or not pay.is_contiguous():
            raise ValueError("payloads must be contiguous CUDA tensors")
        row = pay[0].numel() * pay.element_size() if pay.dim() > 1 else pay.element_size()
        o = torch.empty((n,) + tuple(pay.shape[1:]), dtype=pay.dtype, device=pay.device)
        outs.append(o)
        args += [ctypes.c_void_p(pay.data_ptr()), row]
    _check(lib.gj_gather_payloads(ctx.h, ctypes.c_void_p(pairs.data_ptr()), n, args[0], args[1], rid_base_R,
                                  args[2], args[3], rid_base_S,
                                  ctypes.c_void_p(outs[0].data_ptr()) if outs[0] is not None else None,
                                  ctypes.c_void_p(outs[1].data_ptr()) if outs[1] is not None else None))
    return outs[0], outs[1]


def join_host(ctx: Context, key_R: torch.Tensor, key_S: torch.Tensor, out: torch.Tensor) -> int:
    """End-to-end equi join from HOST tensors (pin them for full PCIe speed).

    out: host int32 tensor (capacity, 2).  Returns |J|; pairs land in out[:|J|]."""
    for t in (key_R, key_S, out):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError("join_host takes contiguous HOST tensors")
    if key_R.dtype != key_S.dtype or key_R.dtype not in (torch.int32, torch.int64):
        raise ValueError("keys must both be int32 or int64")
    n = ctypes.c_uint64()
    _check(lib.join_host(ctx.h, ctypes.c_void_p(key_R.data_ptr()), key_R.numel(),
                         ctypes.c_void_p(key_S.data_ptr()), key_S.numel(),
                         I32 if key_R.dtype == torch.int32 else I64,
                         ctypes.c_void_p(out.data_ptr()), out.shape[0], ctypes.byref(n)))
    return n.value


def join_host_batch(ctx: Context, batches):
    """A stream of independent equi joins from HOST tensors: batches = [(key_R, key_S, out), ...]
    (as join_host).  Consecutive batches' transfers overlap on two internal streams.
    Returns the list of |J_b|."""
    nb = len(batches)
    for kR, kS, o in batches:
        for t in (kR, kS, o):
            if t.is_cuda or not t.is_contiguous():
                raise ValueError("join_host_batch takes contiguous HOST tensors")
        if kR.dtype != kS.dtype or kR.dtype != batches[0][0].dtype or kR.dtype not in (torch.int32, torch.int64):
            raise ValueError("keys must all be int32 or all int64")
    vp, u64 = ctypes.c_void_p, ctypes.c_uint64
    kR = (vp * nb)(*[b[0].data_ptr() for b in batches])
    kS = (vp * nb)(*[b[1].data_ptr() for b in batches])
    nR = (u64 * nb)(*[b[0].numel() for b in batches])
    nS = (u64 * nb)(*[b[1].numel() for b in batches])
    outs = (vp * nb)(*[b[2].data_ptr() for b in batches])
    cap = (u64 * nb)(*[b[2].shape[0] for b in batches])
    n = (u64 * nb)()
    kt = I32 if nb == 0 or batches[0][0].dtype == torch.int32 else I64
    _check(lib.join_host_batch(ctx.h, nb, kR, nR, kS, nS, kt, outs, cap, n))
    return [n[i] for i in range(nb)]


# ---------------------------------------------------------------- multi-GPU (NCCL)

def region_classify(op: str, k: int, m: int = 0, g: int = -1):
    """Region-matrix cell classes (gj_region_classify, §4.2 Fig. 9): a (k, k)
    uint8 array, [x, y] = class of (R bucket x, S bucket y): 0 White, 1 Red, 2 Green.
    band: m = Red radius ceil(eps / w), g = Green radius floor((eps + 1) / w) - 1."""
    import numpy as np
    out = np.zeros(k * k, dtype=np.uint8)
    _check(lib.gj_region_classify(OPS[op], k, m, g, out.ctypes.data_as(ctypes.c_void_p)))
    return out.reshape(k, k)


def dist_plan(counts, rank: int, lbits: int = 0):
    """Host-only receive plan of the equi-join shuffle (gj_dist_plan), the function
    every rank runs on the all-gathered counts.  counts: (G, G, 2^lbits) array,
    counts[q, p, d] = tuples rank q sends to rank p with local digit d.
    Returns (adj (G, 2^lbits) uint32, seg (2^lbits + 1) uint32, need (G) uint64)."""
    import numpy as np
    m = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
    G, L = m.shape[0], 1 << lbits
    if m.shape != (G, G, L):
        raise ValueError("counts must have shape (G, G, 2^lbits)")
    adj = np.zeros(G * L, dtype=np.uint32)
    seg = np.zeros(L + 1, dtype=np.uint32)
    need = np.zeros(G, dtype=np.uint64)
    P32 = ctypes.POINTER(ctypes.c_uint32)
    _check(lib.gj_dist_plan(m.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), G, lbits, rank,
                            adj.ctypes.data_as(P32), seg.ctypes.data_as(P32),
                            need.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    return adj.reshape(G, L), seg, need


class Comm:
    """gj_comm: an NCCL communicator over the ranks of a torch.distributed group.

    Rank 0 creates the ncclUniqueId; it is broadcast with torch.distributed (any
    backend), then every rank calls gj_comm_init on its current CUDA device."""

    def __init__(self, rank: int, world: int, group=None):
        import torch.distributed as dist
        uid = (ctypes.c_uint8 * COMM_ID_BYTES)()
        if rank == 0:
            _check(lib.gj_comm_unique_id(ctypes.cast(uid, ctypes.c_void_p)))
        obj = [bytes(uid)]
        if world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        uid = (ctypes.c_uint8 * COMM_ID_BYTES).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        _check(lib.gj_comm_init(ctypes.byref(h), ctypes.cast(uid, ctypes.c_void_p), world, rank))
        self.h, self.rank, self.world = h, rank, world

    def close(self):
        if getattr(self, "h", None):
            lib.gj_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def join_dist_count(ctx: Context, comm: Comm, R, S):
    """Collective.  Returns (n_local, n_global)."""
    nl, ng = ctypes.c_uint64(), ctypes.c_uint64()
    _check(lib.join_dist_count(ctx.h, comm.h, _rel(R), _rel(S), ctypes.byref(nl), ctypes.byref(ng)))
    return nl.value, ng.value


def join_dist_count_filtered(ctx: Context, comm: Comm, R, S, flags: int = RANGE | BLOOM | TWO_SIDED,
                             bloom_bits_per_key: float = 8.0):
    """Collective pre-filtered equi join count.  Returns (n_local, n_global, (kept_R, kept_S))."""
    nl, ng = ctypes.c_uint64(), ctypes.c_uint64()
    kept = (ctypes.c_uint64 * 2)()
    _check(lib.join_dist_count_filtered(ctx.h, comm.h, _rel(R), _rel(S), int(flags), float(bloom_bits_per_key),
                                        ctypes.byref(nl), ctypes.byref(ng), kept))
    return nl.value, ng.value, (kept[0], kept[1])


def prefilter_dist(ctx: Context, comm: Comm, R, S, flags: int = RANGE | BLOOM | TWO_SIDED, op: str = "eq",
                   eps: int = 0, bloom_bits_per_key: float = 8.0):
    """Collective sharded pre-filter: this rank's surviving (R_keys, R_rids, S_keys, S_rids)."""
    rR, rS = _rel(R), _rel(S)
    kR = (R.key if isinstance(R, Rel) else R)
    kS = (S.key if isinstance(S, Rel) else S)
    okR, orR = torch.empty_like(kR), torch.empty(kR.numel(), dtype=torch.int32, device=kR.device)
    okS, orS = torch.empty_like(kS), torch.empty(kS.numel(), dtype=torch.int32, device=kS.device)
    nR, nS = ctypes.c_uint64(), ctypes.c_uint64()
    _check(lib.prefilter_dist(ctx.h, comm.h, rR, rS, flags, OPS[op], int(eps), float(bloom_bits_per_key),
                              ctypes.c_void_p(okR.data_ptr()), ctypes.c_void_p(orR.data_ptr()), ctypes.byref(nR),
                              ctypes.c_void_p(okS.data_ptr()), ctypes.c_void_p(orS.data_ptr()), ctypes.byref(nS)))
    return okR[: nR.value], orR[: nR.value], okS[: nS.value], orS[: nS.value]


def join_dist_materialize(ctx: Context, comm: Comm, R, S, n_local: Optional[int] = None,
                          out: Optional[torch.Tensor] = None):
    """Collective.  Writes this rank's share of J(R, S) (global rids)."""
    if n_local is None and out is None:
        n_local, _ = join_dist_count(ctx, comm, R, S)
    key = (R.key if isinstance(R, Rel) else R)
    buf = _out(n_local or 0, out, key.device)
    w = ctypes.c_uint64()
    _check(lib.join_dist_materialize(ctx.h, comm.h, _rel(R), _rel(S), ctypes.c_void_p(buf.data_ptr()),
                                     buf.shape[0], ctypes.byref(w)))
    return buf[: w.value]


def theta_join_dist_count(ctx: Context, comm: Comm, R, S, op: str, eps: int = 0):
    nl, ng = ctypes.c_uint64(), ctypes.c_uint64()
    _check(lib.theta_join_dist_count(ctx.h, comm.h, _rel(R), _rel(S), OPS[op], int(eps), ctypes.byref(nl),
                                     ctypes.byref(ng)))
    return nl.value, ng.value


def theta_join_dist_materialize(ctx: Context, comm: Comm, R, S, op: str, eps: int = 0,
                                n_local: Optional[int] = None, out: Optional[torch.Tensor] = None):
    if n_local is None and out is None:
        n_local, _ = theta_join_dist_count(ctx, comm, R, S, op, eps)
    key = (R.key if isinstance(R, Rel) else R)
    buf = _out(n_local or 0, out, key.device)
    w = ctypes.c_uint64()
    _check(lib.theta_join_dist_materialize(ctx.h, comm.h, _rel(R), _rel(S), OPS[op], int(eps),
                                           ctypes.c_void_p(buf.data_ptr()), buf.shape[0], ctypes.byref(w)))
    return buf[: w.value]
