"""torch wrappers over gen/libgjgen.so (the CUDA twin of gen/__init__.py).

Test + bench infrastructure: draws the same keys as the numpy generator, directly
in HBM.  Holds none of the join method's arithmetic.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import perm_consts_flat, stream_key

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgjgen.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        vp, u64, u32, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
        pu = ctypes.POINTER(ctypes.c_uint64)
        L.gjgen_uniform.argtypes = [vp, u64, u64, u64, u64, i32, vp]
        L.gjgen_perm_range.argtypes = [vp, u64, u64, u32, pu, u64, u64, i32, vp]
        L.gjgen_pkfk.argtypes = [vp, u64, u64, u32, pu, u64, u64, u64, vp]
        L.gjgen_zipf.argtypes = [vp, u64, u64, u32, pu, vp, u64, u64, u64, vp]
        L.gjgen_c5s.argtypes = [vp, u64, u64, u32, pu, u64, u64, u64, u64, u64, u64, u64, vp]
        _lib = L
    return _lib


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _perm(b, seed):
    mask, sh, flat = perm_consts_flat(b, seed)
    arr = (ctypes.c_uint64 * 6)(*flat)
    return mask, sh, arr


def _ok(rc):
    if rc != 0:
        raise RuntimeError(f"gjgen kernel launch failed: cuda error {rc}")


def uniform(n, D, seed, stream, dtype=torch.int32, offset=0, device="cuda"):
    out = torch.empty(n, dtype=dtype, device=device)
    _ok(lib().gjgen_uniform(ctypes.c_void_p(out.data_ptr()), n, D, int(stream_key(seed, stream)), offset,
                            int(dtype == torch.int64), _stream()))
    return out


def perm_range(n, b, seed, offset=0, mult=1, dtype=torch.int32, device="cuda"):
    out = torch.empty(n, dtype=dtype, device=device)
    mask, sh, c = _perm(b, seed)
    _ok(lib().gjgen_perm_range(ctypes.c_void_p(out.data_ptr()), n, mask, sh, c, offset, mult,
                               int(dtype == torch.int64), _stream()))
    return out


def pkfk_S(n, b, seed, offset=0, device="cuda", domain=None):
    """S FK draws: perm_b(rank), rank uniform in [0, domain) (default 2^b, i.e. the
    keys of perm_range(2^b, b)); domain = |R| for R = perm_range(|R|, b) with b > log2|R|."""
    out = torch.empty(n, dtype=torch.int32, device=device)
    mask, sh, c = _perm(b, seed)
    D = (1 << b) if domain is None else domain
    _ok(lib().gjgen_pkfk(ctypes.c_void_p(out.data_ptr()), n, mask, sh, c, D, int(stream_key(seed, 1)),
                         offset, _stream()))
    return out


def zipf_S(n, b, cdf_q: torch.Tensor, seed, offset=0, device="cuda"):
    out = torch.empty(n, dtype=torch.int32, device=device)
    mask, sh, c = _perm(b, seed)
    _ok(lib().gjgen_zipf(ctypes.c_void_p(out.data_ptr()), n, mask, sh, c, ctypes.c_void_p(cdf_q.data_ptr()),
                         cdf_q.numel(), int(stream_key(seed, 1)), offset, _stream()))
    return out


def c5_S(n, seed, offset=0, device="cuda", b=31):
    """gen.c5's S column on the device (domain 2^b; b = 31 is configs[4])."""
    out = torch.empty(n, dtype=torch.int64, device=device)
    mask, sh, c = _perm(b, seed)
    thr = int(0.1 * 2**32)
    _ok(lib().gjgen_c5s(ctypes.c_void_p(out.data_ptr()), n, mask, sh, c, int(stream_key(seed, 1)),
                        int(stream_key(seed, 3)), int(stream_key(seed, 4)), thr, 1 << b, int(1.25 * 2**b), offset,
                        _stream()))
    return out


def c5_R(n, seed, offset=0, device="cuda", b=31):
    """gen.c5's R column on the device: 2*perm_b(offset + i) as int64."""
    return perm_range(n, b, seed, offset=offset, mult=2, dtype=torch.int64, device=device)


def zipf_table_device(N: int, device="cuda") -> torch.Tensor:
    from . import zipf_table
    return torch.from_numpy(zipf_table(N).astype(np.uint64).view(np.int64)).to(device)
