"""CPU oracle for the GPU join hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product package
``paper_1904_11201_b200`` never imports it and shares no code with it (the C++ in
``oracle/oracle.cpp`` includes nothing from ``paper_1904_11201_b200/csrc``).

Functions (each cites the passage it follows; see oracle.cpp for the C++ bodies):

* ``nlj``                O1  nested loop join, canonical order
* ``hash_equi``          O2  unordered_multimap build/probe + sort PAPER.md:68
* ``hash_equi_sliced``   O7  O2 per key slice fmix64(k) mod T on T threads (the
                             multi-core CPU baseline); pinned to O2
* ``theta_count_sorted`` O3  sort + binary-search counts          definition (1) in oracle.cpp
* ``theta_count_per_row`` O3r O3's counts per R row              definition (1) in oracle.cpp
* ``band_materialize``   O4  sorted range enumeration             definition (1), band
* ``equi_count_hist``    O5  sum_k cntR(k)*cntS(k)                north star invariant
* ``semijoin_exact``     O6  exact common-key filter mask         PAPER.md:80-81, Alg.1
* ``semijoin_band``      O6b band semi-join mask                  definition (1), band
* ``pkfk_closed_form``   O8  J = {(m_j, j)} for the PK-FK generators (R keys a bijection
                             of R rows, S.key[j] = R.key[m_j]); pinned to O2 in tests.
* ``eq8_from_counts``    O9  the paper's result-size estimate Eq.7-8
* ``eq8_rsize``          O9  Eq.8 over a join's own partitions      (partition_of: the
                             product's key -> Reducer map, a performance choice)
* ``gather_payloads``    O10 late materialisation of result tuples PAPER.md:141

Parity status: every function above is pinned (tests/test_oracle.py); none is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC_PATH = os.path.join(HERE, "oracle.cpp")

OPS = {"eq": 0, "ne": 1, "lt": 2, "le": 3, "gt": 4, "ge": 5, "band": 6}


def build(force: bool = False) -> str:
    """Compile oracle.cpp (plain C++17, -O2, no intrinsics) into liboracle.so."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH):
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-pthread", "-o", LIB_PATH, SRC_PATH])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        u64, i32, u32, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p
        L.orc_nlj.argtypes = [vp, u64, vp, u64, i32, i32, u64, u32, u32, vp, u64]
        L.orc_nlj.restype = u64
        L.orc_hash_equi.argtypes = [vp, u64, vp, u64, i32, u32, u32, vp, u64]
        L.orc_hash_equi.restype = u64
        L.orc_theta_count_sorted.argtypes = [vp, u64, vp, u64, i32, i32, u64]
        L.orc_theta_count_sorted.restype = u64
        L.orc_theta_count_per_row.argtypes = [vp, u64, vp, u64, i32, i32, u64, vp]
        L.orc_theta_count_per_row.restype = None
        L.orc_band_materialize_sorted.argtypes = [vp, u64, vp, u64, i32, u64, u32, u32, vp, u64]
        L.orc_band_materialize_sorted.restype = u64
        L.orc_hash_equi_sliced.argtypes = [vp, u64, vp, u64, i32, u32, u32, vp, u64, i32]
        L.orc_hash_equi_sliced.restype = u64
        L.orc_equi_count_hist.argtypes = [vp, u64, vp, u64, i32]
        L.orc_equi_count_hist.restype = u64
        L.orc_semijoin_exact.argtypes = [vp, u64, vp, u64, i32, vp]
        L.orc_semijoin_exact.restype = u64
        L.orc_semijoin_band.argtypes = [vp, u64, vp, u64, i32, u64, vp]
        L.orc_semijoin_band.restype = u64
        _lib = L
    return _lib


def _keys(R, S):
    R = np.ascontiguousarray(R)
    S = np.ascontiguousarray(S)
    if R.dtype != S.dtype or R.dtype not in (np.int32, np.int64):
        raise TypeError("R and S keys must both be int32 or both int64")
    return R, S, 0 if R.dtype == np.int32 else 1


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def nlj(R, S, op="eq", eps=0, rid_base_R=0, rid_base_S=0, count_only=False, cap=None):
    """O1: returns count, or (count, pairs[count,2] uint32) in canonical order."""
    R, S, t = _keys(R, S)
    L = lib()
    if count_only:
        return L.orc_nlj(_ptr(R), len(R), _ptr(S), len(S), t, OPS[op], eps, rid_base_R, rid_base_S, None, 0)
    if cap is None:
        cap = L.orc_nlj(_ptr(R), len(R), _ptr(S), len(S), t, OPS[op], eps, rid_base_R, rid_base_S, None, 0)
    out = np.empty((max(cap, 1), 2), dtype=np.uint32)
    c = L.orc_nlj(_ptr(R), len(R), _ptr(S), len(S), t, OPS[op], eps, rid_base_R, rid_base_S, _ptr(out), cap)
    return c, out[: min(c, cap)]


def hash_equi(R, S, rid_base_R=0, rid_base_S=0):
    """O2: (count, pairs) in canonical order."""
    R, S, t = _keys(R, S)
    L = lib()
    c = L.orc_equi_count_hist(_ptr(R), len(R), _ptr(S), len(S), t)  # only sizes the buffer
    out = np.empty((max(c, 1), 2), dtype=np.uint32)
    c2 = L.orc_hash_equi(_ptr(R), len(R), _ptr(S), len(S), t, rid_base_R, rid_base_S, _ptr(out), c)
    return c2, out[: min(c, c2)]


def hash_equi_sliced(R, S, threads=0, rid_base_R=0, rid_base_S=0):
    """O7: O2 sliced by fmix64(key) mod T, one slice per host thread (T = 0: all cores);
    (count, pairs) in canonical order."""
    R, S, t = _keys(R, S)
    L = lib()
    c = L.orc_equi_count_hist(_ptr(R), len(R), _ptr(S), len(S), t)  # only sizes the buffer
    out = np.empty((max(c, 1), 2), dtype=np.uint32)
    c2 = L.orc_hash_equi_sliced(_ptr(R), len(R), _ptr(S), len(S), t, rid_base_R, rid_base_S, _ptr(out), c, threads)
    return c2, out[: min(c, c2)]


def theta_count_sorted(R, S, op, eps=0):
    """O3."""
    R, S, t = _keys(R, S)
    return lib().orc_theta_count_sorted(_ptr(R), len(R), _ptr(S), len(S), t, OPS[op], eps)


def theta_count_per_row(R, S, op, eps=0):
    """O3r: uint64 array, |{j : R[i] op S[j]}| for every R row i."""
    R, S, t = _keys(R, S)
    out = np.zeros(max(len(R), 1), dtype=np.uint64)
    lib().orc_theta_count_per_row(_ptr(R), len(R), _ptr(S), len(S), t, OPS[op], eps, _ptr(out))
    return out[: len(R)]


def band_materialize(R, S, eps, rid_base_R=0, rid_base_S=0):
    """O4: (count, pairs) for |R.key - S.key| <= eps in canonical order."""
    R, S, t = _keys(R, S)
    L = lib()
    c = L.orc_theta_count_sorted(_ptr(R), len(R), _ptr(S), len(S), t, OPS["band"], eps)
    out = np.empty((max(c, 1), 2), dtype=np.uint32)
    c2 = L.orc_band_materialize_sorted(_ptr(R), len(R), _ptr(S), len(S), t, eps, rid_base_R, rid_base_S, _ptr(out), c)
    return c2, out[: min(c, c2)]


def equi_count_hist(R, S):
    """O5."""
    R, S, t = _keys(R, S)
    return lib().orc_equi_count_hist(_ptr(R), len(R), _ptr(S), len(S), t)


def semijoin_exact(K, other):
    """O6: boolean keep-mask of K's rows whose key occurs in other."""
    K, other, t = _keys(K, other)
    keep = np.empty(max(len(K), 1), dtype=np.uint8)
    lib().orc_semijoin_exact(_ptr(K), len(K), _ptr(other), len(other), t, _ptr(keep))
    return keep[: len(K)].astype(bool)


def semijoin_band(K, other, eps):
    """O6b: keep-mask of K's rows within eps of some key of other."""
    K, other, t = _keys(K, other)
    keep = np.empty(max(len(K), 1), dtype=np.uint8)
    lib().orc_semijoin_band(_ptr(K), len(K), _ptr(other), len(other), t, eps, _ptr(keep))
    return keep[: len(K)].astype(bool)


def pkfk_closed_form(m, rid_base_S=0, r_rows=None):
    """O8: expected join of a PK-FK workload whose R keys are a bijection of R rows.

    m[j] = the R row drawn for S row j (or -1 for a non-member).  Then
    J = {(m_j, j) : m_j >= 0}; returned as (count, pairs) in canonical order,
    sorted by (m_j, j) with a stable argsort on m_j (j is already ascending).
    ``r_rows`` optionally restricts to R rows present (a shard [lo, hi)).
    """
    m = np.asarray(m, dtype=np.int64)
    j = np.arange(len(m), dtype=np.int64) + rid_base_S
    keep = m >= 0
    if r_rows is not None:
        keep &= (m >= r_rows[0]) & (m < r_rows[1])
    m, j = m[keep], j[keep]
    order = np.argsort(m, kind="stable")
    pairs = np.stack([m[order], j[order]], axis=1).astype(np.uint32)
    return len(pairs), pairs


def eq8_from_counts(s_counts, t_counts, S_total, T_total):
    """O9: the paper's result-size estimate, Eq.7-8, evaluated in
    the paper's order and notation with exact rationals.  Inputs: the per-Reducer
    post-filter tuple counts s_i (S side) and t_i (T side) of k Reducers, and the
    unfiltered table sizes |S|, |T|.

      beta  = sum_i s_i / |S|,  gamma = sum_i t_i / |T|          (filter ratios, :201)
      omega_i = s_i / (beta |S|),  lambda_i = t_i / (gamma |T|)  (shares, Eq.7: sum = 1)
      R_size = gamma * beta * |S| * |T| * sum_i omega_i * lambda_i          (Eq.8)

    Returns R_size as a Fraction (an integer for integer counts).  |S| or |T| = 0, or
    nothing surviving the filter, gives 0 ("DegenerateInput ... all-zero")."""
    from fractions import Fraction
    s_counts = [int(x) for x in s_counts]
    t_counts = [int(x) for x in t_counts]
    if len(s_counts) != len(t_counts):
        raise ValueError("one s and one t count per Reducer")
    if S_total == 0 or T_total == 0 or sum(s_counts) == 0 or sum(t_counts) == 0:
        return Fraction(0)
    beta = Fraction(sum(s_counts), S_total)
    gamma = Fraction(sum(t_counts), T_total)
    omega = [Fraction(x) / (beta * S_total) for x in s_counts]
    lam = [Fraction(x) / (gamma * T_total) for x in t_counts]
    assert sum(omega) == 1 and sum(lam) == 1  # Eq.7
    return gamma * beta * S_total * T_total * sum(o * l for o, l in zip(omega, lam))


def partition_of(K, bits):
    """The Reducer of every key when the library's join runs with 2^bits partitions.

    Eq.8 holds for ANY key -> Reducer map that sends equal keys to the same Reducer
    ("tuples with the same key value are passed to the same Reducer");
    WHICH map is a performance choice of the product (the top ``bits``
    bits of hi32(key * 0x9E3779B97F4A7C15) over the key's two's-complement pattern,
    int64 keys first folded as x ^ (x >> 32)).  It is restated here only so that
    gj_join_stats can be compared with Eq.8 at the SAME map; nothing else in the
    oracle depends on it, and Eq.8 itself is pinned by eq8_from_counts' tests."""
    K = np.asarray(K)
    if bits == 0:
        return np.zeros(len(K), dtype=np.uint64)
    x = K.astype(np.int64).view(np.uint64) if K.dtype == np.int64 else K.astype(np.uint32).astype(np.uint64)
    if K.dtype == np.int64:
        x = x ^ (x >> np.uint64(32))
    with np.errstate(over="ignore"):
        h = (x * np.uint64(0x9E3779B97F4A7C15)) >> np.uint64(32)
    return (h & np.uint64(0xFFFFFFFF)) >> np.uint64(32 - bits)


def eq8_rsize(R, S, bits, reducer_of=None):
    """O9 on two key columns: Eq.8 with the k = 2^bits Reducers given by ``reducer_of``
    (default: the product's partition map, partition_of), no pre-filter (beta = gamma
    = 1).  The join's own R plays the paper's T, S plays S."""
    k = 1 << bits
    f = reducer_of or (lambda K: partition_of(K, bits))
    cR = np.bincount(np.asarray(f(R)).astype(np.int64), minlength=k)
    cS = np.bincount(np.asarray(f(S)).astype(np.int64), minlength=k)
    v = eq8_from_counts(cS, cR, len(S), len(R))
    assert v.denominator == 1
    return int(v)


def gather_payloads(pairs, payload_R=None, payload_S=None, rid_base_R=0, rid_base_S=0):
    """O10: "if the m-th join key of T' and the n-th join key of S' match,
    we extract the m-th record of T' and the n-th record of S'": row rid_R - base of R's
    payload and row rid_S - base of S's payload for every pair, in pair order."""
    pairs = np.asarray(pairs).astype(np.int64) & 0xFFFFFFFF
    oR = None if payload_R is None else np.asarray(payload_R)[pairs[:, 0] - rid_base_R]
    oS = None if payload_S is None else np.asarray(payload_S)[pairs[:, 1] - rid_base_S]
    return oR, oS
