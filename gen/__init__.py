"""Seeded, counter-based synthetic relation generators (test + bench infrastructure).

This module is shared by the oracle side (``oracle/``, ``tests/``) and the GPU side
(``bench.py`` feeds its output, or its bit-identical CUDA twin ``gen/gen_device.cu``,
to the product library).  It holds NONE of the join method's arithmetic: it only
draws keys.  Every draw is a pure function of (seed, stream, i), so a shard of any
relation can be regenerated independently and the CPU and GPU versions agree bit
for bit (checked by ``tests/test_gen.py`` and the ``-m gpu`` twin test).

Recipes follow SURVEY.md §8(d) "Generators" and DESIGN.md §3 (input recipe):

* ``mix64``      splitmix64 finalizer.
* ``rng``        rng(seed, stream, i) = mix64(mix64(seed + G*(stream+1)) + i), G = 0x9E3779B97F4A7C15.
* ``uniform``    uniform(D) = ((rng >> 32) * D) >> 32 for 1 <= D <= 2**32 (exact in uint64).
* ``perm``       keyed bijection on [0, 2**b): 3 rounds of (add, xorshift, odd multiply) mod 2**b.
* ``zipf_table`` quantised Zipf(s) CDF; sampling is integer-only (search on the quantised CDF).

The paper's own synthetic data (§5.1.3) divides uniform keys by an
integer; ``uniform_div`` reproduces that shape for the C1-style workloads.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
BASE_SEED = 0x1904_11201
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_S30, _S27, _S31, _S32 = np.uint64(30), np.uint64(27), np.uint64(31), np.uint64(32)


def mix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = (x ^ (x >> _S30)) * _M1
        x = (x ^ (x >> _S27)) * _M2
        return x ^ (x >> _S31)


def stream_key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        s = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + GOLDEN * np.uint64(stream + 1)
    return mix64(np.array([s], dtype=np.uint64))[0]


def rng(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    """rng(seed, stream, i) for i in [offset, offset+n) as uint64."""
    k = stream_key(seed, stream)
    i = np.arange(offset, offset + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(i + k)


def uniform(n: int, D: int, seed: int, stream: int, offset: int = 0) -> np.ndarray:
    """uniform integers in [0, D), D <= 2**32, as uint64 (caller casts)."""
    assert 1 <= D <= 2**32
    u = rng(seed, stream, n, offset) >> _S32
    with np.errstate(over="ignore"):
        return (u * np.uint64(D)) >> _S32


def _perm_consts(b: int, seed: int):
    mask = (1 << b) - 1
    consts = []
    for r in range(3):
        u = int(rng(seed, 1000 + r, 2)[0]), int(rng(seed, 1000 + r, 2)[1])
        consts.append((u[0] & mask, (u[1] | 1) & mask))
    return mask, (b + 1) // 2, consts


def perm(x: np.ndarray, b: int, seed: int) -> np.ndarray:
    """Keyed bijection on [0, 2**b) (1 <= b <= 32).  Returns uint64."""
    assert 1 <= b <= 32
    mask, sh, consts = _perm_consts(b, seed)
    x = np.asarray(x, dtype=np.uint64).copy()
    M, SH = np.uint64(mask), np.uint64(sh)
    with np.errstate(over="ignore"):
        for add, odd in consts:
            x = (x + np.uint64(add)) & M
            x ^= x >> SH
            x = (x * np.uint64(odd)) & M
    return x


def perm_consts_flat(b: int, seed: int):
    """(mask, shift, [add0, odd0, add1, odd1, add2, odd2]) for the CUDA twin."""
    mask, sh, consts = _perm_consts(b, seed)
    flat = []
    for a, o in consts:
        flat += [a, o]
    return mask, sh, flat


def zipf_table(N: int, s: float = 1.0) -> np.ndarray:
    """Quantised Zipf(s) CDF over ranks 0..N-1 (p_k ∝ 1/(k+1)^s).

    cdf_q[k] = floor(F(k) * 2**32) clipped to 2**32-1, with F(N-1) forced to 2**32
    (stored as uint64).  A draw with 32-bit uniform u has rank = #{k : cdf_q[k] <= u},
    i.e. ``searchsorted(cdf_q, u, 'right')`` -- integer-only, so every consumer that
    receives this table reproduces the same ranks bit for bit.
    """
    w = 1.0 / np.power(np.arange(1, N + 1, dtype=np.float64), s)
    c = np.cumsum(w)
    q = np.floor(c / c[-1] * 2.0**32)
    q = np.minimum(q, 2.0**32).astype(np.uint64)
    q[-1] = np.uint64(2**32)
    return q


def zipf_ranks(n: int, cdf_q: np.ndarray, seed: int, stream: int, offset: int = 0) -> np.ndarray:
    u = rng(seed, stream, n, offset) >> _S32
    return np.searchsorted(cdf_q, u, side="right").astype(np.uint64)


# ---------------------------------------------------------------- workloads
# Each returns (R_key, S_key) numpy arrays (int32 or int64) plus, for the PK-FK
# workloads, the drawn R row of every S row (m_j, or -1 for a non-member), which
# is what the oracle's closed form O8 needs.

def uniform_keys(n: int, D: int, seed: int, stream: int, dtype=np.int32, offset: int = 0):
    return uniform(n, D, seed, stream, offset).astype(dtype)


def uniform_div(n: int, key_max: int, divisor: int, seed: int, stream: int, dtype=np.int32):
    """The paper's synthetic shape: uniform keys in [0,key_max) divided by an integer."""
    return (uniform(n, key_max, seed, stream) // np.uint64(divisor)).astype(dtype)


def c1(seed: int = BASE_SEED, n: int = 10_000, D: int = 10_000):
    """configs[0]: R=S=10^4, uniform keys in [0,10^4)."""
    return uniform_keys(n, D, seed, 0), uniform_keys(n, D, seed, 1)


def pkfk(nR_bits: int, nS: int, seed: int = BASE_SEED, r_offset: int = 0, nR: int | None = None,
         s_offset: int = 0):
    """PK-FK: R.key[i] = perm_b(i) (unique); S.key[j] = perm_b(m_j), m_j = uniform(2**b).

    configs[1] (C2) is pkfk(27, 2**27).  Returns (R_key, S_key, m) with m = drawn R row.
    """
    b = nR_bits
    nR = (1 << b) if nR is None else nR
    R = perm(np.arange(r_offset, r_offset + nR, dtype=np.uint64), b, seed).astype(np.int32)
    m = uniform(nS, 1 << b, seed, 1, s_offset)
    S = perm(m, b, seed).astype(np.int32)
    return R, S, m.astype(np.int64)


def zipf_pkfk(nR_bits: int, nS: int, cdf_q: np.ndarray, seed: int = BASE_SEED, s_offset: int = 0):
    """configs[2] (C3): R unique over 2**b ranks, S = FK drawn Zipf(1) over R's ranks."""
    b = nR_bits
    R = perm(np.arange(1 << b, dtype=np.uint64), b, seed).astype(np.int32)
    m = zipf_ranks(nS, cdf_q, seed, 1, s_offset)
    S = perm(m, b, seed).astype(np.int32)
    return R, S, m.astype(np.int64)


def c4(seed: int = BASE_SEED, nR: int = 1 << 20, nS: int = 1 << 24, D: int = 1 << 30):
    """configs[3]: band join R 2^20 x S 2^24 uniform in [0, 2^30), eps = 53687 (sel ~1e-4)."""
    return uniform_keys(nR, D, seed, 0), uniform_keys(nS, D, seed, 1)


C4_EPS = 53687


def c5_member_mask(nS: int, seed: int, offset: int = 0) -> np.ndarray:
    """C5: S row j is a member w.p. 0.1 (hi32(rng) < 0.1 * 2^32)."""
    thr = np.uint64(int(0.1 * 2**32))
    return (rng(seed, 3, nS, offset) >> _S32) < thr


def c5(nR: int, nS: int, seed: int = BASE_SEED, r_offset: int = 0, s_offset: int = 0, b: int = 31):
    """configs[4] (C5) with int64 keys over a domain of 2^b R rows (b = 31 is configs[4]):
    R.key[i] = 2*perm_b(i) (even, unique); S member rows: 2*perm_b(m_j), m_j = uniform(2^b);
    non-members odd 2*uniform(1.25*2^b)+1."""
    R = (perm(np.arange(r_offset, r_offset + nR, dtype=np.uint64), b, seed) * np.uint64(2)).astype(np.int64)
    mem = c5_member_mask(nS, seed, s_offset)
    m = uniform(nS, 1 << b, seed, 1, s_offset)
    nonm = uniform(nS, int(1.25 * 2**b), seed, 4, s_offset) * np.uint64(2) + np.uint64(1)
    S = np.where(mem, perm(m, b, seed) * np.uint64(2), nonm).astype(np.int64)
    return R, S, np.where(mem, m.astype(np.int64), -1)
