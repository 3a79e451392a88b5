"""Generator checks (gen/): determinism, bijectivity, ranges, shard consistency and
the distributions the workloads claim (DESIGN.md §3 input recipe)."""
import numpy as np

import gen


def test_deterministic_and_shardable():
    a = gen.rng(42, 3, 1000)
    b = gen.rng(42, 3, 1000)
    assert np.array_equal(a, b)
    assert np.array_equal(gen.rng(42, 3, 300, offset=700), a[700:])
    assert not np.array_equal(gen.rng(42, 4, 1000), a)
    assert np.array_equal(gen.uniform(200, 77, 1, 2, offset=100), gen.uniform(300, 77, 1, 2)[100:])


def test_mix64_known_values():
    # splitmix64 finalizer reference values (computed with Python ints, not numpy)
    def ref(z):
        M = (1 << 64) - 1
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)
    xs = np.array([0, 1, 2**63, 2**64 - 1, 0x9E3779B97F4A7C15], dtype=np.uint64)
    assert [int(v) for v in gen.mix64(xs)] == [ref(int(x)) for x in xs]


def test_perm_is_bijection():
    for b in (1, 5, 16, 17):
        x = np.arange(1 << b, dtype=np.uint64)
        y = gen.perm(x, b, seed=123)
        assert y.max() < (1 << b)
        assert len(np.unique(y)) == 1 << b


def test_uniform_range_and_distinct_fraction():
    u = gen.uniform(100_000, 1000, 5, 0)
    assert u.min() >= 0 and u.max() < 1000
    # n draws from n values leave ~ n(1-(1-1/n)^n) ~ 0.632n distinct
    n = 10_000
    d = len(np.unique(gen.uniform(n, n, 9, 1)))
    assert abs(d - n * (1 - (1 - 1 / n) ** n)) < 0.05 * n


def test_zipf_top_rank_frequency():
    N = 1 << 14
    q = gen.zipf_table(N)
    r = gen.zipf_ranks(1 << 20, q, seed=1, stream=1)
    assert r.min() >= 0 and r.max() < N
    H = np.sum(1.0 / np.arange(1, N + 1))
    assert abs((r == 0).mean() - 1 / H) < 0.003
    assert abs((r == 1).mean() - 0.5 / H) < 0.003


def test_pkfk_shapes():
    R, S, m = gen.pkfk(12, 5000, seed=2)
    assert len(np.unique(R)) == 1 << 12
    assert np.array_equal(S, R[m])


def test_c5_shapes():
    R, S, m = gen.c5(1 << 10, 1 << 14, seed=3)
    assert (R % 2 == 0).all() and len(np.unique(R)) == len(R)
    mem = m >= 0
    assert abs(mem.mean() - 0.1) < 0.01
    assert (S[~mem] % 2 == 1).all() and (S[mem] % 2 == 0).all()
