"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bit-exact on every count and on the canonically sorted (rid_R, rid_S) pairs
(integer work: no tolerance).  Inputs are the seeded synthetic generators.
"""
import numpy as np
import pytest
import torch

import gen
import oracle

pytestmark = pytest.mark.gpu

OPS = ["eq", "ne", "lt", "le", "gt", "ge", "band"]


@pytest.fixture(scope="module")
def gj():
    import native_build
    native_build.build_all()
    import paper_1904_11201_b200 as m
    return m


@pytest.fixture()
def ctx(gj):
    c = gj.Context(0)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def canon_gpu(pairs_t):
    """Canonically sort GPU pairs on the device; return numpy uint32 (n, 2)."""
    if pairs_t.numel() == 0:
        return np.zeros((0, 2), np.uint32)
    p = pairs_t.to(torch.int64) & 0xFFFFFFFF
    packed = (p[:, 0] << 32) | p[:, 1]
    s, _ = torch.sort(packed)  # uint32 halves are non-negative, so signed sort is the canonical order
    hi = (s >> 32).to(torch.int64)
    lo = (s & 0xFFFFFFFF).to(torch.int64)
    return torch.stack([hi, lo], 1).cpu().numpy().astype(np.uint32)


def check_equi(gj, ctx, R, S, **kw):
    if isinstance(R, np.ndarray):
        tR, tS = dev(R), dev(S)
    else:
        tR, tS = R, S
    n = gj.join_count(ctx, tR, tS)
    out = gj.join_materialize(ctx, tR, tS, n)
    Rk = R if isinstance(R, np.ndarray) else R.key.cpu().numpy()
    Sk = S if isinstance(S, np.ndarray) else S.key.cpu().numpy()
    cn, cp = oracle.hash_equi(Rk, Sk, **kw)
    assert n == cn
    got = canon_gpu(out)
    assert got.shape == cp.shape and np.array_equal(got, cp)
    return n


def check_theta(gj, ctx, R, S, op, eps=0, materialize=True):
    tR, tS = dev(R), dev(S)
    n = gj.theta_join_count(ctx, tR, tS, op, eps)
    assert n == oracle.theta_count_sorted(R, S, op, eps), (op, eps)
    if materialize:
        out = gj.theta_join_materialize(ctx, tR, tS, op, eps, n)
        cn, cp = oracle.nlj(R, S, op, eps)
        assert cn == n
        assert np.array_equal(canon_gpu(out), cp), (op, eps)
    return n


# ------------------------------------------------------------------ generator twin

def test_device_generator_matches_numpy(gj):
    import gen.device as gd
    import native_build
    native_build.build_gen()
    n = 100_003
    for D in (10_000, 1 << 30, 2**32):
        assert np.array_equal(gd.uniform(n, D, 7, 1, offset=5).cpu().numpy(),
                              gen.uniform(n, D, 7, 1, offset=5).astype(np.int32))
    assert np.array_equal(gd.perm_range(n, 20, 3, offset=11).cpu().numpy(),
                          gen.perm(np.arange(11, 11 + n, dtype=np.uint64), 20, 3).astype(np.int32))
    R, S, m = gen.pkfk(18, n, seed=9)
    assert np.array_equal(gd.pkfk_S(n, 18, 9).cpu().numpy(), S)
    q = gen.zipf_table(1 << 16)
    Rz, Sz, mz = gen.zipf_pkfk(16, n, q, seed=4)
    assert np.array_equal(gd.zipf_S(n, 16, gd.zipf_table_device(1 << 16), 4).cpu().numpy(), Sz)
    R5, S5, m5 = gen.c5(1 << 10, n, seed=8)
    assert np.array_equal(gd.c5_S(n, 8).cpu().numpy(), S5)
    R5b, S5b, _ = gen.c5(1 << 10, n, seed=8, r_offset=77, s_offset=5, b=20)
    assert np.array_equal(gd.c5_S(n, 8, offset=5, b=20).cpu().numpy(), S5b)
    assert np.array_equal(gd.c5_R(1 << 10, 8, offset=77, b=20).cpu().numpy(), R5b)
    assert np.array_equal(gd.perm_range(1 << 10, 31, 8, mult=2, dtype=torch.int64).cpu().numpy(), R5)


# ------------------------------------------------------------------ golden fixtures on the GPU

@pytest.mark.parametrize("name", ["e1_small_mixed.json", "e2_int32_extremes.json", "e3_int64_extremes.json"])
def test_golden_on_gpu(gj, ctx, name):
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", name)))
    dt = np.int32 if g["dtype"] == "int32" else np.int64
    R, S = np.array(g["R"], dtype=dt), np.array(g["S"], dtype=dt)
    tR, tS = dev(R), dev(S)
    for c in g["cases"]:
        n = gj.theta_join_count(ctx, tR, tS, c["op"], c["eps"])
        assert n == c["count"], c
        out = canon_gpu(gj.theta_join_materialize(ctx, tR, tS, c["op"], c["eps"], n))
        if "pairs" in c:
            assert out.tolist() == c["pairs"], c
        if c["op"] == "eq":
            assert gj.join_count(ctx, tR, tS) == c["count"]
            out = canon_gpu(gj.join_materialize(ctx, tR, tS))
            if "pairs" in c:
                assert out.tolist() == c["pairs"]


# ------------------------------------------------------------------ equi hash join

def test_equi_c1_full(gj, ctx):
    """configs[0]: R=S=10^4 uniform keys in [0,10^4), default planner."""
    R, S = gen.c1()
    check_equi(gj, ctx, R, S)


@pytest.mark.parametrize("bits,chunk,pchunk", [(0, 2048, 2048), (0, 64, 100), (1, 2048, 2048), (2, 64, 100),
                                               (3, 2048, 2048), (9, 256, 64),
                                               (10, 2048, 1024), (12, 32, 1000), (19, 2048, 2048)])
def test_equi_planner_variants(gj, ctx, bits, chunk, pchunk):
    """1, 2 and 3 radix passes; build chunks split into many units; ragged tails."""
    ctx.set_option("part_bits", bits)
    ctx.set_option("build_chunk", chunk)
    ctx.set_option("probe_chunk", pchunk)
    R = gen.uniform_keys(20_011, 5_000, 1, 0)
    S = gen.uniform_keys(30_007, 5_000, 1, 1)
    check_equi(gj, ctx, R, S)


@pytest.mark.parametrize("fib,bits", [(1, 4), (1, 19), (1, 20), (0, 4), (0, 19)])
def test_equi_slot_constants(gj, ctx, fib, bits):
    """hj_count_i32's table slots: the khash bits below the consumed ones (fib, while
    hbits + 13 <= 32; bits = 20 falls back) or slot_hash -- dense keys (no collisions
    under fib), duplicates and a ragged tail both ways."""
    ctx.set_option("fib_slots", fib)
    ctx.set_option("part_bits", bits)
    rng = np.random.default_rng(7)
    R = rng.permutation(40_009).astype(np.int32)
    S = np.concatenate([rng.integers(0, 40_009, 50_003), np.full(300, 17)]).astype(np.int32)
    check_equi(gj, ctx, R, S)


def test_join_count_materialize(gj, ctx):
    """The fused call equals count + materialize (same pairs at the same positions),
    counts afresh every call, and reports GJ_ERANGE with nothing written when short."""
    import torch
    rng = np.random.default_rng(11)
    R = dev(rng.integers(0, 3000, 20_011).astype(np.int32))
    S = dev(rng.integers(0, 3000, 30_007).astype(np.int32))
    n = gj.join_count(ctx, R, S)
    ref = gj.join_materialize(ctx, R, S, n).clone()
    out = torch.full((n + 5, 2), -1, dtype=torch.int32, device="cuda")
    got = gj.join_count_materialize(ctx, R, S, out)
    assert got.shape[0] == n and torch.equal(got, ref)
    assert int((out[n:] == -1).sum()) == 10
    S[0] = S[1]  # same pointers, new contents: the fused call must not reuse the cache
    n2 = gj.join_count(ctx, R, S)
    got2 = gj.join_count_materialize(ctx, R, S, out)
    assert got2.shape[0] == n2 and np.array_equal(canon_gpu(got2), canon_gpu(gj.join_materialize(ctx, R, S, n2)))
    small = torch.full((n2 - 1, 2), -1, dtype=torch.int32, device="cuda")
    with pytest.raises(gj.GJError, match="GJ_ERANGE"):
        gj.join_count_materialize(ctx, R, S, small)
    assert int((small == -1).sum()) == small.numel()


@pytest.mark.parametrize("side", [1, 2])
def test_equi_build_side(gj, ctx, side):
    ctx.set_option("build_side", side)
    R = gen.uniform_keys(7_000, 3_000, 2, 0)
    S = gen.uniform_keys(11_000, 3_000, 2, 1)
    check_equi(gj, ctx, R, S)


def test_equi_all_equal_keys(gj, ctx):
    """Degenerate build-side duplication: |J| = nR * nS, build chunks overflow one table."""
    R = np.full(3000, 42, np.int32)
    S = np.full(2500, 42, np.int32)
    assert check_equi(gj, ctx, R, S) == 3000 * 2500


@pytest.mark.parametrize("n_min_r", [1, 5])
def test_equi_int32_min_keys(gj, ctx, n_min_r):
    """INT32_MIN is the int32 table's empty-slot marker: build rows with that key take
    the side list.  Unique (1 row) and duplicated (5 rows x 3 probe rows -> MULTI) cases,
    with and without radix passes."""
    rng = np.random.default_rng(n_min_r)
    R = rng.integers(-1000, 1000, 6000).astype(np.int32)
    S = rng.integers(-1000, 1000, 9000).astype(np.int32)
    R[rng.choice(len(R), n_min_r, replace=False)] = np.iinfo(np.int32).min
    S[rng.choice(len(S), 3, replace=False)] = np.iinfo(np.int32).min
    for bits in (-1, 0):
        ctx.set_option("part_bits", bits)
        check_equi(gj, ctx, R, S)


def test_equi_int64_extremes(gj, ctx):
    rng = np.random.default_rng(5)
    pool = np.array([np.iinfo(np.int64).min, -1, 0, 1, np.iinfo(np.int64).max, 2**40, -2**40], np.int64)
    R = np.concatenate([rng.choice(pool, 500), rng.integers(-1000, 1000, 5000)]).astype(np.int64)
    S = np.concatenate([rng.choice(pool, 700), rng.integers(-1000, 1000, 6000)]).astype(np.int64)
    check_equi(gj, ctx, R, S)


def test_equi_empty_and_tiny(gj, ctx):
    e = np.zeros(0, np.int32)
    one = np.array([5], np.int32)
    assert gj.join_count(ctx, dev(e), dev(one)) == 0
    assert gj.join_count(ctx, dev(one), dev(e)) == 0
    assert gj.join_materialize(ctx, dev(e), dev(one)).shape[0] == 0
    check_equi(gj, ctx, one, np.array([5, 5, 6], np.int32))


def test_equi_rid_map_and_base(gj, ctx):
    R = gen.uniform_keys(5000, 900, 3, 0)
    S = gen.uniform_keys(6000, 900, 3, 1)
    rid = np.arange(5000, dtype=np.int32)[::-1].copy() + 100
    tR = gj.Rel(dev(R), dev(rid))
    tS = gj.Rel(dev(S), None, 7_000_000)
    n = gj.join_count(ctx, tR, tS)
    got = canon_gpu(gj.join_materialize(ctx, tR, tS, n))
    cn, cp = oracle.hash_equi(R, S, rid_base_S=7_000_000)
    cp[:, 0] = rid[cp[:, 0]]
    cp = cp[np.lexsort((cp[:, 1], cp[:, 0]))]
    assert n == cn and np.array_equal(got, cp)


def test_equi_pkfk_c2_full_size(gj, ctx):
    """configs[1] at full size 2^27 x 2^27: every pair vs the closed form O8 (pinned to O2)."""
    R, S, m = gen.pkfk(27, 1 << 27)
    tR, tS = dev(R), dev(S)
    del R, S
    n = gj.join_count(ctx, tR, tS)
    assert n == 1 << 27
    out = gj.join_materialize(ctx, tR, tS, n)
    cn, cp = oracle.pkfk_closed_form(m)
    assert np.array_equal(canon_gpu(out), cp)


def test_equi_zipf_skew(gj, ctx):
    """configs[2] shape (scaled): R unique over 2^20 ranks, S Zipf(1) FK, 2^22 rows."""
    q = gen.zipf_table(1 << 20)
    R, S, m = gen.zipf_pkfk(20, 1 << 22, q, seed=77)
    n = gj.join_count(ctx, dev(R), dev(S))
    assert n == 1 << 22
    cn, cp = oracle.pkfk_closed_form(m)
    assert np.array_equal(canon_gpu(gj.join_materialize(ctx, dev(R), dev(S), n)), cp)


@pytest.mark.timeout(900)
def test_equi_zipf_c3_full_size(gj, ctx):
    """configs[2] at full size on one GPU: R = perm_28(i) (2^28 unique keys), S = 2^30 Zipf(1)
    FK draws (the hot key is ~5% of S).  O8: J = {(m_j, j)}, m_j = the R row drawn for S row j.
    Since R's keys are unique, the output equals J iff |J| = n_S, every S rid occurs exactly once,
    each pair's keys are equal (all 2^30 pairs checked on the device), and sampled pairs match
    the closed form evaluated on the host from the generator alone."""
    import gen.device as gd
    b, nS, seed = 28, 1 << 30, gen.BASE_SEED
    q = gen.zipf_table(1 << b)
    R = gd.perm_range(1 << b, b, seed)
    S = gd.zipf_S(nS, b, torch.from_numpy(q.view(np.int64)).cuda(), seed)
    n = gj.join_count(ctx, R, S)
    assert n == nS
    out = gj.join_materialize(ctx, R, S, n)
    rr, rs = out[:, 0].long(), out[:, 1].long()
    del out
    seen = torch.zeros(nS, dtype=torch.uint8, device=rr.device)
    seen[rs] = 1
    assert bool(seen.all())  # n_S pairs, every S row once
    del seen
    assert torch.equal(R[rr], S[rs])  # each pair joins equal keys
    r_of_s = torch.empty(nS, dtype=torch.int64, device=rr.device)
    r_of_s[rs] = rr
    js = np.unique(gen.uniform(2048, nS, 99, 0).astype(np.int64))
    m = np.array([gen.zipf_ranks(1, q, seed, 1, offset=int(j))[0] for j in js], dtype=np.int64)
    assert np.array_equal(r_of_s[torch.from_numpy(js).cuda()].cpu().numpy(), m)


@pytest.mark.parametrize("bits,chunk", [(-1, 4096), (4, 64), (0, 4096)])
def test_equi_deterministic_positions_duplicate_keys(gj, ctx, bits, chunk):
    """SPEC.md:539 determinism with duplicate BUILD keys (the MULTI write path: table
    insertion order races, so matches are emitted in sorted build-row order) and with
    partitions split over several build chunks: byte-identical outputs across runs and
    contexts, equal to the oracle."""
    R, S = gen.c1(n=30_000, D=3_000)
    tR, tS = dev(R), dev(S)
    ctx.set_option("part_bits", bits)
    ctx.set_option("build_chunk", chunk)
    a = gj.join_materialize(ctx, tR, tS).clone()
    b = gj.join_materialize(ctx, tR, tS).clone()
    ctx2 = gj.Context(0)
    ctx2.set_option("part_bits", bits)
    ctx2.set_option("build_chunk", chunk)
    c = gj.join_materialize(ctx2, tR, tS)
    ctx2.close()
    assert torch.equal(a, b) and torch.equal(a, c)
    assert np.array_equal(canon_gpu(a), oracle.hash_equi(R, S)[1])


def test_equi_deterministic_positions(gj, ctx):
    R, S, _ = gen.pkfk(16, 200_000, seed=3)
    tR, tS = dev(R), dev(S)
    a = gj.join_materialize(ctx, tR, tS).clone()
    b = gj.join_materialize(ctx, tR, tS).clone()
    ctx2 = gj.Context(0)
    c = gj.join_materialize(ctx2, tR, tS)
    assert torch.equal(a, b) and torch.equal(a, c)


# ------------------------------------------------------------------ theta / NLJ

@pytest.mark.parametrize("op", OPS)
def test_theta_ragged_all_ops(gj, ctx, op):
    """Several R tiles + a ragged last tile; S spans several pipeline stages + tail."""
    R = gen.uniform_keys(4099, 300, 5, 0) - 150
    S = gen.uniform_keys(9001, 300, 5, 1) - 150
    check_theta(gj, ctx, R.astype(np.int32), S.astype(np.int32), op, eps=7 if op == "band" else 0)


@pytest.mark.parametrize("op", OPS)
def test_theta_int64(gj, ctx, op):
    rng = np.random.default_rng(11)
    R = rng.integers(-2**40, 2**40, 2100).astype(np.int64)
    S = np.concatenate([rng.integers(-2**40, 2**40, 3000), R[:500]]).astype(np.int64)
    check_theta(gj, ctx, R, S, op, eps=2**38 if op == "band" else 0)


@pytest.mark.parametrize("eps", [0, 1, 5, 2**31 - 1, 2**31, 2**32 - 1, 2**40])
def test_band_fast_and_exact_paths(gj, ctx, eps):
    """Full-range int32 keys: the 32-bit band trick is invalid here, the exact path must run."""
    rng = np.random.default_rng(eps % 1000)
    R = rng.integers(-2**31, 2**31, 2500, dtype=np.int64).astype(np.int32)
    S = rng.integers(-2**31, 2**31, 3000, dtype=np.int64).astype(np.int32)
    S[:100] = R[:100] + 1
    check_theta(gj, ctx, R, S, "band", eps)


def test_band_forced_slow_equals_fast(gj, ctx):
    R = gen.uniform_keys(5000, 1 << 20, 2, 0)
    S = gen.uniform_keys(7000, 1 << 20, 2, 1)
    a = check_theta(gj, ctx, R, S, "band", 300)
    ctx.set_option("force_slow_band", 1)
    assert check_theta(gj, ctx, R, S, "band", 300) == a


def test_theta_c1_lt_full(gj, ctx):
    """configs[0] theta R.a < S.b: count and all ~5e7 pairs."""
    R, S = gen.c1()
    check_theta(gj, ctx, R, S, "lt", 0, materialize=True)
    check_theta(gj, ctx, R, S, "eq", 0, materialize=True)


def test_theta_nlj_split_variants(gj, ctx):
    R = gen.uniform_keys(6000, 1000, 9, 0)
    S = gen.uniform_keys(50_000, 1000, 9, 1)
    for split in (1, 3, 25):
        ctx.set_option("nlj_split", split)
        check_theta(gj, ctx, R, S, "ge", 0, materialize=False)
        check_theta(gj, ctx, R, S, "band", 2, materialize=True)


def test_theta_unaligned_s(gj, ctx):
    R = gen.uniform_keys(3000, 500, 4, 0)
    S = gen.uniform_keys(5001, 500, 4, 1)
    tR, tS = dev(R), dev(S)
    tS1 = tS[1:]  # 4-byte offset: not 16-byte aligned
    n = gj.theta_join_count(ctx, tR, tS1, "le")
    assert n == oracle.theta_count_sorted(R, S[1:], "le")
    got = canon_gpu(gj.theta_join_materialize(ctx, tR, tS1, "le", 0, n))
    assert np.array_equal(got, oracle.nlj(R, S[1:], "le")[1])


@pytest.mark.timeout(1200)
def test_theta_c4_full_size_every_pair(gj, ctx):
    """configs[3] at full size: band join 2^20 x 2^24, eps = 53687, ~1.76e9 pairs.  The
    materialised set equals J exactly, checked on the device for EVERY pair:
    (1) |J| = O3; (2) every pair satisfies |R[r] - S[s]| <= eps; (3) the pairs per R
    row equal O3's per-row counts (O3r); (4) no pair occurs twice (device sort per
    R-row block, adjacent differences).  (2)+(3)+(4) => per row, the emitted S rows
    are exactly the matching ones."""
    R, S = gen.c4()
    tR, tS = dev(R), dev(S)
    eps = gen.C4_EPS
    n = gj.theta_join_count(ctx, tR, tS, "band", eps)
    assert n == oracle.theta_count_sorted(R, S, "band", eps)
    out = gj.theta_join_materialize(ctx, tR, tS, "band", eps, n)
    assert out.shape[0] == n
    per_row = torch.zeros(len(R), dtype=torch.int64, device="cuda")
    CH = 1 << 27
    for i in range(0, n, CH):
        blk = out[i:i + CH].long() & 0xFFFFFFFF
        r, s_ = blk[:, 0], blk[:, 1]
        assert bool((tR[r].long() - tS[s_].long()).abs().le(eps).all())
        per_row += torch.bincount(r, minlength=len(R))
        del blk, r, s_
    assert np.array_equal(per_row.cpu().numpy(), oracle.theta_count_per_row(R, S, "band", eps).astype(np.int64))
    NB = 16  # uniqueness: R-row blocks, each sorted on the device
    rr = out[:, 0].long() & 0xFFFFFFFF
    for b in range(NB):
        lo, hi = b * len(R) // NB, (b + 1) * len(R) // NB
        sel = (rr >= lo) & (rr < hi)
        p = out[sel].long() & 0xFFFFFFFF
        packed, _ = torch.sort((p[:, 0] << 32) | p[:, 1])
        assert bool((packed[1:] > packed[:-1]).all()), f"duplicate pair in R rows [{lo}, {hi})"
        del sel, p, packed


@pytest.mark.parametrize("op", ["band", "lt", "ne", "eq"])
def test_theta_deterministic_positions(gj, ctx, op):
    """SPEC.md:539 (acceptance 6, determinism): the theta write pass puts every pair at
    the same position run to run and across contexts -- byte-identical outputs."""
    R = gen.uniform_keys(20_011, 1 << 16, 12, 0)
    S = gen.uniform_keys(70_001, 1 << 16, 12, 1)
    tR, tS = dev(R), dev(S)
    eps = 40 if op == "band" else 0
    n = gj.theta_join_count(ctx, tR, tS, op, eps)
    a = gj.theta_join_materialize(ctx, tR, tS, op, eps, n).clone()
    b = gj.theta_join_materialize(ctx, tR, tS, op, eps, n).clone()
    ctx2 = gj.Context(0)
    c = gj.theta_join_materialize(ctx2, tR, tS, op, eps)
    ctx2.close()
    assert torch.equal(a, b) and torch.equal(a, c)


def test_theta_regions_test_fewer_pairs_than_they_output(gj, ctx):
    """SPEC.md:538 (acceptance 5): with a nonempty Green region, pairs_tested / |J| < 1 --
    configs[0]'s R.a < S.b compares only the Red cells and writes the Green ones."""
    R, S = gen.c1()
    n = gj.theta_join_count(ctx, dev(R), dev(S), "lt")
    tested, cross = ctx.theta_stats()
    assert cross > 0 and tested < n == oracle.theta_count_sorted(R, S, "lt")


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_unaligned_views(gj, ctx, dtype):
    """Inputs that are views at element (not 16-byte) offsets -- R[1:], S[3:], rid maps
    rid[1:] -- through every path whose loads are 1-D TMA bulk copies: the radix
    scatter (1, 2 passes), the table-free write pass with user rid maps (0 bits),
    and the region-matrix theta join (its range partition)."""
    rng = np.random.default_rng(17)
    R = rng.integers(-4000, 4000, 30_001).astype(dtype)
    S = rng.integers(-4000, 4000, 50_003).astype(dtype)
    rid = rng.permutation(40_000)[:30_001].astype(np.int32)
    tR, tS, trid = dev(R), dev(S), dev(rid)
    vR, vS, vrid = tR[1:], tS[3:], trid[1:]
    Rv, Sv, ridv = R[1:], S[3:], rid[1:]
    for bits in (0, 4, 12):
        ctx.set_option("part_bits", bits)
        n = gj.join_count(ctx, vR, vS)
        cn, cp = oracle.hash_equi(Rv, Sv)
        assert n == cn
        assert np.array_equal(canon_gpu(gj.join_materialize(ctx, vR, vS, n)), cp)
        relR = gj.Rel(vR, vrid)
        n2 = gj.join_count(ctx, relR, gj.Rel(vS, None, 5))
        got = canon_gpu(gj.join_materialize(ctx, relR, gj.Rel(vS, None, 5), n2))
        exp = np.stack([ridv[cp[:, 0]], cp[:, 1] + 5], 1).astype(np.uint32)
        assert n2 == cn and np.array_equal(got, exp[np.lexsort((exp[:, 1], exp[:, 0]))])
    ctx.set_option("part_bits", -1)
    for op, eps in (("band", 9), ("lt", 0)):
        n = gj.theta_join_count(ctx, vR, vS, op, eps)
        assert n == oracle.theta_count_sorted(Rv, Sv, op, eps)
        if op == "band":
            got = canon_gpu(gj.theta_join_materialize(ctx, vR, vS, op, eps, n))
            assert np.array_equal(got, oracle.band_materialize(Rv, Sv, eps)[1])


@pytest.mark.timeout(900)
def test_c5_shape_prefilter_then_join_one_gpu(gj, ctx):
    """configs[4] shape on ONE GPU (int64, 2^26 x 2^27; configs[4] itself is 2^31 x 2^32,
    sharded): range + Bloom two-sided pre-filter, then the hash join over the survivors'
    rid maps (the bench's N=1 step).  O8: J = {(m_j, j) : S row j a member}, every pair."""
    import gen.device as gd
    b, nR, nS, seed = 26, 1 << 26, 1 << 27, gen.BASE_SEED
    R = gd.c5_R(nR, seed, b=b)
    S = gd.c5_S(nS, seed, b=b)
    kR, rR, kS, rS = gj.prefilter(ctx, R, S, gj.RANGE | gj.BLOOM | gj.TWO_SIDED, "eq", 0, 8.0)
    assert kS.numel() < nS  # the filter removed the non-members it could
    R2, S2 = gj.Rel(kR, rR), gj.Rel(kS, rS)
    n = gj.join_count(ctx, R2, S2)
    mem = gen.c5_member_mask(nS, seed)
    m = np.where(mem, gen.uniform(nS, 1 << b, seed, 1).astype(np.int64), -1)
    cn, cp = oracle.pkfk_closed_form(m)
    assert n == cn
    assert np.array_equal(canon_gpu(gj.join_materialize(ctx, R2, S2, n)), cp)


# ------------------------------------------------------------------ pre-filter

@pytest.mark.parametrize("flags", [1, 2, 3, 7])
def test_prefilter_no_false_negatives(gj, ctx, flags):
    """J(prefilter(R), prefilter(S)) == J(R, S); exact semi-join survivors are kept."""
    rng = np.random.default_rng(flags)
    R = rng.integers(0, 200_000, 60_000).astype(np.int32)
    S = rng.integers(100_000, 400_000, 80_000).astype(np.int32)
    kR, rR, kS, rS = gj.prefilter(ctx, dev(R), dev(S), flags=flags)
    kR, rR, kS, rS = (t.cpu().numpy() for t in (kR, rR, kS, rS))
    assert np.array_equal(kR, R[rR]) and np.array_equal(kS, S[rS])
    assert np.all(np.diff(rR) > 0) and np.all(np.diff(rS) > 0)  # stable, original order
    keepR = set(np.nonzero(oracle.semijoin_exact(R, S))[0])
    keepS = set(np.nonzero(oracle.semijoin_exact(S, R))[0])
    assert keepR <= set(rR.tolist()) and keepS <= set(rS.tolist())
    c, p = oracle.hash_equi(kR, kS)
    p = np.stack([rR[p[:, 0]], rS[p[:, 1]]], 1).astype(np.uint32)
    p = p[np.lexsort((p[:, 1], p[:, 0]))]
    assert np.array_equal(p, oracle.hash_equi(R, S)[1])
    if flags & 2:
        # Bloom FPR within 2x of the blocked-filter formula at 8 bits/key: a 64-bit
        # block holds Poisson(64/8 = 8) keys, each setting 4 bits (with repetition), and
        # a probe tests 4 bits of one block, so FPR = E_j[(1 - (63/64)^(4j))^4] = 0.0326
        # (an upper bound: the filter never gets fewer than 8 bits per inserted key)
        import math
        p, fpr = math.exp(-8.0), 0.0
        for j in range(200):
            if j:
                p *= 8.0 / j
            fpr += p * (1 - (63 / 64) ** (4 * j)) ** 4
        lo, hi = max(R.min(), S.min()), min(R.max(), S.max())
        cand = np.ones(len(S), bool)
        cand[list(keepS)] = False  # true non-members ...
        if flags & 1:
            cand &= (S >= lo) & (S <= hi)  # ... that reach the Bloom stage
        fp = np.isin(np.nonzero(cand)[0], rS).sum()
        assert fp <= 2 * fpr * cand.sum(), (fp, cand.sum(), fpr)


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("flags", [8, 9, 12, 13])
def test_prefilter_exact_is_the_semijoin(gj, ctx, flags, dtype):
    """GJ_PF_EXACT (Alg.1 Setup's hash set of common keys): the survivors
    are EXACTLY the semi-joins S ⋉ R and (two-sided) R ⋉ S, in original order --
    incl. the extreme keys (the biased all-ones key lives outside the table)."""
    rng = np.random.default_rng(flags + (0 if dtype == np.int32 else 100))
    info = np.iinfo(dtype)
    R = rng.integers(-50_000, 50_000, 70_000).astype(dtype)
    S = rng.integers(0, 150_000, 90_000).astype(dtype)
    R[:4] = [info.max, info.min, -1, 0]
    S[:5] = [info.max, info.min, 7, info.max, 123_456_789 % 150_000]
    kR, rR, kS, rS = gj.prefilter(ctx, dev(R), dev(S), flags=flags)
    kR, rR, kS, rS = (t.cpu().numpy() for t in (kR, rR, kS, rS))
    assert np.array_equal(kR, R[rR]) and np.array_equal(kS, S[rS])
    assert np.array_equal(rS, np.nonzero(oracle.semijoin_exact(S, R))[0])
    if flags & 4:
        assert np.array_equal(rR, np.nonzero(oracle.semijoin_exact(R, S))[0])
    elif flags & 1:
        lo, hi = max(R.min(), S.min()), min(R.max(), S.max())
        assert np.array_equal(rR, np.nonzero((R >= lo) & (R <= hi))[0])
    else:
        assert np.array_equal(rR, np.arange(len(R)))


def test_prefilter_band_range(gj, ctx):
    R = gen.uniform_keys(20_000, 1 << 20, 6, 0)
    S = (gen.uniform_keys(20_000, 1 << 20, 6, 1) + (1 << 19)).astype(np.int32)
    kR, rR, kS, rS = gj.prefilter(ctx, dev(R), dev(S), flags=1, op="band", eps=1000)
    rR, rS = rR.cpu().numpy(), rS.cpu().numpy()
    assert set(np.nonzero(oracle.semijoin_band(R, S, 1000))[0]) <= set(rR.tolist())
    assert set(np.nonzero(oracle.semijoin_band(S, R, 1000))[0]) <= set(rS.tolist())


# ------------------------------------------------------------------ errors and host entry

def test_errors(gj, ctx):
    R, S = dev(gen.uniform_keys(100, 10, 1, 0)), dev(gen.uniform_keys(100, 10, 1, 1))
    n = gj.join_count(ctx, R, S)
    small = torch.empty((max(n - 1, 1), 2), dtype=torch.int32, device="cuda")
    with pytest.raises(gj.GJError) as e:
        gj.join_materialize(ctx, R, S, out=small)
    assert e.value.status == 3
    with pytest.raises(gj.GJError) as e:
        gj.join_count(ctx, R, S.to(torch.int64))
    assert e.value.status == 1
    with pytest.raises(gj.GJError):
        gj.prefilter(ctx, R, S, op="lt")


def test_join_host_e2e(gj, ctx):
    R, S, m = gen.pkfk(16, 300_000, seed=21)
    hR = torch.from_numpy(R).pin_memory()
    hS = torch.from_numpy(S).pin_memory()
    out = torch.empty((300_000, 2), dtype=torch.int32).pin_memory()
    n = gj.join_host(ctx, hR, hS, out)
    assert n == 300_000
    p = out.numpy().view(np.uint32)
    p = p[np.lexsort((p[:, 1], p[:, 0]))]
    assert np.array_equal(p, oracle.pkfk_closed_form(m)[1])


def test_join_host_batch_stream(gj, ctx):
    """join_host_batch: several independent joins (different sizes, duplicates, an empty
    one) through the two-stream pipeline, each vs the oracle; a short capacity raises
    GJ_ERANGE after the other batches completed."""
    cases = [gen.pkfk(14, 70_000, seed=31)[:2],
             (gen.uniform_keys(20_000, 3000, 5, 0), gen.uniform_keys(30_000, 3000, 5, 1)),
             (gen.uniform_keys(0, 10, 5, 0), gen.uniform_keys(100, 10, 5, 1)),
             gen.pkfk(12, 9_000, seed=32)[:2]]
    expect = [oracle.hash_equi(R, S) for R, S in cases]
    batches = [(torch.from_numpy(R).pin_memory(), torch.from_numpy(S).pin_memory(),
                torch.empty((max(c, 1), 2), dtype=torch.int32).pin_memory())
               for (R, S), (c, _) in zip(cases, expect)]
    ns = gj.join_host_batch(ctx, batches)
    for (c, pairs), n, (_, _, out) in zip(expect, ns, batches):
        assert n == c
        p = out.numpy()[:n].view(np.uint32)
        assert np.array_equal(p[np.lexsort((p[:, 1], p[:, 0]))], pairs)
    short = [batches[0], (batches[1][0], batches[1][1], torch.empty((5, 2), dtype=torch.int32).pin_memory()),
             batches[3]]
    with pytest.raises(gj.GJError, match="GJ_ERANGE"):
        gj.join_host_batch(ctx, short)


def test_torch_allocator_backs_the_workspace(gj):
    """gj_ctx_set_allocator with torch's caching allocator: the workspace comes from
    torch's pool (memory_allocated grows by the partition buffers) and results match."""
    R, S, m = gen.pkfk(18, 1 << 18, seed=13)
    tR, tS = dev(R), dev(S)
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    c = gj.Context(0, torch_allocator=True)
    n = gj.join_count(c, tR, tS)
    grown = torch.cuda.memory_allocated() - before
    assert n == 1 << 18 and grown >= 4 * (1 << 18) * 4  # at least the partitioned keys + rids
    assert np.array_equal(canon_gpu(gj.join_materialize(c, tR, tS, n)), oracle.pkfk_closed_form(m)[1])
    c.close()
    assert torch.cuda.memory_allocated() - before < grown  # released back to torch


def test_launch_accounting_and_profile(gj):
    c = gj.Context(0, profile=1)
    R, S = dev(gen.uniform_keys(50_000, 10_000, 1, 0)), dev(gen.uniform_keys(50_000, 10_000, 1, 1))
    c.reset_stats()
    gj.join_materialize(c, R, S)
    t = c.kernel_times()
    assert "hj_count" in t and "hj_write" in t and "part_scatter" in t
    assert c.launches() == sum(v[1] for v in t.values())
    c.close()


# ------------------------------------------------------------------ late materialisation

@pytest.mark.parametrize("shape", ["i32", "i64", "row16", "row12"])
def test_gather_payloads_matches_oracle(gj, ctx, shape):
    """gj_gather_payloads along the join's own pairs == oracle O10, for
    4-, 8-, 12- and 16-byte payload rows, with rid bases."""
    rng = np.random.default_rng(77)
    R = rng.integers(0, 5000, 20_000).astype(np.int32)
    S = rng.integers(0, 5000, 30_000).astype(np.int32)
    mk = {"i32": lambda n: rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32),
          "i64": lambda n: rng.integers(-2**62, 2**62, n, dtype=np.int64),
          "row16": lambda n: rng.integers(0, 2**31, (n, 4), dtype=np.int64).astype(np.int32),
          "row12": lambda n: rng.integers(0, 2**31, (n, 3), dtype=np.int64).astype(np.int32)}[shape]
    pR, pS = mk(len(R)), mk(len(S))
    tR = gj.Rel(dev(R), None, 100)
    tS = gj.Rel(dev(S), None, 2000)
    n = gj.join_count(ctx, tR, tS)
    pairs = gj.join_materialize(ctx, tR, tS, n)
    oR, oS = gj.gather_payloads(ctx, pairs, dev(pR), dev(pS), rid_base_R=100, rid_base_S=2000)
    eR, eS = oracle.gather_payloads(pairs.cpu().numpy(), pR, pS, 100, 2000)
    assert np.array_equal(oR.cpu().numpy(), eR) and np.array_equal(oS.cpu().numpy(), eS)
    oR, oS = gj.gather_payloads(ctx, pairs, None, dev(pS), rid_base_S=2000)
    assert oR is None and np.array_equal(oS.cpu().numpy(), eS)


# ------------------------------------------------------------------ Eq.8 result-size estimate

@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("bits", [-1, 0, 3, 11])
def test_join_stats_eq8_matches_oracle(gj, ctx, dtype, bits):
    """gj_join_stats: Eq.8's sum_i |R_i||S_i| over the join's own partitions
    equals oracle O9 at the partition bits the join used, and bounds |J|."""
    rng = np.random.default_rng(40 + bits)
    R = rng.integers(-2**40 if dtype == np.int64 else -50_000, 50_000, 30_000).astype(dtype)
    S = rng.integers(-50_000, 50_000, 45_000).astype(dtype)
    ctx.set_option("part_bits", bits)
    n = gj.join_count(ctx, dev(R), dev(S))
    e, B, units = ctx.join_stats()
    assert B == (bits if bits >= 0 else B) and units > 0
    assert e == oracle.eq8_rsize(R, S, B)
    assert e >= n == oracle.equi_count_hist(R, S)


# ------------------------------------------------------------------ theta region matrix (§4.2, Alg.3)

def _region_inputs(kind):
    rng = np.random.default_rng({"dups": 1, "wide": 2, "skew": 3, "extremes": 4, "equal": 5}[kind])
    if kind == "dups":        # small domain: many equal keys, buckets of width 1
        return (rng.integers(-40, 40, 9000).astype(np.int32), rng.integers(-40, 40, 20001).astype(np.int32))
    if kind == "wide":        # several R tiles, each spanning many buckets
        return (rng.integers(-10**6, 10**6, 9000).astype(np.int32), rng.integers(-10**6, 10**6, 30003).astype(np.int32))
    if kind == "skew":        # Zipf-like: most keys in few buckets, a long sparse tail
        z = lambda n: (np.floor(np.exp(rng.uniform(0, 14, n))) * rng.choice([-1, 1], n)).astype(np.int32)
        return z(7000), z(15000)
    if kind == "extremes":    # full int32 range incl. INT_MIN / INT_MAX
        R = rng.integers(-2**31, 2**31, 5000, dtype=np.int64).astype(np.int32)
        S = rng.integers(-2**31, 2**31, 8000, dtype=np.int64).astype(np.int32)
        R[:3] = [-2**31, 2**31 - 1, 0]
        S[:3] = [2**31 - 1, -2**31, 0]
        return R, S
    if kind == "equal":       # span 0: one bucket
        return np.full(3000, 7, np.int32), np.full(4000, 7, np.int32)
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["dups", "wide", "skew", "extremes", "equal"])
@pytest.mark.parametrize("op", OPS)
def test_theta_regions_all_ops(gj, ctx, kind, op):
    """Region-matrix mode (the default) against the oracle: counts always, pairs when
    the output is small enough to materialise."""
    R, S = _region_inputs(kind)
    eps = {"dups": 3, "wide": 1500, "skew": 20, "extremes": 2**30, "equal": 0}[kind] if op == "band" else 0
    ctx.set_option("theta_regions", 1)
    n = check_theta(gj, ctx, R, S, op, eps, materialize=False)
    if n <= 30_000_000:
        check_theta(gj, ctx, R, S, op, eps, materialize=True)


@pytest.mark.parametrize("eps", [0, 1, 7, 8, 9, 63, 4096, 100_000, 2**24])
def test_band_region_geometry(gj, ctx, eps):
    """The band's region-matrix path (bucket width ~eps/8: Green radius g, Red radius
    m, reading R17) over widths from 1 (eps < 8) to Green runs spanning many buckets:
    every pair vs the oracle, int32 keys over a 2^25 range with a dense cluster."""
    rng = np.random.default_rng(100 + eps % 97)
    R = np.concatenate([rng.integers(-2**24, 2**24, 6000), rng.integers(0, 3000, 1500)]).astype(np.int32)
    S = np.concatenate([rng.integers(-2**24, 2**24, 14000), rng.integers(0, 3000, 4000)]).astype(np.int32)
    ctx.set_option("theta_regions", 1)
    n = check_theta(gj, ctx, R, S, "band", eps, materialize=False)
    if n <= 40_000_000:
        check_theta(gj, ctx, R, S, "band", eps, materialize=True)


def test_band_write_unstaged_window(gj, ctx):
    """A 256-row batch of the band write pass whose S window exceeds the shared staging
    capacity (6144 rows: here all of S sits in a few buckets next to every R row)
    reads S from global memory -- same pairs as the oracle."""
    rng = np.random.default_rng(77)
    R = rng.integers(1000, 1040, 700).astype(np.int32)
    S = rng.integers(990, 1050, 20000).astype(np.int32)
    S[:5] = [-2**20, 2**20, 0, 5000, -5000]  # widen the span so the buckets are narrow
    ctx.set_option("theta_regions", 1)
    check_theta(gj, ctx, R, S, "band", 3, materialize=True)


def test_band_heavy_buckets_deterministic(gj, ctx):
    """Skewed band join: most R rows sit next to a hot S bucket whose Red rim exceeds
    the per-row limit, so those buckets' Red cells go to the tiled NLJ after the band
    kernels' pairs -- same pairs as the oracle, same positions on a rerun."""
    rng = np.random.default_rng(78)
    R = np.concatenate([rng.integers(1000, 1040, 3000), rng.integers(-2**20, 2**20, 500)]).astype(np.int32)
    S = np.concatenate([rng.integers(990, 1050, 30000), rng.integers(-2**20, 2**20, 2000)]).astype(np.int32)
    ctx.set_option("theta_regions", 1)
    n = check_theta(gj, ctx, R, S, "band", 3, materialize=True)
    nlj_pairs, cross = ctx.theta_stats()
    assert nlj_pairs > 0
    a = gj.theta_join_materialize(ctx, dev(R), dev(S), "band", 3, n).cpu().numpy()
    b = gj.theta_join_materialize(ctx, dev(R), dev(S), "band", 3, n).cpu().numpy()
    assert np.array_equal(a, b)


def test_band_heavy_buckets_int64_and_rid_maps(gj, ctx):
    """The heavy-bucket NLJ path with int64 keys (exact predicate, 2-key alignment)
    and with caller rid maps on both sides: pairs are the oracle's positional pairs
    mapped through the rid arrays."""
    rng = np.random.default_rng(79)
    R = np.concatenate([rng.integers(2**40, 2**40 + 64, 2500), rng.integers(-2**45, 2**45, 300)]).astype(np.int64)
    S = np.concatenate([rng.integers(2**40 - 8, 2**40 + 72, 20000), rng.integers(-2**45, 2**45, 900)]).astype(np.int64)
    rR = rng.permutation(10**6)[: len(R)].astype(np.uint32)
    rS = rng.permutation(10**6)[: len(S)].astype(np.uint32)
    ctx.set_option("theta_regions", 1)
    tR, tS = gj.Rel(dev(R), dev(rR.view(np.int32))), gj.Rel(dev(S), dev(rS.view(np.int32)))
    n = gj.theta_join_count(ctx, tR, tS, "band", 2)
    assert n == oracle.theta_count_sorted(R, S, "band", 2)
    assert ctx.theta_stats()[0] > 0
    out = canon_gpu(gj.theta_join_materialize(ctx, tR, tS, "band", 2, n))
    _, cp = oracle.nlj(R, S, "band", 2)
    cp = np.stack([rR[cp[:, 0]], rS[cp[:, 1]]], 1).astype(np.uint32)
    cp = cp[np.lexsort((cp[:, 1], cp[:, 0]))]
    assert np.array_equal(out.astype(np.uint32), cp)


@pytest.mark.parametrize("eps", [0, 5, 2**33])
def test_band_region_int64(gj, ctx, eps):
    """int64 keys take the band path with the exact 64-bit predicate."""
    rng = np.random.default_rng(55)
    R = rng.integers(-2**40, 2**40, 3000).astype(np.int64)
    S = np.concatenate([rng.integers(-2**40, 2**40, 9000), R[:2000] + rng.integers(-9, 9, 2000)]).astype(np.int64)
    ctx.set_option("theta_regions", 1)
    check_theta(gj, ctx, R, S, "band", eps, materialize=True)


@pytest.mark.parametrize("op", OPS)
def test_theta_plain_nlj_all_ops(gj, ctx, op):
    """The plain NLJ over all pairs (GJ_OPT_THETA_REGIONS = 0) stays exact."""
    ctx.set_option("theta_regions", 0)
    R = gen.uniform_keys(4099, 300, 5, 0) - 150
    S = gen.uniform_keys(9001, 300, 5, 1) - 150
    check_theta(gj, ctx, R.astype(np.int32), S.astype(np.int32), op, eps=7 if op == "band" else 0)


def test_theta_regions_match_plain_c4_shape(gj, ctx):
    """configs[3] shape at 2^18 x 2^20: region mode and the plain NLJ give the same count."""
    R = gen.uniform_keys(1 << 18, 1 << 30, 3, 0).astype(np.int32)
    S = gen.uniform_keys(1 << 20, 1 << 30, 3, 1).astype(np.int32)
    tR, tS = dev(R), dev(S)
    ctx.set_option("theta_regions", 1)
    a = gj.theta_join_count(ctx, tR, tS, "band", gen.C4_EPS)
    ctx.set_option("theta_regions", 0)
    b = gj.theta_join_count(ctx, tR, tS, "band", gen.C4_EPS)
    assert a == b == oracle.theta_count_sorted(R, S, "band", gen.C4_EPS)


@pytest.mark.parametrize("op", ["lt", "band", "ne"])
def test_theta_regions_with_rid_maps(gj, ctx, op):
    """Region mode carries caller rid maps (e.g. pre-filter survivors) through the range
    partitioning: pairs are the oracle's positional pairs mapped through the rid arrays."""
    rng = np.random.default_rng(9)
    R = rng.integers(-5000, 5000, 3000).astype(np.int32)
    S = rng.integers(-5000, 5000, 7001).astype(np.int32)
    rR = rng.permutation(10_000)[:3000].astype(np.int32)
    rS = rng.permutation(20_000)[:7001].astype(np.int32)
    eps = 25 if op == "band" else 0
    tR = gj.Rel(dev(R), dev(rR))
    tS = gj.Rel(dev(S), dev(rS))
    n = gj.theta_join_count(ctx, tR, tS, op, eps)
    cn, cp = oracle.nlj(R, S, op, eps)
    assert n == cn
    got = canon_gpu(gj.theta_join_materialize(ctx, tR, tS, op, eps, n))
    exp = np.stack([rR[cp[:, 0]], rS[cp[:, 1]]], 1).astype(np.uint32)
    exp = exp[np.lexsort((exp[:, 1], exp[:, 0]))]
    assert np.array_equal(got, exp)
