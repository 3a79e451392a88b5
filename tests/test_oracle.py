"""Pins for the CPU oracle (oracle/) against things other than itself.

* hand-worked golden examples (tests/golden/*.json, each with its citation);
* SPEC.md worked examples;
* agreement between INDEPENDENT algorithms (O1 double loop, O2 hash multimap,
  O3 sort + binary search, O4 sorted range enumeration, O5 sort-merge histogram,
  O6 hash-set semi-join, O8 generator closed form) on thousands of tiny random
  instances with forced duplicates and INT32/INT64 extremes -- a dropped term, a
  wrong sign, an off-by-one bound or a swapped operand in any one of them breaks
  the agreement;
* closed-form invariants (LT+GE = EQ+NE = nR*nS, operand-swap symmetry, band
  monotonicity, BAND(0) = EQ) and statistical expectations of the generators.
"""
import glob
import json
import os

import numpy as np
import pytest

import gen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
OPS = ["eq", "ne", "lt", "le", "gt", "ge", "band"]
SWAP = {"eq": "eq", "ne": "ne", "lt": "gt", "le": "ge", "gt": "lt", "ge": "le", "band": "band"}


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.mark.parametrize("name", ["e1_small_mixed.json", "e2_int32_extremes.json", "e3_int64_extremes.json"])
def test_golden_hand_worked(name):
    g = _load(name)
    dt = np.int32 if g["dtype"] == "int32" else np.int64
    R, S = np.array(g["R"], dtype=dt), np.array(g["S"], dtype=dt)
    for c in g["cases"]:
        op, eps = c["op"], c["eps"]
        cnt, pairs = oracle.nlj(R, S, op, eps)
        assert cnt == c["count"], (name, c)
        assert oracle.theta_count_sorted(R, S, op, eps) == c["count"], (name, c)
        if "pairs" in c:
            assert pairs.tolist() == c["pairs"], (name, c)
        if op == "eq":
            hc, hp = oracle.hash_equi(R, S)
            assert hc == c["count"] and oracle.equi_count_hist(R, S) == c["count"]
            if "pairs" in c:
                assert hp.tolist() == c["pairs"]
        if op == "band":
            bc, bp = oracle.band_materialize(R, S, eps)
            assert bc == c["count"]
            if "pairs" in c:
                assert bp.tolist() == c["pairs"]


def test_spec_examples():
    g = _load("spec_examples.json")
    for c in g["cases"]:
        R, S = np.array(c["R"], dtype=np.int32), np.array(c["S"], dtype=np.int32)
        cnt, pairs = oracle.nlj(R, S, c["op"], c["eps"])
        assert cnt == c["count"], c["cite"]
        assert pairs.tolist() == c["pairs"], c["cite"]
        if c["op"] == "eq":
            assert oracle.hash_equi(R, S)[1].tolist() == c["pairs"]


def _random_instance(rng, dtype):
    nR, nS = int(rng.integers(0, 40)), int(rng.integers(0, 40))
    info = np.iinfo(dtype)
    kind = rng.integers(0, 4)
    if kind == 0:      # tiny domain: forces duplicates on both sides
        R, S = rng.integers(-3, 4, nR), rng.integers(-3, 4, nS)
    elif kind == 1:    # extremes mixed in
        pool = np.array([info.min, info.min + 1, -1, 0, 1, info.max - 1, info.max], dtype=np.int64)
        R, S = rng.choice(pool, nR), rng.choice(pool, nS)
    elif kind == 2:    # full range
        R = rng.integers(info.min, info.max, nR, dtype=np.int64, endpoint=True)
        S = rng.integers(info.min, info.max, nS, dtype=np.int64, endpoint=True)
    else:              # medium domain
        R, S = rng.integers(-50, 50, nR), rng.integers(-50, 50, nS)
    return R.astype(dtype), S.astype(dtype)


EPS_LIST = [0, 1, 2, 2**31 - 1, 2**31, 2**32 - 2, 2**32 - 1, 2**63 - 1, 2**63, 2**64 - 1]


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_independent_algorithms_agree(dtype):
    rng = np.random.default_rng(20190426 + (dtype == np.int64))
    for trial in range(2500):
        R, S = _random_instance(rng, dtype)
        op = OPS[trial % len(OPS)]
        eps = int(EPS_LIST[rng.integers(0, len(EPS_LIST))]) if op == "band" else 0
        c1, p1 = oracle.nlj(R, S, op, eps)
        assert oracle.theta_count_sorted(R, S, op, eps) == c1, (R, S, op, eps)
        if op == "eq":
            c2, p2 = oracle.hash_equi(R, S)
            assert c2 == c1 and np.array_equal(p1, p2)
            assert oracle.equi_count_hist(R, S) == c1
        if op == "band":
            c4, p4 = oracle.band_materialize(R, S, eps)
            assert c4 == c1 and np.array_equal(p1, p4), (R, S, eps)
        # operand swap: R OP S  <=>  S SWAP(OP) R, pairs transposed
        cs, ps = oracle.nlj(S, R, SWAP[op], eps)
        assert cs == c1
        assert np.array_equal(_canon(ps[:, ::-1]), p1)


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_theta_count_per_row_matches_double_loop(dtype):
    """O3r: per-R-row counts equal the per-row tallies of O1's double loop, and sum to O3."""
    rng = np.random.default_rng(31 + (dtype == np.int64))
    for trial in range(700):
        R, S = _random_instance(rng, dtype)
        op = OPS[trial % len(OPS)]
        eps = int(EPS_LIST[rng.integers(0, len(EPS_LIST))]) if op == "band" else 0
        c, p = oracle.nlj(R, S, op, eps)
        per = oracle.theta_count_per_row(R, S, op, eps)
        assert np.array_equal(per, np.bincount(p[:, 0].astype(np.int64), minlength=len(R)).astype(np.uint64))
        assert int(per.sum()) == oracle.theta_count_sorted(R, S, op, eps) == c


def _canon(p):
    p = np.asarray(p).reshape(-1, 2)
    return p[np.lexsort((p[:, 1], p[:, 0]))]


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_sliced_oracle_equals_o2(dtype):
    """O7 (O2 per key slice, T threads) equals O2 -- the slices partition J by key
    (equal keys share a slice): random tiny instances with duplicates and extremes,
    T in {1, 2, 3, 8, all cores}, and rid bases."""
    rng = np.random.default_rng(77 + (dtype == np.int64))
    for trial in range(300):
        R, S = _random_instance(rng, dtype)
        T = [1, 2, 3, 8, 0][trial % 5]
        c2, p2 = oracle.hash_equi(R, S, rid_base_R=5, rid_base_S=9)
        c7, p7 = oracle.hash_equi_sliced(R, S, T, rid_base_R=5, rid_base_S=9)
        assert c7 == c2 and np.array_equal(p7, p2), (R, S, T)
    R, S, m = gen.pkfk(14, 50_000, seed=3)
    assert np.array_equal(oracle.hash_equi_sliced(R, S, 6)[1], oracle.pkfk_closed_form(m)[1])


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_closed_form_invariants(dtype):
    rng = np.random.default_rng(7)
    for _ in range(200):
        R, S = _random_instance(rng, dtype)
        n = len(R) * len(S)
        c = {op: oracle.theta_count_sorted(R, S, op) for op in OPS[:6]}
        assert c["lt"] + c["ge"] == n
        assert c["le"] + c["gt"] == n
        assert c["eq"] + c["ne"] == n
        assert c["lt"] + c["eq"] + c["gt"] == n
        assert oracle.theta_count_sorted(R, S, "band", 0) == c["eq"]
        # BAND monotone in eps and saturates at the full cross product
        prev = -1
        for eps in sorted(EPS_LIST):
            b = oracle.theta_count_sorted(R, S, "band", eps)
            assert b >= prev
            prev = b
        assert oracle.theta_count_sorted(R, S, "band", 2**64 - 1) == n


def test_equi_count_is_histogram_product():
    """North star invariant: |J_=| = sum_k cntR(k)*cntS(k), here with numpy's unique."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        R = rng.integers(0, 200, rng.integers(0, 3000)).astype(np.int32)
        S = rng.integers(0, 200, rng.integers(0, 3000)).astype(np.int32)
        kr, cr = np.unique(R, return_counts=True)
        ks, cs = np.unique(S, return_counts=True)
        common, ir, is_ = np.intersect1d(kr, ks, return_indices=True)
        expect = int(np.sum(cr[ir].astype(np.int64) * cs[is_].astype(np.int64)))
        assert oracle.equi_count_hist(R, S) == expect
        assert oracle.hash_equi(R, S)[0] == expect


def test_pkfk_closed_form_matches_hash_oracle():
    R, S, m = gen.pkfk(14, 20_000, seed=11)
    c8, p8 = oracle.pkfk_closed_form(m)
    c2, p2 = oracle.hash_equi(R, S)
    assert c8 == c2 == 20_000
    assert np.array_equal(p8, p2)


def test_c5_closed_form_matches_hash_oracle():
    R, S, m = gen.c5(1 << 12, 1 << 14, seed=5)
    # restrict R to the first 2^12 rows: members drawn outside are non-matches
    c8, p8 = oracle.pkfk_closed_form(m, r_rows=(0, 1 << 12))
    c2, p2 = oracle.hash_equi(R, S)
    assert c8 == c2
    assert np.array_equal(p8, p2)


def test_semijoin_exact_is_projection_of_join():
    rng = np.random.default_rng(9)
    for _ in range(30):
        R = rng.integers(0, 300, 800).astype(np.int32)
        S = rng.integers(100, 600, 900).astype(np.int32)
        _, pairs = oracle.hash_equi(R, S)
        keepR = np.zeros(len(R), bool)
        keepS = np.zeros(len(S), bool)
        keepR[pairs[:, 0]] = True
        keepS[pairs[:, 1]] = True
        assert np.array_equal(oracle.semijoin_exact(R, S), keepR)
        assert np.array_equal(oracle.semijoin_exact(S, R), keepS)
        eps = int(rng.integers(0, 5))
        _, bp = oracle.band_materialize(R, S, eps)
        kb = np.zeros(len(R), bool)
        kb[bp[:, 0]] = True
        assert np.array_equal(oracle.semijoin_band(R, S, eps), kb)


def test_c1_statistics():
    """configs[0]: E[EQ] = n^2/D = 1e4; E[LT] = (1e8 - E[EQ])/2."""
    R, S = gen.c1()
    eq = oracle.theta_count_sorted(R, S, "eq")
    lt = oracle.theta_count_sorted(R, S, "lt")
    gt = oracle.theta_count_sorted(R, S, "gt")
    assert abs(eq - 1e4) < 0.08e4
    assert abs(lt - (1e8 - eq) / 2) < 0.01 * 1e8
    assert lt + gt + eq == 10**8


def test_c4_statistics_small():
    """Band selectivity ((2eps+1)D - eps(eps+1))/D^2 for uniform keys."""
    D, eps = 1 << 30, gen.C4_EPS
    R, S = gen.c4(nR=1 << 12, nS=1 << 16)
    c = oracle.theta_count_sorted(R, S, "band", eps)
    p = ((2 * eps + 1) * D - eps * (eps + 1)) / D**2
    expect = p * (1 << 12) * (1 << 16)
    assert abs(c - expect) < 5 * np.sqrt(expect) + 0.02 * expect



# ---- O9: Eq.8 result-size estimate

def test_eq8_spec_worked_example_1250():
    """SPEC.md:322 (hand evaluation of Eq.8): k = 2, |S| = |T| = 100, 50 + 50 tuples
    survive the filter, split evenly -> beta = gamma = 0.5, omega = lambda = (0.5, 0.5),
    R_size = 0.5 * 0.5 * 100 * 100 * (0.25 + 0.25) = 1250."""
    assert oracle.eq8_from_counts([25, 25], [25, 25], 100, 100) == 1250


def test_eq8_single_reducer_is_the_cartesian_product():
    """SPEC.md:323 / PAPER.md:197: one Reducer holding everything, no filtering ->
    R_size = |S| |T| (the Cartesian allocation the paper starts from)."""
    assert oracle.eq8_from_counts([70], [30], 70, 30) == 70 * 30
    R, S = gen.c1(n=500, D=50)
    assert oracle.eq8_rsize(R, S, 0) == len(R) * len(S)


def test_eq8_degenerate_and_filter_ratios():
    """|S| = 0 -> 0; a filter keeping beta of S scales the bound by beta:
    with one Reducer, R_size = (beta |S|) (gamma |T|)."""
    assert oracle.eq8_from_counts([0, 0], [5, 5], 0, 10) == 0
    assert oracle.eq8_from_counts([10], [4], 40, 16) == 10 * 4
    # uneven split, hand-evaluated: s = (30, 10), t = (5, 15), |S| = 80, |T| = 40:
    # beta = 1/2, gamma = 1/2, omega = (3/4, 1/4), lambda = (1/4, 3/4)
    # R_size = 1/2 * 1/2 * 80 * 40 * (3/16 + 3/16) = 800 * 3/8 = 300
    assert oracle.eq8_from_counts([30, 10], [5, 15], 80, 40) == 300


def test_eq8_bounds_random_8_reducer_splits():
    """for 200 random instances split over 8 Reducers by an arbitrary map
    that keeps equal keys together, R_size >= the actual join count (O5): each Reducer's
    Cartesian product contains its share of the join."""
    rng = np.random.default_rng(8)
    for _ in range(200):
        R = rng.integers(0, 60, rng.integers(1, 300)).astype(np.int32)
        S = rng.integers(0, 60, rng.integers(1, 300)).astype(np.int32)
        table = rng.integers(0, 8, 60)  # an arbitrary key -> Reducer map
        e = oracle.eq8_rsize(R, S, 3, reducer_of=lambda K: table[np.asarray(K)])
        # brute force: per Reducer, count tuples of each side by looping
        brute = sum(sum(1 for r in R if table[r] == i) * sum(1 for s in S if table[s] == i) for i in range(8))
        assert e == brute >= oracle.equi_count_hist(R, S)


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_eq8_bounds_the_join_and_shrinks_with_more_reducers(dtype):
    """At the product's partition map: sum_i |S_i||T_i| >= |J| (equal keys share a
    Reducer), and splitting a Reducer never increases it ((a+b)(c+d) >= ac+bd)."""
    rng = np.random.default_rng(5)
    R = rng.integers(-3000, 3000, 4000).astype(dtype)
    S = rng.integers(-3000, 3000, 5000).astype(dtype)
    j = oracle.equi_count_hist(R, S)
    prev = None
    for b in range(0, 17):
        e = oracle.eq8_rsize(R, S, b)
        assert e >= j
        if prev is not None:
            assert e <= prev
        prev = e


# ---- O10: late materialisation

def test_gather_of_the_key_columns_reproduces_matching_keys():
    """Gathering the KEY columns along the join's pairs gives, pair by pair, keys that
    satisfy the predicate: equal for the equi join, ordered for <."""
    R, S = gen.c1(n=400, D=60)
    _, p = oracle.hash_equi(R, S)
    kR, kS = oracle.gather_payloads(p, R, S)
    assert len(kR) == len(p) and np.array_equal(kR, kS)
    _, q = oracle.nlj(R, S, "lt")
    kR, kS = oracle.gather_payloads(q, R, S)
    assert np.all(kR < kS)
    # rid bases: a shard whose rids start at 1000
    _, p2 = oracle.hash_equi(R, S, rid_base_R=1000, rid_base_S=7)
    kR2, kS2 = oracle.gather_payloads(p2, R, S, rid_base_R=1000, rid_base_S=7)
    assert np.array_equal(kR2, kS2) and len(kR2) == len(p)
