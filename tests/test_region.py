"""Region-matrix accounting (NEXT row f1; §4.2, Fig. 9, Alg.3) through the
library's own classifier gj_region_classify -- the function the theta path uses to
decide which cells the NLJ compares (Red), writes as cross products (Green) or skips
(White).  Host-only: no GPU.  Orientation: the paper's S table (abscissa x) is the
join's R, its T table (ordinate y) is S (reading R1)."""
import numpy as np
import pytest

import paper_1904_11201_b200 as gj

W, RED, GREEN = 0, 1, 2


def counts(c):
    return {"green": int((c == GREEN).sum()), "red": int((c == RED).sum()), "white": int((c == W).sum())}


@pytest.mark.parametrize("op", ["gt", "ge", "lt", "le"])
def test_k4_accounting_6_4_6(op):
    """SPEC.md:538 acceptance 5: op = GT with k = 4 -> Green 6, Red 4, White 6 (the
    k(k-1)/2 / k / k(k-1)/2 split of Fig. 9a); the same split for >=, <, <= (Fig. 9b)."""
    assert counts(gj.region_classify(op, 4)) == {"green": 6, "red": 4, "white": 6}


def test_paper_worked_cells():
    gt = gj.region_classify("gt", 4)
    assert gt[3, 1] == GREEN  # PAPER.md:301 "the A region coordinates are (3, 1) ... any tuple satisfies"
    assert gt[2, 2] == RED    # PAPER.md:301 "When the abscissa is equal to the ordinate ... send it to the GPU"
    assert gj.region_classify("lt", 4)[3, 1] == W  # SPEC.md:408 mirror of GT (Fig. 9b)
    ne = gj.region_classify("ne", 4)
    assert ne[1, 2] == GREEN and ne[2, 2] == RED   # SPEC.md:407 Fig. 9c
    assert counts(ne) == {"green": 12, "red": 4, "white": 0}
    eq = gj.region_classify("eq", 4)
    assert counts(eq) == {"green": 0, "red": 4, "white": 12}


def test_theta_map_rows_and_columns():
    """SPEC.md:416-418 (Alg.3 Map): for GT, k = 4, an x-side tuple in bucket 3 goes to
    (3,0),(3,1),(3,2),(3,3) = 3 Green + 1 Red; a y-side tuple in bucket 3 only to
    (3,3); for != every tuple reaches exactly k non-White cells."""
    gt = gj.region_classify("gt", 4)
    assert list(gt[3]) == [GREEN, GREEN, GREEN, RED]
    assert [x for x in range(4) if gt[x, 3] != W] == [3]
    ne = gj.region_classify("ne", 4)
    assert all((ne[x] != W).sum() == 4 and (ne[:, x] != W).sum() == 4 for x in range(4))


def test_band_neighbour_cells():
    b = gj.region_classify("band", 6, m=1)
    for x in range(6):
        for y in range(6):
            assert b[x, y] == (RED if abs(x - y) <= 1 else W)
    assert counts(gj.region_classify("band", 5, m=0)) == {"green": 0, "red": 5, "white": 20}


@pytest.mark.parametrize("op", ["eq", "ne", "lt", "le", "gt", "ge", "band"])
def test_classes_are_sound_by_brute_force(op):
    """Green soundness / White soundness: keys bucketed into k
    equal-width buckets ((key - lo) >> sh, reading R15); every pair in a
    Green cell satisfies the predicate, no pair in a White cell does -- checked
    pair by pair on random keys with dense bucket-boundary ties."""
    rng = np.random.default_rng(3)
    sh, k = 3, 8
    R = rng.integers(0, k << sh, 400)
    S = rng.integers(0, k << sh, 500)
    eps = 11
    m = -(-eps // (1 << sh))
    g = (eps + 1) // (1 << sh) - 1
    cls = gj.region_classify(op, k, m, g)
    pred = {"eq": np.equal, "ne": np.not_equal, "lt": np.less, "le": np.less_equal, "gt": np.greater,
            "ge": np.greater_equal, "band": lambda a, b: np.abs(a - b) <= eps}[op]
    P = pred(R[:, None], S[None, :])
    cell = cls[(R >> sh)[:, None], (S >> sh)[None, :]]
    assert P[cell == GREEN].all()
    assert not P[cell == W].any()


def test_band_green_cells():
    """Band Green cells: with width w the farthest pair of cell (x, y) is
    (|x-y| + 1) w - 1 apart, so |x - y| <= g = floor((eps + 1) / w) - 1 is all-match;
    the nearest is (|x-y| - 1) w + 1, so |x - y| <= m = ceil(eps / w) can match.
    configs[3]'s geometry (w = 4096, eps = 53687): g = 12, m = 14."""
    w, eps = 4096, 53687
    g, m = (eps + 1) // w - 1, -(-eps // w)
    assert (g, m) == (12, 14)
    b = gj.region_classify("band", 40, m=m, g=g)
    assert list(b[20, 20 - 14:20 + 15]) == [RED, RED] + [GREEN] * 25 + [RED, RED]
    assert b[20, 5] == W and b[20, 35] == W
    # extreme pairs at the cell edges, brute force over every key of two buckets
    for d, cls in ((12, GREEN), (13, RED), (14, RED), (15, W)):
        lo_r, lo_s = 0, d * w
        dmax = (lo_s + w - 1) - lo_r
        dmin = lo_s - (lo_r + w - 1)
        assert (cls == GREEN) == (dmax <= eps)
        assert (cls == W) == (dmin > eps)
    assert counts(gj.region_classify("band", 6, m=1, g=0)) == {"green": 6, "red": 10, "white": 20}


def test_errors():
    with pytest.raises(gj.GJError):
        gj.region_classify("gt", 0)
