"""gj_dist_plan -- the host-side receive plan of the multi-GPU equi-join shuffle
(the B200 analogue of the Hadoop shuffle by key) --
checked without a GPU or NCCL by simulating the scatter it drives for 1..8 ranks,
including empty runs, empty ranks and the >= 2^32 guard."""
import numpy as np
import pytest

import paper_1904_11201_b200 as gj
from tests.test_dist_gloo import _simulate


@pytest.mark.parametrize("G,lbits,seed", [(1, 0, 1), (2, 0, 2), (2, 3, 3), (4, 1, 4), (8, 0, 5), (8, 2, 6)])
def test_plan_places_every_tuple_once_in_digit_sender_order(G, lbits, seed):
    rng = np.random.default_rng(seed)
    L = 1 << lbits
    M = rng.integers(0, 12, (G, G, L)).astype(np.uint64)
    M[rng.random((G, G, L)) < 0.3] = 0  # empty runs
    plans = [gj.dist_plan(M, r, lbits) for r in range(G)]
    adjs = [p[0] for p in plans]
    for me in range(G):
        assert _simulate(M, adjs, me, plans[me][1], plans[me][2], lbits)


def test_plan_empty_rank_and_overflow_guard():
    M = np.zeros((2, 2, 1), dtype=np.uint64)
    adj, seg, need = gj.dist_plan(M, 1, 0)
    assert list(need) == [0, 0] and list(seg) == [0, 0]
    M[0, 1, 0] = 1 << 31
    M[1, 1, 0] = 1 << 31
    with pytest.raises(gj.GJError):
        gj.dist_plan(M, 0, 0)
    with pytest.raises(gj.GJError):
        gj.dist_plan(np.zeros((2, 2, 1), dtype=np.uint64), 2, 0)  # rank out of range
