"""Pins for oracle/actions.py -- against itertools enumeration orders (brute force)."""
import itertools
import random

import pytest

from oracle import actions as A
from oracle import space as SP

S10 = tuple(range(10, 100, 10))


@pytest.mark.parametrize("W,C", [(4, 1), (4, 2), (7, 3), (9, 4), (6, 6)])
def test_rank_comb_matches_itertools(W, C):
    for r, g in enumerate(itertools.combinations(range(W), C)):
        assert A.rank_comb(g, W) == r
        assert A.unrank_comb(r, W, C) == g


@pytest.mark.parametrize("C", [1, 2, 3, 4])
def test_lehmer_matches_itertools(C):
    for r, s in enumerate(itertools.permutations(range(C))):
        assert A.lehmer(s) == r
        assert A.unlehmer(r, C) == s


def test_decode_round_trip_config1_all():
    sp = SP.build_space(4, 2, (25, 50, 75))
    off = A.offsets(sp)
    seen = set()
    for idx in range(A.n_actions(sp)):
        l, g, s = A.decode(sp, idx, off)
        assert len(g) == sp.layouts[l].C == len(s)
        assert A.action_index(sp, l, g, s, off) == idx
        seen.add((l, g, s))
    assert len(seen) == 92


def test_index_order_is_layout_then_group_then_perm():
    # brute-force enumeration order: layouts in order, groups lexicographic, perms lexicographic
    sp = SP.build_space(5, 3, (25, 50, 75))
    idx = 0
    for l, lay in enumerate(sp.layouts):
        for g in itertools.combinations(range(5), lay.C):
            for s in itertools.permutations(range(lay.C)):
                assert A.action_index(sp, l, g, s) == idx
                idx += 1
    assert idx == A.n_actions(sp)


def test_decode_round_trip_config4_random():
    sp = SP.build_space(64, 4, S10)
    off = A.offsets(sp)
    rng = random.Random(1)
    N = A.n_actions(sp)
    for _ in range(2000):
        idx = rng.randrange(N)
        l, g, s = A.decode(sp, idx, off)
        assert list(g) == sorted(set(g)) and max(g) < 64
        assert A.action_index(sp, l, g, s, off) == idx


@pytest.mark.parametrize("W,cmax,S", [(4, 2, (25, 50, 75)), (6, 3, (25, 50, 75)),
                                      (5, 4, (50,))])
def test_kth_valid_matches_filtered_list(W, cmax, S):
    sp = SP.build_space(W, cmax, S)
    off = A.offsets(sp)
    allv = [A.decode(sp, i, off) for i in range(A.n_actions(sp))]
    for sched in range(1 << W):
        valid = [i for i, (l, g, s) in enumerate(allv) if A.group_mask(g) & sched == 0]
        if sched == (1 << W) - 1:
            assert A.n_valid(sp, sched) == 0
            continue
        assert A.n_valid(sp, sched) == len(valid)
        for k in range(len(valid)):
            assert A.kth_valid(sp, sched, k, off) == valid[k]


def test_explore_k_range():
    for nv in (1, 7, 92, 191312, 4817494208):
        assert A.explore_k(0, nv) == 0
        assert A.explore_k((1 << 64) - 1, nv) == nv - 1
