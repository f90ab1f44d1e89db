"""Pins for oracle/pruned.py and oracle/brute.py."""
import numpy as np
import pytest

import synth
from oracle import actions as A
from oracle import brute as BR
from oracle import corun as CR
from oracle import env as EV
from oracle import pruned as PR
from oracle import space as SP

S10 = tuple(range(10, 100, 10))


@pytest.mark.parametrize("W,cmax,S", [(3, 1, (50,)), (4, 2, (25, 50, 75)),
                                      (5, 3, (25, 50, 75)), (6, 3, S10), (5, 4, (25, 50, 75)),
                                      (7, 4, (50,))])
def test_pruned_equals_explicit(W, cmax, S):
    sp = SP.build_space(W, cmax, S)
    tab = EV.Tables(sp)
    rng = np.random.default_rng(11)
    for k in range(60):
        hi = [1, 2, 3, 1 << 16][k % 4]       # heavy integer ties
        Fv = int(rng.integers(-3, 3))
        FcL = [int(x) for x in rng.integers(-hi, hi + 1, sp.L)]
        FcJ = [[int(x) for x in r] for r in rng.integers(-hi, hi + 1, (W, sp.T))]
        sched = int(rng.integers(0, (1 << W) - 1))
        assert PR.greedy_pruned(sp, Fv, FcL, FcJ, sched) == \
            EV.greedy_explicit(tab, Fv, FcL, FcJ, sched)


def _window(pool, W, seed):
    return [int(x) for x in synth.make_windows(pool, 1, W, step=seed)[0]]


@pytest.mark.parametrize("W,cmax,S,mig", [(3, 2, (25, 50, 75), True), (4, 2, (25, 50, 75), True),
                                          (4, 3, (25, 50, 75), True), (5, 4, (50,), True),
                                          (5, 3, (25, 50, 75), False)])
def test_three_algorithms_agree_small(W, cmax, S, mig):
    pool = synth.make_pool(27)
    sp = SP.build_space(W, cmax, S, mig)
    for seed in range(4):
        win = _window(pool, W, seed)
        lit = BR.literal_opt(sp, win, pool)
        rgs = BR.rgs_opt(sp, win, pool)
        dp = BR.dp_opt(sp, win, pool)
        assert lit == rgs == dp


def test_vectorised_block_best_equals_loops():
    pool = synth.make_pool(27)
    sp = SP.build_space(6, 4, S10)
    win = _window(pool, 6, 3)
    best = BR.all_block_best(sp, win, pool)
    import itertools
    for C in range(1, 5):
        for blk in itertools.combinations(range(6), C):
            assert best[A.group_mask(blk)] == BR.block_best_literal(sp, win, blk, pool)


def test_rgs_equals_dp_with_heavy_ties():
    # a pool of identical jobs makes many partitions tie: the block-order rule decides
    from types import SimpleNamespace
    pool = SimpleNamespace(solo_ticks=np.array([1000, 1000, 2000], np.int64),
                           compute_pm=np.array([100, 100, 100], np.int16),
                           memory_pm=np.array([100, 100, 100], np.int16))
    sp = SP.build_space(7, 3, (25, 50, 75))
    rng = np.random.default_rng(4)
    for _ in range(5):
        win = [int(x) for x in rng.integers(0, 3, 7)]
        assert BR.rgs_opt(sp, win, pool) == BR.dp_opt(sp, win, pool)


def test_table_v_windows_invariants():
    # Q1..Q12 (Table V) at W=12, Cmax=4: feasibility, partition, time sharing bound
    pool = synth.make_pool(27)
    sp = SP.build_space(12, 4, S10)
    wins = synth.table_v_windows(pool)
    for q in (0, 5):
        win = [int(x) for x in wins[q]]
        res = BR.dp_opt(sp, win, pool)
        assert res["cost"] <= res["solo"]
        seen = 0
        for b in res["blocks"]:
            assert seen & b == 0 and 1 <= bin(b).count("1") <= 4
            seen |= b
        assert seen == (1 << 12) - 1
        off = A.offsets(sp)
        for k, b in enumerate(res["blocks"]):
            l, g, s = A.decode(sp, res["block_action"][k], off)
            assert A.group_mask(g) == b
            _, cr, solo = CR.corun(sp.layouts[l], CR.assign(sp.layouts[l], g, s, win), pool)
            assert cr <= solo                     # P:122 constraint per job set
        # RGS is a restricted growth string
        m = -1
        for x in res["rgs"]:
            assert x <= m + 1
            m = max(m, x)


def test_cmax1_is_time_sharing_and_monotone():
    pool = synth.make_pool(27)
    win = _window(pool, 8, 1)
    costs = []
    for cmax in (1, 2, 3):
        sp = SP.build_space(8, cmax, (25, 50, 75))
        costs.append(BR.dp_opt(sp, win, pool)["cost"])
    assert costs[0] == sum(int(pool.solo_ticks[j]) for j in win)   # ratio exactly 1.0
    assert costs[0] >= costs[1] >= costs[2]                         # Fig. 10 trend
    # restricted baselines are never better than MIG+MPS
    full = BR.dp_opt(SP.build_space(8, 3, S10), win, pool)["cost"]
    mps = BR.dp_opt(SP.build_space(8, 3, S10, mig=False), win, pool)["cost"]
    assert full <= mps


def test_restricted_baseline_spaces_table_v():
    # The compared methods of P:245-248 as search spaces (synth.BASELINE_SPACES): MIG Only
    # (C = 2, Fig. 2's two options), MPS Only (C <= 4), MIG+MPS (C <= 4).  The MIG-only table
    # entries must be valid hierarchical partitions of the oracle's own enumeration; each
    # baseline's optimum is a minimum over a subset of the full space's choices, so it is never
    # better than MIG+MPS, and never worse than time sharing (ratio >= 1).
    sc, lay = synth.BASELINE_SPACES["mig_only"]
    L = SP.select_layouts(lay, sc.cmax, sc.shares)
    assert [len(l.slots) for l in L] == [1, 2, 2] and not L[0].mig and L[1].mig and L[2].mig
    assert len({s.dom for s in L[2].slots}) == 2 and len({s.dom for s in L[1].slots}) == 1
    with pytest.raises(ValueError):
        SP.select_layouts([[(400, 8, 0), (300, 8, 1)]], 2, sc.shares)  # 16 memory eighths
    pool = synth.make_pool(27)
    Q = synth.table_v_windows(pool)[:6]
    cost = {}
    for name, (scfg, lay) in synth.BASELINE_SPACES.items():
        L = SP.select_layouts(lay, scfg.cmax, scfg.shares) if lay else None
        sp = SP.build_space(scfg.window, scfg.cmax, scfg.shares, scfg.mig, layouts=L)
        cost[name] = [BR.dp_opt(sp, [int(x) for x in w], pool) for w in Q]
    for i in range(len(Q)):
        solo = cost["mig_mps"][i]["solo"]
        assert all(cost[n][i]["solo"] == solo for n in cost)
        assert cost["mig_mps"][i]["cost"] <= cost["mps_only"][i]["cost"] <= solo
        assert cost["mig_mps"][i]["cost"] <= cost["mig_only"][i]["cost"] <= solo
        # MIG-only job sets have at most 2 members
        rgs = cost["mig_only"][i]["rgs"]
        assert max(rgs.count(b) for b in set(rgs)) <= 2
