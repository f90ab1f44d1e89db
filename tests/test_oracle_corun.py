"""Pins for oracle/corun.py -- time-sharing invariant, class rule, hand-computed cases."""
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import corun as CR
from oracle import space as SP
import synth


def _pool(T, c, m):
    return SimpleNamespace(solo_ticks=np.array(T, np.int64), compute_pm=np.array(c, np.int16),
                           memory_pm=np.array(m, np.int16))


@pytest.mark.parametrize("P", [27, 256])
def test_time_sharing_is_exactly_one(P):
    # a job alone on the whole GPU (MIG off) is the time-sharing baseline
    pool = synth.make_pool(P)
    sp = SP.build_space(4, 2, (25, 50, 75))
    whole = sp.layouts[0]
    assert not whole.mig and whole.C == 1
    for p in range(pool.n):
        r, cr, solo = CR.reward(whole, (0,), (0,), [p], pool)
        assert cr == solo == int(pool.solo_ticks[p])
        assert r == 0.0


@pytest.mark.parametrize("P", [27, 256])
def test_class_rule_reproduces_pool(P):
    # P:189/P:207 class rule applied to the co-run model reproduces Table IV's classes
    pool = synth.make_pool(P)
    for p in range(pool.n):
        got = CR.app_class(int(pool.solo_ticks[p]), int(pool.compute_pm[p]),
                           int(pool.memory_pm[p]))
        assert got == int(pool.classes[p]), pool.names[p]


def test_hand_computed_mps_pair():
    # A: T=1000 c=600 m=200; B: T=2000 c=300 m=700 on MPS 50/50 (MIG off): computed by hand
    # sigma=0.5 beta=1 D=0.9 n=2: A = 1000*max(1, .6/.5, .9*1.125) = 1200
    #                             B = 2000*max(1, .3/.5, 1.0125) = 2025
    pool = _pool([1000, 2000], [600, 300], [200, 700])
    sp = SP.build_space(4, 2, (25, 50, 75))
    lay = next(l for l in sp.layouts if not l.mig and l.slots[0].sm800 == 400)
    t, cr, solo = CR.corun(lay, [0, 1], pool)
    assert t == [1200, 2025] and cr == 2025 and solo == 3000
    assert CR.r_final(solo, cr) == pytest.approx((3000 / 2025 - 1) * 100, rel=1e-15)


def test_hand_computed_mig_private_pair():
    # [{0.5},0.5m]+[{0.375},0.5m]: A on 4g (sigma .5, beta .5), B on 3g (sigma .375, beta .5)
    # A = 1000*max(1, 1.2, 0.2/0.5) = 1200 ; B = 2000*max(1, 0.8, 0.7/0.5=1.4) = 2800
    pool = _pool([1000, 2000], [600, 300], [200, 700])
    sp = SP.build_space(4, 2, (25, 50, 75))
    lay = next(l for l in sp.layouts if l.mig and len({s.dom for s in l.slots}) == 2
               and l.slots[0].sm800 == 400)
    t, cr, solo = CR.corun(lay, [0, 1], pool)
    assert t == [1200, 2800] and cr == 2800
    # and with the members swapped (A on the 3g slot): A = 1000*max(1, .6/.375=1.6) = 1600,
    # B = 2000*max(1, .3/.5, 1.4) = 2800
    t, cr, _ = CR.corun(lay, [1, 0], pool)
    assert t == [2800, 1600]


def test_ceil_rounding():
    # 1000 * 8100 / 8000 = 1012.5 -> 1013 (ceil)
    assert CR.slot_time(1000, 100, 800, 8, 900, 2) == 1013


def test_intermediate_reward_closed_form():
    # r_i = (SmAllocRatio*ComputeRatio + MemoryAllocRatio*MemoryRatio) * DurationRatio^2
    pool = _pool([1000, 3000], [600, 200], [200, 600])
    slot = SP.Slot(400, 4, 0)          # sigma = 0.5, beta = 0.5
    # job 0: ComputeRatio 600/400 = 1.5, MemoryRatio 200/400 = .5, DurationRatio 1000/2000 = .5
    assert CR.r_intermediate(slot, 0, [0, 1], pool) == pytest.approx(
        (0.5 * 1.5 + 0.5 * 0.5) * 0.25, rel=1e-15)
