"""Pins for oracle/metrics.py -- AppSlowdown and Fairness."""
from fractions import Fraction
from types import SimpleNamespace

import numpy as np

import synth
from oracle import actions as A
from oracle import brute as BR
from oracle import metrics as MT
from oracle import space as SP

S10 = tuple(range(10, 100, 10))


def test_time_sharing_slowdown_and_fairness_are_one():
    # time sharing runs every job alone on the whole GPU: CoRunAppTime = SoloRunAppTime
    # for every job, so AppSlowdown = 1, Fairness = 1 (its maximum) and throughput 1
    pool = synth.make_pool(27)
    sp = SP.build_space(12, 4, S10)
    for w in synth.table_v_windows(pool):
        m = MT.queue_metrics(sp, w, MT.time_sharing_actions(sp, 12), pool)
        assert all(s == 1 for s in m["slowdown"])
        assert m["fairness"] == 1 and m["mean_slowdown"] == 1 and m["throughput"] == 1


def test_hand_computed_mps_pair_slowdowns():
    # tests/test_oracle_corun.py::test_hand_computed_mps_pair: A (T 1000) runs 1200, B (T 2000)
    # runs 2025 on MPS 50/50 -> AppSlowdown 1.2 and 1.0125, mean 1.10625,
    # Fairness = 1.0125 / 1.2 = 0.84375, queue throughput 3000 / 2025
    pool = SimpleNamespace(solo_ticks=np.array([1000, 2000], np.int64),
                           compute_pm=np.array([600, 300], np.int16),
                           memory_pm=np.array([200, 700], np.int16))
    sp = SP.build_space(2, 2, (25, 50, 75))
    l = next(i for i, lay in enumerate(sp.layouts) if not lay.mig and lay.C == 2
             and lay.slots[0].sm800 == 400)
    idx = A.action_index(sp, l, (0, 1), (0, 1))
    m = MT.queue_metrics(sp, [0, 1], [idx], pool)
    assert m["slowdown"] == [Fraction(6, 5), Fraction(81, 80)]
    assert m["mean_slowdown"] == Fraction(177, 160)
    assert m["fairness"] == Fraction(27, 32)
    assert m["throughput"] == Fraction(3000, 2025)


def test_optimum_schedule_metrics_match_brute_force():
    # the exhaustive optimum's job sets, re-scored through the metrics: throughput = Solo / OPT
    pool = synth.make_pool(27)
    sp = SP.build_space(8, 3, S10)
    for w in synth.make_windows(pool, 4, 8, step=3):
        ref = BR.dp_opt(sp, [int(x) for x in w], pool)
        acts = [a for a in ref["block_action"] if a >= 0]
        m = MT.queue_metrics(sp, w, acts, pool)
        assert m["corun"] == ref["cost"] and m["solo"] == ref["solo"]
        assert all(s >= 1 for s in m["slowdown"])          # co-running never speeds a job up
        assert 0 < m["fairness"] <= 1
