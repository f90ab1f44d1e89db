"""schedule-quality metrics of the paper's evaluation (ORACLE, test
infrastructure only).

Paper: throughput of a queue relative to time sharing (Fig. 8); per-application
slowdown AppSlowdown(J) = CoRunAppTime(J) / SoloRunAppTime(J) averaged over the queue
(Fig. 11); Fairness(Q_i) = min_J AppSlowdown(J) / max_J AppSlowdown(J)
(Fig. 12, after [55]).  CoRunAppTime(J) is J's own execution time in its job set
under the chosen partition -- here the slot time t_k of the co-run model (reading R8,
oracle/corun.py); SoloRunAppTime(J) = T_p.  A schedule of a window is a list of actions (one
per job set, each job exactly once); the queue's co-run time is the sum of the job
sets' CoRunTimes (they run one after another) and its time-sharing time the sum of the solo
times.

Pins: tests/test_oracle_metrics.py -- time sharing gives every AppSlowdown = 1 and Fairness = 1
exactly; hand-computed 2-job MPS / MIG cases (the slot times of tests/test_oracle_corun.py);
throughput ratio = Solo / CoRun of the exhaustive optimum equals oracle.brute's optimum.
"""
from __future__ import annotations

from fractions import Fraction

from . import actions as A
from . import corun as CR


def member_times(space, window, idx, pool, q3: int = 1, off=None):
    """Action idx on window -> (CoRun, Solo, [(position g_i, pool id, t_k of its slot)])."""
    l, g, sg = A.decode(space, int(idx), off)
    lay = space.layouts[l]
    jobs = CR.assign(lay, g, sg, window)
    t, cr, solo = CR.corun(lay, jobs, pool, q3)
    return cr, solo, [(gi, int(window[gi]), t[sg[i]]) for i, gi in enumerate(g)]


def queue_metrics(space, window, actions, pool, q3: int = 1):
    """A schedule (list of action indices covering every window position once) -> dict with
    co-run time (sum of CoRun), solo time, throughput ratio, per-position AppSlowdown (exact
    Fractions), mean AppSlowdown and Fairness."""
    off = A.offsets(space)
    W = len(window)
    slow = [None] * W
    corun_sum = solo_sum = 0
    for idx in actions:
        cr, solo, mem = member_times(space, window, idx, pool, q3, off)
        corun_sum += cr
        solo_sum += solo
        for gi, p, t in mem:
            assert slow[gi] is None, "job scheduled twice"
            slow[gi] = Fraction(t, int(pool.solo_ticks[p]))
    assert all(s is not None for s in slow), "job not scheduled"
    return {"corun": corun_sum, "solo": solo_sum,
            "throughput": Fraction(solo_sum, corun_sum), "slowdown": slow,
            "mean_slowdown": sum(slow) / W, "fairness": min(slow) / max(slow)}


def time_sharing_actions(space, W: int):
    """Every job alone on the whole GPU: the singleton action on the single-slot
    layout with the whole GPU (sm800 = 800, b8 = 8)."""
    whole = [l for l, lay in enumerate(space.layouts)
             if lay.C == 1 and lay.slots[0].sm800 == 800 and lay.slots[0].b8 == 8]
    assert whole, "space has no whole-GPU layout"
    off = A.offsets(space)
    return [A.action_index(space, whole[0], (j,), (0,), off) for j in range(W)]


__all__ = ["member_times", "queue_metrics", "time_sharing_actions"]
