"""Schedule-quality evaluation through libhrp (Fig. 8 P:263-269,
AppSlowdown, Fairness P:307-309).

Marshalling and reporting only: the greedy policy's actions come from hrp_env_step (epsilon 0,
P:158 "online"), the exhaustive optimum from hrp_brute_run, and every co-run time from
hrp_job_times; this module strings the calls together and aggregates the integer times
(sums, ratios, min / max) for the report.
"""
from __future__ import annotations

import numpy as np
import torch

from . import hrp


def greedy_rollout(sess, windows):
    """Greedy episodes of the session's policy, one env per window (sess.E == len(windows)):
    reset to the windows, step with epsilon = 0 until each env has scheduled its whole window
    once.  Returns one action list per window (the job sets in the order chosen)."""
    n, W = windows.shape
    assert sess.E == n
    dev = sess.dev
    sess.reset(windows)
    zeros32 = torch.zeros(n, dtype=torch.int32, device=dev)
    zeros64 = torch.zeros(n, dtype=torch.int64, device=dev)
    nxt = torch.from_numpy(np.ascontiguousarray(windows)).to(dev)
    out = [[] for _ in range(n)]
    live = np.ones(n, bool)
    for _ in range(W):
        sess.step(0, zeros32, zeros64, nxt)
        sess.sync()
        a = sess.actions.cpu().numpy()
        d = sess.done.cpu().numpy()
        for e in np.nonzero(live)[0]:
            out[e].append(int(a[e]))
            if d[e]:
                live[e] = False
        if not live.any():
            break
    assert not live.any(), "an episode did not finish within W steps"
    return out


def job_metrics(plan, pool, windows, schedules, device=0, stream=None):
    """Per window: the schedule's co-run time (sum of its job sets' CoRunTime), time-sharing
    time, throughput ratio, each job's AppSlowdown t_k / T_p, their mean and the Fairness
    min / max -- co-run times from hrp_job_times."""
    dev = torch.device("cuda", device)
    st = stream or torch.cuda.current_stream(dev)
    rows_w, rows_a, owner = [], [], []
    for i, (w, acts) in enumerate(zip(windows, schedules)):
        for a in acts:
            rows_w.append(w)
            rows_a.append(a)
            owner.append(i)
    n = len(rows_a)
    W = windows.shape[1]
    dw = torch.from_numpy(np.ascontiguousarray(np.stack(rows_w), np.uint8)).to(dev)
    da = torch.tensor(rows_a, dtype=torch.int64, device=dev)
    cr = torch.empty(n, dtype=torch.int64, device=dev)
    so = torch.empty(n, dtype=torch.int64, device=dev)
    mt = torch.empty((n, 4), dtype=torch.int64, device=dev)
    hrp.hrp_job_times(plan, n, dw, da, cr, so, mt, st.cuda_stream)
    torch.cuda.synchronize(dev)
    cr, so, mt = cr.cpu().numpy(), so.cpu().numpy(), mt.cpu().numpy()
    T = np.asarray(pool.solo_ticks, np.int64)
    res = [{"corun": 0, "solo": 0, "t": [None] * W} for _ in windows]
    space = plan_space(plan)
    for r in range(n):
        i = owner[r]
        res[i]["corun"] += int(cr[r])
        res[i]["solo"] += int(so[r])
        _, g, _ = hrp.hrp_decode_action(space, rows_a[r])
        for k, gi in enumerate(g):
            assert res[i]["t"][gi] is None, "job scheduled twice"
            res[i]["t"][gi] = int(mt[r, k])
    for i, w in enumerate(windows):
        t = res[i]["t"]
        assert all(x is not None for x in t), "job not scheduled"
        slow = [t[j] / float(T[w[j]]) for j in range(W)]
        res[i].update(throughput=res[i]["solo"] / res[i]["corun"], slowdown=slow,
                      mean_slowdown=float(np.mean(slow)), fairness=min(slow) / max(slow))
    return res


_PLAN_SPACES = {}


def make_plan(space, profiles, device=0, stream=None):
    """hrp_brute_create, remembering the space for decoding (hrp_decode_action)."""
    dev = torch.device("cuda", device)
    st = stream or torch.cuda.current_stream(dev)
    plan = hrp.hrp_brute_create(space, profiles, device, st.cuda_stream)
    _PLAN_SPACES[plan.value] = space
    return plan


def plan_space(plan):
    return _PLAN_SPACES[plan.value]


def optimum_schedules(plan, windows, device=0, stream=None):
    """The exhaustive optimum's job sets per window (hrp_brute_run's per-block actions)."""
    dev = torch.device("cuda", device)
    st = stream or torch.cuda.current_stream(dev)
    n, W = windows.shape
    w = torch.from_numpy(np.ascontiguousarray(windows, np.uint8)).to(dev)
    best = torch.empty(n, dtype=torch.int64, device=dev)
    solo = torch.empty(n, dtype=torch.int64, device=dev)
    rgs = torch.empty((n, W), dtype=torch.uint8, device=dev)
    bact = torch.empty((n, W), dtype=torch.int64, device=dev)
    hrp.hrp_brute_run(plan, n, w, best, solo, rgs, bact, st.cuda_stream)
    torch.cuda.synchronize(dev)
    b = bact.cpu().numpy()
    return [[int(x) for x in row if x >= 0] for row in b], best.cpu().numpy()


def time_sharing_schedules(space, windows):
    """Every job alone on the whole GPU, as actions of `space` (its whole-GPU
    single-slot layout; hrp_layout_table / hrp_decode_action only)."""
    tab = hrp.hrp_layout_table(space)
    whole = [l for l in range(tab["n_layouts"]) if tab["nslots"][l] == 1
             and int(tab["slots"][l, 0]["sm800"]) == 800 and int(tab["slots"][l, 0]["b8"]) == 8]
    assert whole, "space has no whole-GPU layout"
    l0 = whole[0]
    # action index of (l0, {j}, identity): off[l0] + j (C = 1: rank_lex({j}) = j, 1! = 1)
    off = 0
    W = windows.shape[1]
    for l in range(l0):
        C = int(tab["nslots"][l])
        p = 1
        for i in range(C):
            p *= W - i
        off += p
    return [[off + j for j in range(W)] for _ in windows]


def mig_partitions(W, cmax):
    """The MIG partitions with at most cmax CIs (the whole GPU and every maximal GI config x CI
    packing), from libhrp's layout table of the space with no MPS splits (each CI one process at
    100 %): tuples of (sm800, b8, domain) per CI."""
    tab = hrp.hrp_layout_table(hrp.make_space(W, cmax, (), True))
    return [tuple((int(x["sm800"]), int(x["b8"]), int(x["dom"]))
                  for x in tab["slots"][l][:tab["nslots"][l]]) for l in range(tab["n_layouts"])]


def default_mps_table(partition, cmax):
    """MIG+MPS Default (R27): the partition fixed, k >= 0 job-set members per
    CI under MPS's default mode as equal shares (sm800 = CI compute // k), 1 <= sum k <= cmax:
    an explicit layout table for hrp_space.n_layouts.  A job left alone may also take the whole
    GPU (time sharing, as in the MIG-only baseline): that layout comes first."""
    import itertools
    out = [[(800, 8, 0)]]
    for ks in itertools.product(range(cmax + 1), repeat=len(partition)):
        if not 1 <= sum(ks) <= cmax:
            continue
        lay = []
        for (sm, b8, dom), k in zip(partition, ks):
            if k:
                lay += [(sm // k, b8, dom)] * k
        out.append(lay)
    return out
