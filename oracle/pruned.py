"""a5 (config 4) -- exact top-C pruned argmax (ORACLE, test infrastructure only).

Same result as the explicit argmax of env.greedy_explicit (max of the fixed-point Q^ over
all valid actions, ties to the lowest index) without enumerating P(W, C) groups per layout:

For slot type tau let Top_tau = the C best unscheduled positions j ordered by
(F(cJ[j][tau]) descending, j ascending).  Exchange argument: if a
lowest-index maximiser put job j on a slot of type tau with j outside Top_tau, some
j' in Top_tau is unused by the other C-1 slots; moving the slot to j' does not lower the
(integer, exact) score, and when it ties j' < j, which makes the sorted group
lexicographically smaller and hence the index smaller -- a contradiction.  So every
lowest-index maximiser uses only Top-lists, and enumerating the <= C^C distinct assignments
per layout finds it.

Pins: tests/test_oracle_pruned.py -- equals greedy_explicit / greedy_bruteforce on random
heads with heavy integer ties and random scheduled masks (W 3..8, Cmax 1..4, both share sets).
"""
from __future__ import annotations

import itertools
from math import factorial

from . import actions as A


def top_lists(FcJ, sched: int, W: int, T: int, C: int):
    free = [j for j in range(W) if not (sched >> j) & 1]
    tops = []
    for tau in range(T):
        order = sorted(free, key=lambda j: (-FcJ[j][tau], j))
        tops.append(order[:C])
    return tops


def greedy_pruned(space, Fv, FcL, FcJ, sched: int, off=None):
    off = off or A.offsets(space)
    W, T = space.W, space.T
    cmax = max(l.C for l in space.layouts)
    tops = top_lists(FcJ, sched, W, T, cmax)
    best, bi = None, -1
    for l, lay in enumerate(space.layouts):
        C = lay.C
        st = space.slot_type[l]
        cand = [tops[st[k]][:C] for k in range(C)]
        if any(len(c) < C for c in cand):
            continue
        lbest, lidx = None, None
        for js in itertools.product(*cand):
            if len(set(js)) < C:
                continue
            score = Fv + FcL[l] + sum(FcJ[js[k]][st[k]] for k in range(C))
            if lbest is not None and score < lbest:
                continue                              # the index only breaks ties
            g = tuple(sorted(js))
            sigma = tuple(js.index(gi) for gi in g)   # member i (job g_i) -> its slot
            w = A.rank_comb(g, W) * factorial(C) + A.lehmer(sigma)
            if lbest is None or score > lbest or w < lidx:
                lbest, lidx = score, w
        if lbest is not None and (best is None or lbest > best):
            best, bi = lbest, off[l] + lidx
    return bi, best
