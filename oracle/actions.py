"""a5 -- the joint action space and its index (ORACLE, test infrastructure only).

Paper: an action selects a co-scheduling job set JS (1 <= C <= Cmax jobs of the window) and
its resource partitioning R; the action count is
sum_C binom(W, C) * C! * N_C (this space adds the C = 1 term, reading R2/SURVEY Q1).

Action a = (l, g, sigma): layout l with C_l slots; g = (g_0 < ... < g_{C-1}) window
positions; sigma a permutation of 0..C-1 sending member i (job g_i) to slot sigma(i).
    idx = off[l] + rank_lex(g) * C! + lehmer(sigma),   off[l] = sum_{l' < l} P(W, C_l').
Valid iff no member of g is already scheduled.  Random (exploration) actions are drawn
uniformly from the valid ones: the k-th valid action in index order (reading R14).

Pins: tests/test_oracle_actions.py -- rank/unrank against itertools enumeration order
(brute force), |A| against the P:315 closed form plus the C=1 term, round trips, and the
k-th-valid unranking against an explicit filtered list.
"""
from __future__ import annotations

from math import comb, factorial


def perm_count(n: int, k: int) -> int:
    """P(n, k) = n! / (n-k)!  (0 if k > n)."""
    if k > n or k < 0:
        return 0
    return factorial(n) // factorial(n - k)


def rank_comb(g, W: int) -> int:
    """Lexicographic rank of the sorted combination g among the len(g)-subsets of range(W)."""
    C = len(g)
    r = 0
    prev = -1
    for i, gi in enumerate(g):
        for v in range(prev + 1, gi):
            r += comb(W - 1 - v, C - 1 - i)
        prev = gi
    return r


def unrank_comb(r: int, W: int, C: int) -> tuple:
    out = []
    v = 0
    for i in range(C):
        while True:
            c = comb(W - 1 - v, C - 1 - i)
            if r < c:
                break
            r -= c
            v += 1
        out.append(v)
        v += 1
    return tuple(out)


def lehmer(sigma) -> int:
    """Rank of the permutation tuple (sigma(0), ..., sigma(C-1)) in lexicographic order."""
    C = len(sigma)
    r = 0
    for i in range(C):
        d = sum(1 for j in range(i + 1, C) if sigma[j] < sigma[i])
        r += d * factorial(C - 1 - i)
    return r


def unlehmer(r: int, C: int) -> tuple:
    avail = list(range(C))
    out = []
    for i in range(C):
        f = factorial(C - 1 - i)
        d, r = divmod(r, f)
        out.append(avail.pop(d))
    return tuple(out)


def offsets(space) -> list:
    off = [0]
    for l in space.layouts:
        off.append(off[-1] + perm_count(space.W, l.C))
    return off


def n_actions(space) -> int:
    return offsets(space)[-1]


def action_index(space, l: int, g, sigma, off=None) -> int:
    off = off or offsets(space)
    C = space.layouts[l].C
    return off[l] + rank_comb(g, space.W) * factorial(C) + lehmer(sigma)


def decode(space, idx: int, off=None):
    """idx -> (l, g, sigma)."""
    off = off or offsets(space)
    lo, hi = 0, space.L
    while hi - lo > 1:  # last l with off[l] <= idx
        mid = (lo + hi) // 2
        if off[mid] <= idx:
            lo = mid
        else:
            hi = mid
    l = lo
    C = space.layouts[l].C
    w = idx - off[l]
    rg, rs = divmod(w, factorial(C))
    return l, unrank_comb(rg, space.W, C), unlehmer(rs, C)


def group_mask(g) -> int:
    m = 0
    for j in g:
        m |= 1 << j
    return m


def n_valid(space, sched: int) -> int:
    U = space.W - bin(sched).count("1")
    return sum(perm_count(U, l.C) for l in space.layouts)


def kth_valid(space, sched: int, k: int, off=None) -> int:
    """Index of the k-th valid action (0-based, index order).  Unscheduled positions
    u_0 < u_1 < ... ; the k-th valid action of layout l is the lexicographic unranking over
    them, which preserves index order."""
    off = off or offsets(space)
    free = [j for j in range(space.W) if not (sched >> j) & 1]
    U = len(free)
    for l, lay in enumerate(space.layouts):
        cnt = perm_count(U, lay.C)
        if k < cnt:
            C = lay.C
            rg, rs = divmod(k, factorial(C))
            gp = unrank_comb(rg, U, C)
            g = tuple(free[x] for x in gp)
            return off[l] + rank_comb(g, space.W) * factorial(C) + rs
        k -= cnt
    raise ValueError("k >= n_valid")


def explore_k(u64: int, nv: int) -> int:
    """k = floor(u64 * n_valid / 2^64)."""
    return (int(u64) * int(nv)) >> 64
