"""a14 -- exhaustive optimum of the co-scheduling problem (ORACLE, test infrastructure only).

Paper: given W, Cmax and Q = {J_1..J_W}, choose job sets JS_i that partition Q
with 1 <= |JS_i| <= Cmax and partitionings R_i, minimising sum_i CoRunTime(JS_i, R_i)
subject to CoRunTime(JS_i, R_i) <= SoloRunTime(JS_i).  The paper's baselines search this
exhaustively.

  best(B) = min over layouts l with C_l = |B| and permutations sigma of CoRun(B, l, sigma)
            among feasible choices; ties to the lowest action index (l, then lehmer(sigma)).
  OPT     = min over set partitions of Q into blocks of size <= Cmax of sum best(B).
  Canonical tie-break between optimal partitions ("block order", reading R21b): list blocks
  by their minimum element; at the first block where two partitions differ, prefer the one
  containing the smallest element of the two blocks' symmetric difference.

Three independent algorithms, which the pins require to agree:
  literal_opt  every (partition, per-block action) vector, W <= 5 (no best() decomposition)
  rgs_opt      restricted-growth-string enumeration of set partitions, minimising
               (sum best, block-order key)
  dp_opt       subset DP: OPT(S) = min over B containing min(S) of best(B) + OPT(S \\ B)

Pins: tests/test_oracle_brute.py -- the three agree; Cmax = 1 gives exactly the time-sharing
cost (ratio 1.0); OPT is monotone in Cmax and in layout-set inclusion;
restricted baselines (MPS-only, MIG-only C<=2) are never better than the full space; every
solution partitions Q and satisfies CoRun <= Solo per block.
"""
from __future__ import annotations

import itertools
from math import factorial

import numpy as np

from . import actions as A
from . import corun as CR


def block_best_literal(space, window, block, pool, q3=1, off=None):
    """best(B) by plain loops: (cost, idx) or (None, -1) if no feasible choice."""
    off = off or A.offsets(space)
    C = len(block)
    best, bidx = None, -1
    for l, lay in enumerate(space.layouts):
        if lay.C != C:
            continue
        for sg in itertools.permutations(range(C)):
            jobs = CR.assign(lay, block, sg, window)
            _, cr, solo = CR.corun(lay, jobs, pool, q3)
            if cr > solo:
                continue
            idx = off[l] + A.rank_comb(block, space.W) * factorial(C) + A.lehmer(sg)
            if best is None or cr < best:
                best, bidx = cr, idx
    return best, bidx


def all_block_best(space, window, pool, q3=1):
    """best(B) for every block B (bitmask) with 1 <= |B| <= Cmax, vectorised over
    (block, permutation) with numpy -- the same formula as corun.slot_time elementwise.
    Returns dict mask -> (cost, idx), cost None when infeasible."""
    off = A.offsets(space)
    W = space.W
    T = pool.solo_ticks.astype(np.int64)
    cc = pool.compute_pm.astype(np.int64)
    mm = pool.memory_pm.astype(np.int64)
    ids = np.array([int(x) for x in window], np.int64)
    out = {}
    for C in sorted({l.C for l in space.layouts}):
        if C > W:
            continue
        blocks = np.array(list(itertools.combinations(range(W), C)), np.int64)   # [nb][C]
        perms = np.array(list(itertools.permutations(range(C))), np.int64)        # [np][C]
        nb, npm = len(blocks), len(perms)
        job = ids[blocks]                                                         # [nb][C]
        # jobs_on_slot[b, p, sigma_p(i)] = job[b, i]
        jos = np.zeros((nb, npm, C), np.int64)
        for p in range(npm):
            for i in range(C):
                jos[:, p, perms[p, i]] = job[:, i]
        solo = T[job].sum(1)                                                      # [nb]
        best = np.full(nb, np.iinfo(np.int64).max, np.int64)
        bidx = np.full(nb, -1, np.int64)
        ranks = np.array([A.rank_comb(tuple(b), W) for b in blocks], np.int64)
        lehm = np.array([A.lehmer(tuple(p)) for p in perms], np.int64)
        for l, lay in enumerate(space.layouts):
            if lay.C != C:
                continue
            tk = []
            for k, s in enumerate(lay.slots):
                dk = [k2 for k2, s2 in enumerate(lay.slots) if s2.dom == s.dom]
                D = sum(mm[jos[:, :, k2]] for k2 in dk)
                n = len(dk)
                Tk, ck = T[jos[:, :, k]], cc[jos[:, :, k]]
                comp = -((-(Tk * np.maximum(5 * s.sm800, 4 * ck))) // (5 * s.sm800))
                mem = -((-(Tk * np.maximum(1000 * s.b8, D * (8 + q3 * (n - 1)))))
                        // (1000 * s.b8))
                tk.append(np.maximum(comp, mem))
            cr = np.max(np.stack(tk, -1), -1)                                     # [nb][np]
            cr = np.where(cr <= solo[:, None], cr, np.iinfo(np.int64).max)
            p_best = np.argmin(cr, 1)                                             # first min
            c_best = cr[np.arange(nb), p_best]
            better = c_best < best   # strict: earlier layout wins ties (lower idx)
            best = np.where(better, c_best, best)
            bidx = np.where(better, off[l] + ranks * factorial(C) + lehm[p_best], bidx)
        for b in range(nb):
            mask = A.group_mask(tuple(blocks[b]))
            feas = best[b] != np.iinfo(np.int64).max
            out[mask] = (int(best[b]) if feas else None, int(bidx[b]) if feas else -1)
    return out


def bitrev(mask: int, W: int) -> int:
    r = 0
    for j in range(W):
        if (mask >> j) & 1:
            r |= 1 << (W - 1 - j)
    return r


def block_order_key(blocks, W):
    """Lexicographically smaller key = preferred partition (blocks sorted by min element)."""
    return tuple(-bitrev(b, W) for b in sorted(blocks, key=lambda m: (m & -m)))


def _result(space, window, pool, blocks, best):
    W = space.W
    blocks = sorted(blocks, key=lambda m: (m & -m))
    rgs = [0] * W
    bact = [-1] * W
    for k, b in enumerate(blocks):
        for j in range(W):
            if (b >> j) & 1:
                rgs[j] = k
        bact[k] = best[b][1]
    cost = sum(best[b][0] for b in blocks)
    solo = sum(int(pool.solo_ticks[int(x)]) for x in window)
    return {"cost": cost, "solo": solo, "rgs": rgs, "block_action": bact, "blocks": blocks}


def dp_opt(space, window, pool, q3=1, best=None):
    W = space.W
    best = best or all_block_best(space, window, pool, q3)
    full = (1 << W) - 1
    INF = None
    opt = {0: (0, ())}   # mask -> (cost, key tuple of chosen blocks' -bitrev in order)
    choice = {}
    for S in range(1, full + 1):
        low = S & -S
        rest = S ^ low
        bestv = INF
        # blocks B containing low, B subset of S, |B| <= Cmax
        sub = rest
        cands = []
        while True:
            B = sub | low
            if bin(B).count("1") <= space.cmax and B in best and best[B][0] is not None \
                    and (S ^ B) in opt and opt[S ^ B] is not None:
                cands.append(B)
            if sub == 0:
                break
            sub = (sub - 1) & rest
        for B in cands:
            c = best[B][0] + opt[S ^ B][0]
            key = (-bitrev(B, W),) + opt[S ^ B][1]
            if bestv is None or (c, key) < bestv:
                bestv = (c, key)
                choice[S] = B
        opt[S] = bestv
    blocks = []
    S = full
    while S:
        B = choice[S]
        blocks.append(B)
        S ^= B
    return _result(space, window, pool, blocks, best)


def set_partitions_rgs(W: int, cmax: int):
    """All set partitions of range(W) with blocks <= cmax, via restricted growth strings."""
    a = [0] * W
    sizes = [0] * W

    def rec(i, m):
        if i == W:
            yield list(a)
            return
        for k in range(m + 1):
            if sizes[k] < cmax:
                a[i] = k
                sizes[k] += 1
                yield from rec(i + 1, max(m, k + 1))
                sizes[k] -= 1

    yield from rec(0, 0)


def rgs_opt(space, window, pool, q3=1, best=None):
    W = space.W
    best = best or all_block_best(space, window, pool, q3)
    bestv, bestp = None, None
    for rgs in set_partitions_rgs(W, space.cmax):
        nb = max(rgs) + 1
        blocks = [0] * nb
        for j, k in enumerate(rgs):
            blocks[k] |= 1 << j
        if any(best[b][0] is None for b in blocks):
            continue
        c = sum(best[b][0] for b in blocks)
        key = (c, block_order_key(blocks, W))
        if bestv is None or key < bestv:
            bestv, bestp = key, blocks
    return _result(space, window, pool, bestp, best)


def literal_opt(space, window, pool, q3=1):
    """Every (partition, per-block (layout, sigma)) vector; W <= 5 only."""
    W = space.W
    off = A.offsets(space)
    bestv, best_sol = None, None
    for rgs in set_partitions_rgs(W, space.cmax):
        nb = max(rgs) + 1
        blocks = [tuple(j for j in range(W) if rgs[j] == k) for k in range(nb)]
        per_block = []
        for blk in blocks:
            opts = []
            for l, lay in enumerate(space.layouts):
                if lay.C != len(blk):
                    continue
                for sg in itertools.permutations(range(lay.C)):
                    _, cr, solo = CR.corun(lay, CR.assign(lay, blk, sg, window), pool, q3)
                    if cr <= solo:
                        opts.append((cr, A.action_index(space, l, blk, sg, off)))
            per_block.append(opts)
        if any(not o for o in per_block):
            continue
        masks = [A.group_mask(b) for b in blocks]
        for combo in itertools.product(*per_block):
            tot = sum(c for c, _ in combo)
            key = (tot, block_order_key(masks, W), tuple(i for _, i in combo))
            if bestv is None or key < bestv:
                bestv, best_sol = key, (masks, combo)
    masks, combo = best_sol
    best = {m: c for m, c in zip(masks, combo)}
    return _result(space, window, pool, masks, best)
