"""a1 -- the partition-configuration space R (ORACLE, test infrastructure only).

Paper: MIG splits the GPU into GPU Instances (GIs, GPC granularity, private LLC/HBM) and each
GI into Compute Instances (CIs, exclusive GPCs, shared GI memory); MPS splits a CI (or the
whole GPU when MIG is off) by SM percentage (Fig. 2).  One GPC is
disabled with MIG on (MIG totals 87.5%); only 19 GI variants exist.
Partition notation and Table VII: P:252.

Readings: R3/R4 GI and CI placement = the A100 MIG placement table, maximal fills
only; R5 MPS splits are ascending multisets from S (sum 100%); R6 compute in 1/8 GPCs;
R23 MPS shares are CI-relative.  Units: sm800 = compute in 1/800 of the GPU (GPCs x percent),
b8 = memory bandwidth in 1/8 of the GPU, dom = memory domain (GI index; 0 with MIG off).

Canonical order (reading R24): MIG-off layouts first (k ascending, then share tuple
lexicographic); then GI configs in lexicographic order of their [(start, gpcs)] lists; inside
one, the product of per-GI CI packings (lexicographic [(start, gpcs)], first GI slowest); then
the product of per-CI compositions (first CI slowest).  Slot order: GI start, CI start,
share position.  Slot types: distinct (sm800, b8) numbered in ascending order.

Pins: tests/test_oracle_space.py (19 GI configs P:64; no 2+5 / 1+6; MIG compute <= 7/8 P:102;
Table VII members P:275-277 in tests/golden/table7.txt; hand-listed config-1 layouts; share
sums; counts vs an independent brute-force placement search).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass
from fractions import Fraction

# [ext] A100 MIG GI profiles: gpcs -> (memory slices of 8, allowed start slices).
GI_PROFILES = {1: (1, tuple(range(7))), 2: (2, (0, 2, 4)), 3: (4, (0, 4)), 4: (4, (0,)),
               7: (8, (0,))}
# [ext] CI placements inside a GI of g GPCs: ci gpcs -> allowed GPC starts.
CI_PROFILES = {
    7: {1: tuple(range(7)), 2: (0, 2, 4), 3: (0, 4), 4: (0,), 7: (0,)},
    4: {1: (0, 1, 2, 3), 2: (0, 2), 4: (0,)},
    3: {1: (0, 1, 2), 2: (0,), 3: (0,)},
    2: {1: (0, 1), 2: (0,)},
    1: {1: (0,)},
}
MIG_GPCS = 7  # one of the 8 GPCs is disabled with MIG on


def _maximal_sets(placements, occupies, budget_ok):
    """All maximal sets of pairwise-disjoint placements (brute force over subsets)."""
    out = []
    n = len(placements)

    def ok(sel):
        used = set()
        for p in sel:
            occ = occupies(p)
            if used & occ:
                return False
            used |= occ
        return budget_ok(sel)

    valid = []
    for r in range(1, n + 1):
        for sel in itertools.combinations(placements, r):
            if ok(sel):
                valid.append(sel)
    vs = set(valid)
    for sel in valid:
        maximal = True
        for p in placements:
            if p in sel:
                continue
            if tuple(sorted(sel + (p,))) in vs or ok(sel + (p,)):
                maximal = False
                break
        if maximal:
            out.append(tuple(sorted(sel)))
    return sorted(set(out)), valid


def gi_placements():
    return [(s, g) for g, (_, starts) in GI_PROFILES.items() for s in starts]


def gi_configs(maximal_only: bool = True):
    """GI configs as sorted lists of (start, gpcs) (reading R3/R4)."""
    pl = sorted(gi_placements())
    maxi, valid = _maximal_sets(
        pl, lambda p: set(range(p[0], p[0] + GI_PROFILES[p[1]][0])),
        lambda sel: sum(g for _, g in sel) <= MIG_GPCS)
    return maxi if maximal_only else sorted(set(tuple(sorted(v)) for v in valid))


def ci_packings(g: int):
    """Maximal CI packings of a GI with g GPCs as sorted lists of (start, gpcs)."""
    pl = sorted((s, c) for c, starts in CI_PROFILES[g].items() for s in starts)
    maxi, _ = _maximal_sets(pl, lambda p: set(range(p[0], p[0] + p[1])),
                            lambda sel: sum(c for _, c in sel) <= g)
    return maxi


def compositions(shares, kmax: int):
    """MPS compositions of one CI: (100,) and ascending multisets of k>=2 shares from S
    summing to 100 (reading R5), ordered by k then lexicographically."""
    out = [(100,)]
    S = sorted(set(shares))
    for k in range(2, kmax + 1):
        for combo in itertools.combinations_with_replacement(S, k):
            if sum(combo) == 100:
                out.append(tuple(combo))
    return out


@dataclass(frozen=True)
class Slot:
    sm800: int   # compute: CI gpcs x MPS share percent (MIG off: 8 x share)
    b8: int      # memory bandwidth in eighths (GI memory slices; 8 with MIG off)
    dom: int     # memory domain (GI index in start order; 0 with MIG off)


@dataclass(frozen=True)
class Layout:
    mig: bool
    gis: tuple      # ((start, gpcs), ...) -- empty with MIG off
    cis: tuple      # per GI: ((start, gpcs), ...)
    comps: tuple    # per CI in slot order: share tuple
    slots: tuple    # Slot, in slot order

    @property
    def C(self) -> int:
        return len(self.slots)

    def notation(self) -> str:
        """Table VII / P:252 notation, e.g. [{0.375},0.5m]+[(0.1)+(0.9),{0.5},0.5m]."""
        def num(fr):
            return f"{float(fr):g}"
        if not self.mig:
            inner = "+".join(f"({num(Fraction(s, 100))})" for s in self.comps[0])
            return f"[{inner},1m]"
        parts = []
        ci_iter = iter(self.comps)
        for (gs, g), cis in zip(self.gis, self.cis):
            mem = GI_PROFILES[g][0]
            ci_strs = []
            for (_, c) in cis:
                comp = next(ci_iter)
                beta = f"{{{num(Fraction(c, 8))}}}"
                if len(comp) == 1:
                    ci_strs.append(beta)
                else:
                    ci_strs.append("+".join(f"({num(Fraction(s, 100))})" for s in comp)
                                   + "," + beta)
            parts.append("[" + "+".join(ci_strs) + f",{num(Fraction(mem, 8))}m]")
        return "+".join(parts)


def enumerate_layouts(cmax: int, shares, mig: bool = True):
    """All layouts with <= cmax slots in canonical order (see module docstring)."""
    out = []
    for comp in compositions(shares, cmax):
        out.append(Layout(False, (), (), (comp,), tuple(Slot(8 * s, 8, 0) for s in comp)))
    if not mig:
        return out
    for gic in gi_configs():
        per_gi = [ci_packings(g) for _, g in gic]
        for packs in itertools.product(*per_gi):
            ci_list = [(d, g, c) for d, ((_, g), pk) in enumerate(zip(gic, packs))
                       for (_, c) in pk]
            if len(ci_list) > cmax:
                continue
            per_ci = [compositions(shares, cmax) for _ in ci_list]
            for comps in itertools.product(*per_ci):
                if sum(len(x) for x in comps) > cmax:
                    continue
                slots = []
                for (d, g, c), comp in zip(ci_list, comps):
                    for s in comp:
                        slots.append(Slot(c * s, GI_PROFILES[g][0], d))
                out.append(Layout(True, tuple(gic), tuple(packs), tuple(comps),
                                  tuple(slots)))
    return out


def mig_partitions(cmax: int):
    """The MIG partitions with at most cmax CIs -- the whole GPU (MIG off) and every maximal GI
    config x CI packing (R3/R4) -- as tuples of CIs (compute sm800 at 100 %, memory b8, domain),
    in canonical layout order (they are the layouts whose CIs each host one process)."""
    return [tuple((s.sm800, s.b8, s.dom) for s in lay.slots)
            for lay in enumerate_layouts(cmax, (), True)]


def default_mps_layouts(partition, cmax: int):
    """MIG+MPS Default under reading R27: the MIG partition is fixed; each CI hosts
    k >= 0 of the job set's members under MPS's default mode, modelled as equal shares
    (sm800 = the CI's compute // k); 1 <= sum k <= cmax; CIs may stay idle.  A job left alone
    may also take the whole GPU (time sharing, P:245 -- as in the MIG-only baseline), so every
    window has a feasible schedule: that layout comes first, then the partition's layouts in
    lexicographic order of the per-CI counts, slots in CI order."""
    out = [Layout(False, (), (), ((100,),), (Slot(800, 8, 0),))]
    n = len(partition)
    for ks in itertools.product(range(cmax + 1), repeat=n):
        if not 1 <= sum(ks) <= cmax:
            continue
        slots = []
        for (sm, b8, dom), k in zip(partition, ks):
            if k:
                slots += [Slot(sm // k, b8, dom)] * k
        out.append(Layout(True, (), (), (), tuple(slots)))
    return out


@dataclass
class Space:
    """The layout table plus slot types for one (W, Cmax, S, MIG) configuration."""
    W: int
    cmax: int
    layouts: list
    types: list          # [(sm800, b8)] ascending
    slot_type: list      # per layout: tuple of type ids in slot order
    seq: bool = False    # sequential agent (reading R28): flat head [v, aL]

    @property
    def L(self) -> int:
        return len(self.layouts)

    @property
    def T(self) -> int:
        return len(self.types)

    @property
    def H(self) -> int:
        """Head width 1 + L + W*T (value, layout advantages, job-slot-type advantages); the
        sequential agent's flat head has 1 + L (value, one advantage per partition setup)."""
        return 1 + self.L + (0 if self.seq else self.W * self.T)


def build_space(W: int, cmax: int, shares, mig: bool = True, layouts=None,
                seq: bool = False) -> Space:
    lay = layouts if layouts is not None else enumerate_layouts(cmax, shares, mig)
    types = sorted({(s.sm800, s.b8) for l in lay for s in l.slots})
    tid = {t: i for i, t in enumerate(types)}
    st = [tuple(tid[(s.sm800, s.b8)] for s in l.slots) for l in lay]
    return Space(W, cmax, lay, types, st, seq)


def parse_notation(text: str):
    """Parse P:252 notation into a canonical structure (sorted GIs of sorted CIs), e.g.
    '[{0.375},0.5m]+[(0.1)+(0.9),{0.5},0.5m]'.  Returns a hashable tuple; the MPS-only form
    '[(0.1)+(0.9),1m]' gives ('off', shares)."""
    text = text.replace(" ", "")
    gis = []
    depth = 0
    cur = ""
    for ch in text:
        if ch == "[":
            depth += 1
            cur = ""
        elif ch == "]":
            depth -= 1
            gis.append(cur)
        elif depth > 0:
            cur += ch
    if len(gis) == 1 and "{" not in gis[0]:
        body, mem = gis[0].rsplit(",", 1)
        sh = tuple(sorted(round(float(x.strip("()")) * 100) for x in body.split("+")))
        return ("off", sh)
    parsed = []
    for g in gis:
        body, mem = g.rsplit(",", 1)
        alpha = Fraction(mem.rstrip("m")).limit_denominator(8)
        cis = []
        pending = []
        for tok in body.replace(",", "+").split("+"):
            if tok.startswith("("):
                pending.append(round(float(tok.strip("()")) * 100))
            elif tok.startswith("{"):
                beta = Fraction(tok.strip("{}")).limit_denominator(8)
                cis.append((beta, tuple(sorted(pending)) if pending else (100,)))
                pending = []
        parsed.append((alpha, tuple(sorted(cis))))
    return ("mig", tuple(sorted(parsed)))


def canonical(layout: Layout):
    """Same canonical structure as parse_notation, from a Layout."""
    if not layout.mig:
        return ("off", tuple(sorted(layout.comps[0])))
    parsed = []
    ci_iter = iter(layout.comps)
    for (gs, g), cis in zip(layout.gis, layout.cis):
        alpha = Fraction(GI_PROFILES[g][0], 8)
        lst = []
        for (_, c) in cis:
            lst.append((Fraction(c, 8), tuple(sorted(next(ci_iter)))))
        parsed.append((alpha, tuple(sorted(lst))))
    return ("mig", tuple(sorted(parsed)))


def select_layouts(slot_table, cmax: int, shares) -> list:
    """Restricted baselines: the layouts of this oracle's own enumeration whose
    slots are exactly the given (sm800, b8, dom) tuples, in the table's order.  A table entry
    that is not a valid hierarchical partition raises (so the baseline tables are pinned to the
    placement rules of R3/R4 and R23)."""
    full = enumerate_layouts(cmax, shares, True) + enumerate_layouts(cmax, shares, False)
    by_slots = {}
    for l in full:
        by_slots.setdefault(tuple((s.sm800, s.b8, s.dom) for s in l.slots), l)
    out = []
    for entry in slot_table:
        key = tuple(tuple(x) for x in entry)
        if key not in by_slots:
            raise ValueError(f"not a valid hierarchical partition: {entry}")
        out.append(by_slots[key])
    return out
