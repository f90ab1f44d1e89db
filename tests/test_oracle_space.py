"""Pins for oracle/space.py (a1) -- checked against PAPER.md statements, not against itself."""
import os
from fractions import Fraction
from math import comb, factorial

import pytest

from oracle import space as SP
from oracle import actions as A

S10 = tuple(range(10, 100, 10))
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "table7.txt")


def test_nineteen_gi_variants():
    # P:64 "the partitioning choices are limited only to 19 variants"
    gis = SP.gi_configs()
    assert len(gis) == 19
    # 7 GPCs cannot be split 2+5 or 1+6
    for cfg in gis:
        sizes = sorted(g for _, g in cfg)
        assert sizes not in ([2, 5], [1, 6])
        assert sum(g for _, g in cfg) <= 7   # one GPC disabled


def test_independent_placement_search_counts():
    # independent brute force over all 2^14 subsets of the GI placement table
    pl = SP.gi_placements()
    valid, maximal = [], []
    for mask in range(1, 1 << len(pl)):
        sel = [pl[i] for i in range(len(pl)) if mask >> i & 1]
        mem = [0] * 8
        ok = sum(g for _, g in sel) <= 7
        for s, g in sel:
            for x in range(s, s + SP.GI_PROFILES[g][0]):
                mem[x] += 1
        ok = ok and max(mem) <= 1
        if ok:
            valid.append(mask)
    vs = set(valid)
    for m in valid:
        if not any((m | 1 << i) in vs for i in range(len(pl)) if not m >> i & 1):
            maximal.append(m)
    assert len(maximal) == 19
    assert len(valid) == len(SP.gi_configs(maximal_only=False))


def test_mig_compute_total_and_share_sums():
    for W, cmax, S in [(4, 2, (25, 50, 75)), (16, 3, S10), (12, 4, S10)]:
        sp = SP.build_space(W, cmax, S)
        for lay in sp.layouts:
            tot = Fraction(sum(s.sm800 for s in lay.slots), 800)
            if lay.mig:
                assert tot <= Fraction(7, 8)      # P:102 "87.5% in each case"
            else:
                assert tot == 1
            for comp in lay.comps:
                assert sum(comp) == 100           # MPS shares inside a CI sum to 100%
            assert 1 <= lay.C <= cmax
            doms = {s.dom for s in lay.slots}
            for d in doms:
                b8s = {s.b8 for s in lay.slots if s.dom == d}
                assert len(b8s) == 1              # CIs of a GI share its memory
            assert sum(next(s.b8 for s in lay.slots if s.dom == d) for d in doms) <= 8


def _golden():
    out = []
    with open(GOLDEN) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            C, yes, text = line.split(None, 2)
            out.append((int(C), yes == "yes", text))
    return out


@pytest.mark.parametrize("cmax", [3, 4])
def test_table7_members(cmax):
    # Table VII: explicit entries with C <= Cmax are in the layout set
    sp = SP.build_space(12, cmax, S10)
    have = {SP.canonical(l) for l in sp.layouts}
    for C, yes, text in _golden():
        if C > cmax:
            continue
        assert (SP.parse_notation(text) in have) == yes, text


def test_table7_mps_only_c2_count():
    # the MPS-only C=2 list runs (0.1)+(0.9) ... (0.5)+(0.5): 5 unordered splits
    sp = SP.build_space(12, 2, S10, mig=False)
    assert sum(1 for l in sp.layouts if l.C == 2) == 5


def test_notation_round_trip():
    sp = SP.build_space(12, 4, S10)
    for lay in sp.layouts:
        assert SP.parse_notation(lay.notation()) == SP.canonical(lay)


def test_config1_layouts_hand_listed():
    # Config 1 (W=4, Cmax=2, S={25,50,75}): enumerated by hand from P:64-66 + reading R3-R5
    sp = SP.build_space(4, 2, (25, 50, 75))
    got = sorted(tuple(sorted((s.sm800, s.b8) for s in l.slots)) + (len({s.dom for s in l.slots}),)
                 for l in sp.layouts)
    want = sorted([
        ((800, 8), 1),                         # MIG off, one job on the whole GPU
        ((200, 8), (600, 8), 1),               # MPS 25/75
        ((400, 8), (400, 8), 1),               # MPS 50/50
        ((700, 8), 1),                         # 7g GI, 7c CI
        ((175, 8), (525, 8), 1),               # 7g/7c + MPS 25/75
        ((350, 8), (350, 8), 1),               # 7g/7c + MPS 50/50
        ((300, 8), (400, 8), 1),               # [{0.375}+{0.5},1m]
        ((300, 4), (300, 4), 2),               # 3g + 3g
        ((300, 4), (400, 4), 2),               # [{0.375},0.5m]+[{0.5},0.5m]
    ])
    assert got == want
    assert sp.T == 11 and sp.H == 1 + 9 + 4 * 11


@pytest.mark.parametrize("W,cmax,S,mig", [(4, 2, (25, 50, 75), True), (16, 3, S10, True),
                                          (12, 4, S10, True), (64, 4, S10, True),
                                          (12, 4, S10, False)])
def test_action_count_closed_form(W, cmax, S, mig):
    # max count = sum_{C=2}^{Cmax} binom(W,C) C! N_C ; plus the C=1 term (reading R2)
    sp = SP.build_space(W, cmax, S, mig)
    NC = {C: sum(1 for l in sp.layouts if l.C == C) for C in range(1, cmax + 1)}
    closed = sum(comb(W, C) * factorial(C) * NC[C] for C in range(1, cmax + 1))
    assert A.n_actions(sp) == closed


def test_config_sizes_survey_table():
    # sizes quoted in SURVEY.md §8(a) for the BASELINE.json configs
    assert A.n_actions(SP.build_space(4, 2, (25, 50, 75))) == 92
    sp2 = SP.build_space(16, 3, S10)
    assert (sp2.L, sp2.T, sp2.H, A.n_actions(sp2)) == (71, 52, 904, 191312)
    sp3 = SP.build_space(12, 4, S10)
    assert (sp3.L, sp3.T, A.n_actions(sp3)) == (386, 78, 3817860)
    sp4 = SP.build_space(64, 4, S10)
    assert (sp4.H, A.n_actions(sp4)) == (5379, 4817494208)
