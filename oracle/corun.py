"""a6 -- co-run performance model and rewards (ORACLE, test infrastructure only).

Paper: CoRunTime(JS, R) = total execution time when co-locating JS with R; SoloRunTime(JS) =
total time with time sharing (Table I).  Feasibility CoRun <= Solo.
Final reward r_f = (SoloRunTime/CoRunTime - 1) x 100; intermediate reward
r_i = (SmAllocRatio x ComputeRatio + MemoryAllocRatio x MemoryRatio) x DurationRatio^2
(Table VI; ratios defined at P:240).  The paper measures co-runs on an A100;
here the measurement is replaced by the integer model of reading R8:

  slot k hosts job p (solo ticks T, compute c, memory m in permille) with compute share sm800
  (1/800 GPU) and memory b8 (1/8 GPU) in domain d; D_d = sum of m over the domain's jobs,
  n_d = #jobs in the domain, q = interference numerator in 1/8 units (default 1):
    t_k = max( ceil(T * max(5 sm800, 4 c) / (5 sm800)),
               ceil(T * max(1000 b8, D_d (8 + q (n_d - 1))) / (1000 b8)) )
  i.e. T x max(1, c/sigma, (D/beta)(1 + q (n-1)/8)),  sigma = sm800/800, beta = b8/8.
  CoRun = max_k t_k (makespan, reading R7), Solo = sum_k T_k.

Pins: tests/test_oracle_corun.py -- time sharing (singleton on the whole GPU) gives ratio
exactly 1 and r_f = 0; the class rule of P:189/P:207 reproduces the pool's
Table IV classes; hand-computed 2-job MPS / MIG cases; r_f, r_i closed forms on literals.
"""
from __future__ import annotations

from fractions import Fraction


def ceil_div(a: int, b: int) -> int:
    return -((-a) // b)


def slot_time(T: int, c: int, sm800: int, b8: int, D: int, n: int, q3: int = 1) -> int:
    comp = ceil_div(T * max(5 * sm800, 4 * c), 5 * sm800)
    mem = ceil_div(T * max(1000 * b8, D * (8 + q3 * (n - 1))), 1000 * b8)
    return max(comp, mem)


def corun(layout, jobs_on_slots, pool, q3: int = 1):
    """jobs_on_slots[k] = pool id hosted on slot k.  Returns (t list, CoRun, Solo)."""
    T = pool.solo_ticks
    c = pool.compute_pm
    m = pool.memory_pm
    D = {}
    n = {}
    for s, p in zip(layout.slots, jobs_on_slots):
        D[s.dom] = D.get(s.dom, 0) + int(m[p])
        n[s.dom] = n.get(s.dom, 0) + 1
    t = [slot_time(int(T[p]), int(c[p]), s.sm800, s.b8, D[s.dom], n[s.dom], q3)
         for s, p in zip(layout.slots, jobs_on_slots)]
    return t, max(t), sum(int(T[p]) for p in jobs_on_slots)


def assign(layout, g, sigma, window):
    """Pool id hosted on each slot for action members g (window positions) and sigma."""
    jobs = [None] * layout.C
    for i, gi in enumerate(g):
        jobs[sigma[i]] = int(window[gi])
    return jobs


def r_final(solo: int, corun_t: int) -> float:
    """r_f = (SoloRunTime / CoRunTime - 1) x 100 (Table VI)."""
    return (solo / corun_t - 1.0) * 100.0


def r_intermediate(slot, p: int, window, pool) -> float:
    """r_i of one job (Table VI, ratios of P:240): SmAllocRatio = sm800/800,
    MemoryAllocRatio = b8/8; Compute/Memory/Duration ratio = job value / window mean."""
    ids = [int(x) for x in window]
    cbar = sum(int(pool.compute_pm[j]) for j in ids) / len(ids)
    mbar = sum(int(pool.memory_pm[j]) for j in ids) / len(ids)
    tbar = sum(int(pool.solo_ticks[j]) for j in ids) / len(ids)
    return ((slot.sm800 / 800.0) * (int(pool.compute_pm[p]) / cbar)
            + (slot.b8 / 8.0) * (int(pool.memory_pm[p]) / mbar)) * \
        (int(pool.solo_ticks[p]) / tbar) ** 2


def reward(layout, g, sigma, window, pool, lam: float = 0.0, q3: int = 1):
    """Returns (r, CoRun, Solo): r = r_f + lam * sum_k r_i (reading R9)."""
    jobs = assign(layout, g, sigma, window)
    _, cr, solo = corun(layout, jobs, pool, q3)
    r = r_final(solo, cr)
    if lam != 0.0:
        r += lam * sum(r_intermediate(s, p, window, pool) for s, p in zip(layout.slots, jobs))
    return r, cr, solo


def app_class(T: int, c: int, m: int) -> int:
    """Class rule of P:189 / P:207: US if the 1-GPC private-memory run loses < 10% vs the
    full 8-GPC run; else CI if Compute%/Memory% > 0.80; else MI.  (0 CI, 1 MI, 2 US)"""
    full = slot_time(T, c, 800, 8, m, 1)
    one = slot_time(T, c, 100, 1, m, 1)
    if Fraction(one, full) < Fraction(11, 10):
        return 2
    return 0 if Fraction(c, m) > Fraction(8, 10) else 1
