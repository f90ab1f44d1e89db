"""Synthetic job-profile pool (input generator; no method arithmetic).

Program names and classes: Table IV.  Unseen programs ("*"): PAPER.md:209.
Job mixes Q1-Q12: Table V; "qs_Coral_Pl" is read as
qs_Coral_P1 (reading R22).

Per-profile quantities (SURVEY.md §8(c) "Synthetic profiles"):
  T  solo-run time in ticks (1 tick = 1 us), T = floor(2^(17 + 7u))
  c  "Compute (SM) [%]" in permille, m  "Memory [%]" in permille (Table III counters)
  CI: c ~ U[600, 950], m ~ U[150, 700)     MI: m ~ U[600, 950], c ~ U[100, 0.8 m)
  US: c, m ~ U[30, 130]
and the 12 Table III counters derived from (T, c, m) plus Philox noise,
log1p on the count-like columns, z-scored over the pool, stored as fp32.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .streams import SEED, philox

# Table IV.  Order inside a class is the table's order.
TABLE_IV = {
    "CI": ["lavaMD", "huffman", "hotspot3D", "hotspot", "heartwall",
           "bt_solver_A", "bt_solver_B", "bt_solver_C"],
    "MI": ["lud_A", "lud_B", "lud_C", "sp_solver_A", "sp_solver_B", "sp_solver_C",
           "randomaccess", "cfd", "gaussian", "stream"],
    "US": ["kmeans", "dwt2d", "needle", "pathfinder", "backprop",
           "qs_Coral_P1", "qs_Coral_P2", "qs_NoFission", "qs_NoCollisions"],
}
# Programs marked "*" in Table IV (unseen in training).
UNSEEN = {"huffman", "hotspot", "heartwall", "lud_C", "cfd", "gaussian", "needle",
          "backprop", "qs_NoFission"}

# Table V, in the table's job order.
TABLE_V = {
    "Q1": ["huffman", "bt_solver_C", "bt_solver_B", "hotspot3D", "heartwall", "lavaMD",
           "lud_B", "cfd", "sp_solver_B", "pathfinder", "needle", "qs_NoFission"],
    "Q2": ["bt_solver_C", "heartwall", "lavaMD", "huffman", "hotspot", "hotspot3D", "cfd",
           "sp_solver_C", "gaussian", "pathfinder", "needle", "qs_Coral_P1"],
    "Q3": ["huffman", "bt_solver_C", "hotspot3D", "hotspot", "heartwall", "lavaMD", "lud_B",
           "stream", "sp_solver_C", "qs_NoFission", "pathfinder", "needle"],
    "Q4": ["bt_solver_B", "heartwall", "bt_solver_C", "lud_B", "gaussian", "sp_solver_B",
           "cfd", "sp_solver_C", "stream", "qs_NoCollisions", "pathfinder", "qs_Coral_P2"],
    "Q5": ["heartwall", "hotspot", "bt_solver_B", "lud_B", "gaussian", "randomaccess",
           "stream", "lud_C", "sp_solver_B", "qs_Coral_P2", "dwt2d", "qs_Coral_P1"],
    "Q6": ["bt_solver_C", "huffman", "lavaMD", "sp_solver_B", "gaussian", "randomaccess",
           "lud_C", "stream", "cfd", "qs_NoFission", "needle", "qs_Coral_P1"],
    "Q7": ["heartwall", "hotspot", "hotspot3D", "gaussian", "stream", "lud_B", "pathfinder",
           "qs_NoFission", "qs_Coral_P2", "backprop", "qs_NoCollisions", "dwt2d"],
    "Q8": ["bt_solver_C", "hotspot3D", "lavaMD", "stream", "cfd", "lud_B", "qs_Coral_P1",
           "needle", "kmeans", "qs_Coral_P2", "qs_NoFission", "qs_NoCollisions"],
    "Q9": ["lavaMD", "hotspot3D", "hotspot", "sp_solver_B", "lud_C", "randomaccess",
           "qs_Coral_P1", "dwt2d", "kmeans", "needle", "qs_NoCollisions", "qs_Coral_P2"],
    "Q10": ["lavaMD", "huffman", "hotspot3D", "bt_solver_C", "lud_C", "lud_B", "stream",
            "sp_solver_C", "qs_NoCollisions", "needle", "pathfinder", "qs_Coral_P1"],
    "Q11": ["huffman", "hotspot3D", "hotspot", "bt_solver_B", "cfd", "lud_C", "stream",
            "gaussian", "qs_Coral_P2", "needle", "pathfinder", "dwt2d"],
    "Q12": ["lavaMD", "hotspot", "huffman", "heartwall", "sp_solver_C", "lud_C",
            "randomaccess", "gaussian", "needle", "pathfinder", "qs_NoCollisions", "backprop"],
}
CLASSES = ("CI", "MI", "US")
N_FEATURES = 12  # Table III lists 12 counters


@dataclass
class Pool:
    """The profile table handed to hrp_env_create / the oracle (host arrays)."""
    names: list
    classes: np.ndarray      # int8 [P]: 0 CI, 1 MI, 2 US
    solo_ticks: np.ndarray   # int64 [P]
    compute_pm: np.ndarray   # int16 [P] Compute (SM) [%] in permille
    memory_pm: np.ndarray    # int16 [P] Memory [%] in permille
    features: np.ndarray     # float32 [P][12], z-scored

    @property
    def n(self) -> int:
        return len(self.names)

    def index(self, name: str) -> int:
        return self.names.index(name)


def class_counts(P: int) -> tuple:
    """Class split of a pool of P programs: Table IV's 8:10:9 (27) mix scaled (P=256 ->
    76/95/85)."""
    if P == 27:
        return (8, 10, 9)
    ci = int(round(P * 8 / 27))
    mi = int(round(P * 10 / 27))
    return (ci, mi, P - ci - mi)


def make_pool(P: int = 27, seed: int = SEED + 0) -> Pool:
    """Generate the synthetic pool.  P=27 uses the Table IV names/classes; larger pools
    repeat the class mix with suffixed names."""
    g = philox(seed)
    if P == 27:
        names = TABLE_IV["CI"] + TABLE_IV["MI"] + TABLE_IV["US"]
        classes = np.array([0] * 8 + [1] * 10 + [2] * 9, dtype=np.int8)
    else:
        nci, nmi, nus = class_counts(P)
        names, cl = [], []
        for k, (cname, cnt) in enumerate(zip(CLASSES, (nci, nmi, nus))):
            base = TABLE_IV[cname]
            for i in range(cnt):
                names.append(f"{base[i % len(base)]}#{i // len(base)}")
                cl.append(k)
        classes = np.array(cl, dtype=np.int8)
    c = np.zeros(P, np.int64)
    m = np.zeros(P, np.int64)
    T = np.zeros(P, np.int64)
    for i in range(P):
        u = g.random(3)
        if classes[i] == 0:      # CI
            c[i] = int(np.floor(600 + 350 * u[0]))
            m[i] = int(np.floor(150 + 550 * u[1]))
        elif classes[i] == 1:    # MI
            m[i] = int(np.floor(600 + 350 * u[1]))
            c[i] = int(np.floor(100 + (0.8 * m[i] - 100) * u[0]))
        else:                    # US
            c[i] = int(np.floor(30 + 100 * u[0]))
            m[i] = int(np.floor(30 + 100 * u[1]))
        T[i] = int(np.floor(2.0 ** (17 + 7 * u[2])))
    feats = _features(g, T, c, m)
    return Pool(names=names, classes=classes, solo_ticks=T,
                compute_pm=c.astype(np.int16), memory_pm=m.astype(np.int16), features=feats)


def _features(g, T, c, m) -> np.ndarray:
    """The 12 Table III counters in table order, synthesised."""
    P = len(T)
    u = g.random((P, 8))
    dur = T.astype(np.float64)
    mem = m / 10.0
    elapsed = 1.41 * dur
    grid = 2.0 ** (7 + 13 * u[:, 0])
    regs = 16 + np.floor(240 * u[:, 1])
    dram = mem * (0.8 + 0.2 * u[:, 2])
    l1 = 10 + 80 * u[:, 3]
    l2 = np.minimum(100.0, mem * (0.5 + 0.7 * u[:, 4]))
    smact = elapsed * (0.5 + 0.5 * u[:, 5])
    comp = c / 10.0
    waves = grid / (108 * (1 + np.floor(8 * u[:, 6])))
    warps = 8 + 56 * u[:, 7]
    F = np.stack([dur, mem, elapsed, grid, regs, dram, l1, l2, smact, comp, waves, warps], 1)
    for col in (0, 2, 3, 8, 10):  # count-like columns
        F[:, col] = np.log1p(F[:, col])
    mu = F.mean(0)
    sd = F.std(0)
    sd[sd == 0] = 1.0
    return ((F - mu) / sd).astype(np.float32)
