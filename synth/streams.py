"""Seeded windows, per-step random streams and initial weights (input generator only).

Streams are numpy Philox4x32-10 (counter-based): key = (SEED + stream) + (rank << 40) +
(step << 64), so every (stream, rank, step) triple is an independent, reproducible stream.
"""
from __future__ import annotations

import numpy as np

SEED = 240508754  # arXiv id 2405.08754
S_PROFILES, S_WINDOWS, S_EXPLORE, S_ACTION, S_REPLAY, S_INIT, S_STATES = range(7)


def philox(seed: int, step: int = 0, rank: int = 0) -> np.random.Generator:
    key = (int(seed) + (int(rank) << 40) + (int(step) << 64)) & ((1 << 128) - 1)
    return np.random.Generator(np.random.Philox(key=key))


def _class_template(W: int, cat: int) -> np.ndarray:
    """Class of each window slot for job-mix category cat (reading R18):
    0 CI-, 1 MI-, 2 US-dominant: ceil(W/2) of the dominant class, the rest round-robin over
    the other two classes; 3 Balanced: round-robin over CI, MI, US."""
    if cat == 3:
        return np.array([k % 3 for k in range(W)], np.int8)
    dom = cat
    others = [c for c in range(3) if c != dom]
    nd = (W + 1) // 2
    return np.array([dom] * nd + [others[k % 2] for k in range(W - nd)], np.int8)


def make_windows(pool, n: int, W: int, seed: int = None, step: int = 0, rank: int = 0,
                 first_env: int = 0) -> np.ndarray:
    """n class-stratified windows of W pool ids (uint8 [n][W]).  Env e (global index
    first_env + i) uses category e mod 4; jobs are drawn uniformly within their class with
    replacement, then the window's positions are shuffled."""
    g = philox(SEED + S_WINDOWS if seed is None else seed, step, rank)
    members = [np.nonzero(pool.classes == c)[0] for c in range(3)]
    cats = (first_env + np.arange(n)) % 4
    cls = np.stack([_class_template(W, int(c)) for c in range(4)])[cats]  # [n][W]
    cls = g.permuted(cls, axis=1)
    ids = np.empty((n, W), np.int64)
    for c in range(3):
        mask = cls == c
        draws = g.integers(0, len(members[c]), size=int(mask.sum()))
        ids[mask] = members[c][draws]
    return ids.astype(np.uint8)


def table_v_windows(pool) -> np.ndarray:
    """Q1..Q12 of Table V as pool ids, uint8 [12][12]."""
    from .pool import TABLE_V
    return np.array([[pool.index(nm) for nm in TABLE_V[f"Q{i}"]] for i in range(1, 13)],
                    np.uint8)


def step_streams(step: int, E: int, B: int, W: int, pool, rank: int = 0,
                 first_env: int = 0) -> dict:
    """The host-generated per-step inputs of one DQN step (SURVEY.md §8(c) parity protocol):
    u_explore u32[E], u_action u64[E], u_replay u32[B], next_windows u8[E][W]."""
    ge = philox(SEED + S_EXPLORE, step, rank)
    ga = philox(SEED + S_ACTION, step, rank)
    gr = philox(SEED + S_REPLAY, step, rank)
    return {
        "u_explore": ge.integers(0, 1 << 32, size=E, dtype=np.uint64).astype(np.uint32),
        "u_action": ga.integers(0, 1 << 64, size=E, dtype=np.uint64, endpoint=False),
        "u_replay": gr.integers(0, 1 << 32, size=B, dtype=np.uint64).astype(np.uint32),
        "next_windows": make_windows(pool, E, W, step=step + 1, rank=rank,
                                     first_env=first_env),
    }


def eps_threshold(t: int, n_decay: int, eps_min: float = 0.01) -> int:
    """Epsilon-greedy schedule of PAPER.md:242 (from 1 down to 0.01), as the integer
    threshold thr = floor(eps * 2^32) in [0, 2^32]; explore iff u32 < thr."""
    eps = max(eps_min, 1.0 - (1.0 - eps_min) * t / max(1, n_decay))
    return int(np.floor(eps * 4294967296.0))


def init_weights(dims: list, seed: int = SEED + S_INIT) -> np.ndarray:
    """Initial Q-network parameters, flat fp32: for each Linear layer l (dims[l] ->
    dims[l+1]) W_l [out][in] row-major, then b_l [out].  Kaiming-uniform for hidden
    layers (bound sqrt(6/in)), PyTorch-default bound 1/sqrt(in) for the head and biases."""
    g = philox(seed)
    out = []
    nl = len(dims) - 1
    for l in range(nl):
        fi, fo = dims[l], dims[l + 1]
        bw = np.sqrt(6.0 / fi) if l < nl - 1 else 1.0 / np.sqrt(fi)
        out.append(g.uniform(-bw, bw, size=fi * fo))
        bb = 1.0 / np.sqrt(fi)
        out.append(g.uniform(-bb, bb, size=fo))
    return np.concatenate(out).astype(np.float32)


def sched_states(n: int, W: int, seed: int = SEED + S_STATES, step: int = 0,
                 rank: int = 0) -> np.ndarray:
    """Scheduled-job masks for inference states: U ~ U[1, W] jobs left unscheduled, the
    scheduled ones a uniform random subset (uint64 [n])."""
    g = philox(seed, step, rank)
    U = g.integers(1, W + 1, size=n)
    keys = g.random((n, W))
    order = np.argsort(keys, axis=1)
    sched = np.zeros(n, np.uint64)
    pos = np.arange(W)
    for k in range(W):
        col = order[:, k]
        take = k >= U  # positions after the first U in random order are scheduled
        sched |= np.where(take, np.left_shift(np.uint64(1), col.astype(np.uint64)),
                          np.uint64(0)).astype(np.uint64)
    del pos
    return sched
