"""a2/a5/a7/a8/a9/a12/a13 -- state encoding, greedy / epsilon-greedy action selection, the
vectorised environment step, replay, and the double-DQN update (ORACLE, test infra only).

Paper: state = the W jobs of the window with their profile features; input layer
W x (f + 5) (Table VI); ComputeRatio / MemoryRatio / DurationRatio = job value over the
window mean; action = job set + partitioning; epsilon-greedy from 1 to 0.01,
random actions from the whole search space, epsilon = 0 online; Q-learning update
(P:178); duelling double DQN.  Experience replay and the vectorised env are
required by BASELINE.json's north star (not in the paper).

Readings: R10 the "+5" inputs = [c/cbar, m/mbar, T/Tbar, scheduled, U/W];
R12 hyper-parameters; R13 deterministic transitions; R14 random action = k-th valid action;
R15 fixed-point argmax with near-tie lockstep; R19 an episode = one window until every job is
scheduled, then auto-reset from the host stream.

Transition: s = (window, sched); a = (l, g, sigma) with g disjoint from sched;
s' = (window, sched | bits(g)); done iff every job is scheduled (each job exactly once).

Pins: tests/test_oracle_dqn.py -- epsilon = 1 -> every action is the k-th valid action,
epsilon = 0 -> greedy; the explicit argmax equals a brute-force max over decode(idx);
episodes schedule every job exactly once; replay index formula; the tabular special
case of the Q-update rule; gamma = 0 / done -> y = r.
"""
from __future__ import annotations

import itertools
import multiprocessing as mp

import numpy as np

from . import actions as A
from . import corun as CR
from . import pruned as PR
from . import qnet as QN

NEAR_TIE = 1e-4  # reading R15: argmax mismatch allowed iff oracle gap <= 1e-4 max(1, |Q|)
RELU_NEAR = 1e-4  # reading R25: ReLU' decision may differ iff |pre-activation| <= 1e-4 rms


class Tables:
    """Per-space enumeration tables in index order (plain products of itertools orders)."""

    def __init__(self, space):
        self.space = space
        self.off = A.offsets(space)
        W = space.W
        self.members = {}
        self.slot_of = {}
        self.gmask = {}
        for C in sorted({l.C for l in space.layouts}):
            mem, so, gm = [], [], []
            for g in itertools.combinations(range(W), C):
                m = A.group_mask(g)
                for sg in itertools.permutations(range(C)):
                    mem.append(g)
                    so.append(sg)
                    gm.append(m)
            self.members[C] = np.array(mem, np.int64).reshape(-1, C)
            self.slot_of[C] = np.array(so, np.int64).reshape(-1, C)
            self.gmask[C] = np.array(gm, np.uint64)


def encode(window, sched: int, pool, W: int) -> np.ndarray:
    """x = W rows of [features (f) | c/cbar, m/mbar, T/Tbar | scheduled | U/W]."""
    ids = [int(x) for x in window]
    c = np.array([float(pool.compute_pm[j]) for j in ids])
    m = np.array([float(pool.memory_pm[j]) for j in ids])
    T = np.array([float(pool.solo_ticks[j]) for j in ids])
    sbit = np.array([float((sched >> j) & 1) for j in range(W)])
    U = W - int(sbit.sum())
    rows = []
    for j in range(W):
        rows.append(np.concatenate([pool.features[ids[j]].astype(np.float64),
                                    [c[j] / c.mean(), m[j] / m.mean(), T[j] / T.mean(),
                                     sbit[j], U / W]]))
    return np.concatenate(rows)


def head_fixed(z, space):
    v, aL, aJ = QN.split_head(np.asarray(z, np.float64), space)
    cL, cJ = QN.center(aL, aJ)
    Fv = QN.fixed(v)
    FcL = [QN.fixed(x) for x in cL]
    FcJ = [[QN.fixed(x) for x in row] for row in cJ]
    return v, cL, cJ, Fv, FcL, FcJ


def greedy_explicit(tab: Tables, Fv, FcL, FcJ, sched: int):
    """argmax over every valid action of Q^ (exact integers), ties to the lowest index.
    Returns (idx, Q^max) or (-1, None) when no action is valid."""
    sp = tab.space
    FJ = np.array(FcJ, dtype=np.int64)
    assert np.abs(FJ).max(initial=0) < (1 << 58)
    best, best_idx = None, -1
    for l, lay in enumerate(sp.layouts):
        C = lay.C
        mem, so, gm = tab.members[C], tab.slot_of[C], tab.gmask[C]
        valid = (gm & np.uint64(sched)) == 0
        if not valid.any():
            continue
        types = np.array(sp.slot_type[l], np.int64)[so]          # [n][C]
        score = np.full(len(mem), FcL[l] + Fv, dtype=np.int64)
        for i in range(C):
            score += FJ[mem[:, i], types[:, i]]
        score = np.where(valid, score, np.iinfo(np.int64).min)
        k = int(np.argmax(score))                                 # first max = lowest idx
        s = int(score[k])
        if best is None or s > best:
            best, best_idx = s, tab.off[l] + k
    return best_idx, best


# -- all-core mode: the per-state argmax (the oracle's dominant cost) mapped over worker
# processes.  Each state's argmax is independent of every other, so this only changes where
# the same function runs, not what it computes.
_WORKER = {}


def _worker_init(space, argmax):
    if getattr(space, "seq", False):
        off = A.offsets(space)
        _WORKER["fn"] = lambda Fv, FcL, FcJ, s: greedy_seq(space, Fv, FcL, s, off)
    elif argmax == "pruned":
        off = A.offsets(space)
        _WORKER["fn"] = lambda Fv, FcL, FcJ, s: PR.greedy_pruned(space, Fv, FcL, FcJ, s, off)
    else:
        tab = Tables(space)
        _WORKER["fn"] = lambda Fv, FcL, FcJ, s: greedy_explicit(tab, Fv, FcL, FcJ, s)


def _worker_call(item):
    return _WORKER["fn"](*item)


class OracleDQN:
    """The vectorised DQN environment + agent of SURVEY §8(c) Q1-Q4, one rank.

    argmax: "explicit" (every valid action, env.greedy_explicit) or "pruned" (the exact top-C
    search of oracle/pruned.py, same result); workers > 1 maps the per-state argmax over that
    many processes (all-core mode; results are identical)."""

    def __init__(self, space, pool, net, theta0, n_envs, batch, replay_capacity,
                 gamma=0.99, lr=1e-3, reward_lambda=0.0, q3=1, greedy=None, argmax="explicit",
                 workers=0, optimizer="sgd", adam=(0.9, 0.999, 1e-8), loss="squared",
                 huber_kappa=1.0):
        self.sp = space
        self.pool = pool
        self.argmax = argmax
        self.workers = workers
        self._procs = None
        if greedy is None and getattr(space, "seq", False):
            off = A.offsets(space)
            greedy = lambda Fv, FcL, FcJ, s: greedy_seq(space, Fv, FcL, s, off)
        elif greedy is None and argmax == "pruned":
            off = A.offsets(space)
            greedy = lambda Fv, FcL, FcJ, s: PR.greedy_pruned(space, Fv, FcL, FcJ, s, off)
        self.custom_greedy = greedy is not None
        self.tab = Tables(space) if greedy is None else None
        self.greedy_fn = greedy or (lambda Fv, FcL, FcJ, sched:
                                    greedy_explicit(self.tab, Fv, FcL, FcJ, sched))
        self.off = A.offsets(space)
        self.dims = QN.net_dims(space, net)
        self.theta = np.asarray(theta0, np.float64).copy()
        self.theta_t = self.theta.copy()
        self.E, self.B, self.N = n_envs, batch, replay_capacity
        self.gamma, self.lr, self.lam, self.q3 = gamma, lr, reward_lambda, q3
        # Adam (Kingma & Ba, bias-corrected moments) instead of the plain
        # SGD step, Huber instead of (1/2) delta^2 (P:178 states neither; both are variants)
        self.optimizer, self.adam, self.loss_kind, self.kappa = optimizer, adam, loss, huber_kappa
        self.adam_m = np.zeros_like(self.theta)
        self.adam_v = np.zeros_like(self.theta)
        self.adam_t = 0
        self.windows = None
        self.sched = None
        self.rep_win = np.zeros((self.N, space.W), np.uint8)
        self.rep_sched = np.zeros(self.N, np.uint64)
        self.rep_act = np.zeros(self.N, np.int64)
        self.rep_r = np.zeros(self.N, np.float64)
        self.rep_done = np.zeros(self.N, np.uint8)
        self.inserted = 0
        self.t = 0
        self.near_ties = 0       # GPU argmax adopted under R15 (oracle gap within the window)
        self.near_tie_gap = 0.0  # largest adopted gap, in units of max(1, |Q|)
        self.greedy_calls = 0    # greedy argmaxes taken (the population near_ties is out of)
        self.relu_near = 0       # ReLU' decisions adopted under R25
        self.relu_decisions = 0  # ReLU' decisions compared (hidden units x samples)

    # -- helpers -----------------------------------------------------------------------
    def close(self):
        if self._procs is not None:
            self._procs.terminate()
            self._procs = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _greedy_many(self, items):
        """[(Fv, FcL, FcJ, sched)] -> [(idx, Q^max)], in order."""
        self.greedy_calls += len(items)
        if self.workers > 1 and not self.custom_greedy and len(items) > 1:
            if self._procs is None:
                ctx = mp.get_context("spawn")
                self._procs = ctx.Pool(self.workers, _worker_init, (self.sp, self.argmax))
            ch = max(1, len(items) // (4 * self.workers))
            return self._procs.map(_worker_call, items, chunksize=ch)
        return [self.greedy_fn(*it) for it in items]

    def _heads(self, theta, windows, scheds, pre=None):
        X = np.stack([encode(w, int(s), self.pool, self.sp.W) for w, s in zip(windows, scheds)])
        z, acts = QN.forward(theta, self.dims, X, pre)
        return z, acts

    def _adopt_masks(self, pre, gpu_masks):
        """Reading R25 (the R15 lockstep for ReLU'): the backward's mask [pre > 0] is decided in
        floating point; where the GPU's decision differs and the oracle's pre-activation is
        within RELU_NEAR x rms(layer) of zero, the oracle takes the GPU's decision (counted).
        Any other difference fails."""
        masks = []
        for l, (y, g) in enumerate(zip(pre, gpu_masks)):
            m = y > 0
            g = np.asarray(g, bool).reshape(m.shape)
            diff = m != g
            self.relu_decisions += m.size
            if diff.any():
                band = RELU_NEAR * max(1e-30, float(np.sqrt(np.mean(y ** 2))))
                far = diff & (np.abs(y) > band)
                if far.any():
                    b, j = np.argwhere(far)[0]
                    raise AssertionError(f"ReLU mask mismatch layer {l} sample {b} unit {j}: "
                                         f"oracle pre-activation {y[b, j]:.3e}, band {band:.3e}")
                self.relu_near += int(diff.sum())
            masks.append(g)
        return masks

    def _adopt(self, mine, theirs, Fv, FcL, FcJ, qmax, sched):
        """Near-tie lockstep (reading R15): adopt the GPU's action if our Q^ gap <= 1e-4."""
        if theirs is None or theirs == mine:
            return mine, 0
        theirs = int(theirs)
        l, g, sg = A.decode(self.sp, theirs, self.off)
        if A.group_mask(g) & sched:
            raise AssertionError(f"GPU chose invalid action {theirs}")
        if getattr(self.sp, "seq", False) and theirs != seq_action(self.sp, l, sched, self.off):
            raise AssertionError(f"GPU chose a non-sequential action {theirs}")
        qt = QN.q_fixed(Fv, FcL, FcJ, self.sp, l, g, sg)
        gap = (qmax - qt) / 4294967296.0
        rel = gap / max(1.0, abs(qmax / 4294967296.0))
        if rel <= NEAR_TIE:
            self.near_ties += 1
            self.near_tie_gap = max(self.near_tie_gap, rel)
            return theirs, 1
        raise AssertionError(f"argmax mismatch: oracle {mine} gpu {theirs} gap {gap}")

    # -- API mirrored by libhrp ---------------------------------------------------------
    def reset(self, windows):
        self.windows = np.array(windows, np.uint8).copy()
        self.sched = np.zeros(len(windows), np.uint64)

    def q_forward(self, windows, scheds, gpu_argmax=None):
        z, _ = self._heads(self.theta, windows, scheds)
        out_a, out_q = [], []
        hf = [head_fixed(z[b], self.sp) for b in range(len(windows))]
        res = self._greedy_many([(h[3], h[4], h[5], int(scheds[b])) for b, h in enumerate(hf)])
        for b in range(len(windows)):
            v, cL, cJ, Fv, FcL, FcJ = hf[b]
            a, q = res[b]
            if gpu_argmax is not None and a >= 0:
                a, _ = self._adopt(a, gpu_argmax[b], Fv, FcL, FcJ, q, int(scheds[b]))
                q = q_fixed_idx_any(self.sp, self.off, Fv, FcL, FcJ, a)
            out_a.append(a)
            out_q.append(q / 4294967296.0 if q is not None else float("nan"))
        return np.array(out_a, np.int64), np.array(out_q), z

    def env_step(self, thr, u_explore, u_action, next_windows, gpu_actions=None):
        E, sp = self.E, self.sp
        z, _ = self._heads(self.theta, self.windows, self.sched)
        acts = np.zeros(E, np.int64)
        rew = np.zeros(E)
        done = np.zeros(E, np.uint8)
        cor = np.zeros(E, np.int64)
        qsel = np.zeros(E)
        hf = [head_fixed(z[e], sp) for e in range(E)]
        greedy_e = [e for e in range(E) if not int(u_explore[e]) < int(thr)]
        res = dict(zip(greedy_e, self._greedy_many(
            [(hf[e][3], hf[e][4], hf[e][5], int(self.sched[e])) for e in greedy_e])))
        for e in range(E):
            sched = int(self.sched[e])
            v, cL, cJ, Fv, FcL, FcJ = hf[e]
            if int(u_explore[e]) < int(thr) and getattr(sp, "seq", False):
                vl = seq_valid_layouts(sp, sched)        # uniform over the valid setups
                a = seq_action(sp, vl[A.explore_k(int(u_action[e]), len(vl))], sched, self.off)
            elif int(u_explore[e]) < int(thr):
                nv = A.n_valid(sp, sched)
                a = A.kth_valid(sp, sched, A.explore_k(int(u_action[e]), nv), self.off)
            else:
                a, q = res[e]
                if gpu_actions is not None:
                    a, _ = self._adopt(a, gpu_actions[e], Fv, FcL, FcJ, q, sched)
            l, g, sg = A.decode(sp, a, self.off)
            assert A.group_mask(g) & sched == 0
            r, cr, solo = CR.reward(sp.layouts[l], g, sg, self.windows[e], self.pool,
                                    self.lam, self.q3)
            qsel[e] = QN.q_fixed(Fv, FcL, FcJ, sp, l, g, sg) / 4294967296.0
            s2 = sched | A.group_mask(g)
            d = int(s2 == (1 << sp.W) - 1)
            slot = (self.t * E + e) % self.N
            self.rep_win[slot] = self.windows[e]
            self.rep_sched[slot] = np.uint64(sched)
            self.rep_act[slot] = a
            self.rep_r[slot] = r
            self.rep_done[slot] = d
            acts[e], rew[e], done[e], cor[e] = a, r, d, cr
            if d:
                self.windows[e] = next_windows[e]
                self.sched[e] = np.uint64(0)
            else:
                self.sched[e] = np.uint64(s2)
        self.inserted += E
        self.t += 1
        return acts, rew, done, cor, qsel

    def sample(self, u_replay):
        nf = min(self.N, self.inserted)
        return np.array([(int(u) * nf) >> 32 for u in u_replay], np.int64)

    def dqn_update(self, u_replay, sync_target, gpu_astar=None, b_total=None, apply=True,
                   gpu_masks=None):
        """One double-DQN step on a replay batch.  Returns a dict with loss, idx, a*, y,
        Q(s,a), grad (sum-form / B_total).  With apply=False the caller applies the SGD
        step (multi-rank simulation).  gpu_masks: the GPU's ReLU' decisions of the s rows per
        hidden layer (bool [B][w]) for the near-zero lockstep of reading R25."""
        sp, B = self.sp, len(u_replay)
        b_total = b_total or B
        idx = self.sample(u_replay)
        win = self.rep_win[idx]
        sch = self.rep_sched[idx].astype(np.uint64)
        act = self.rep_act[idx]
        r = self.rep_r[idx]
        dn = self.rep_done[idx]
        dec = [A.decode(sp, int(a), self.off) for a in act]
        sch2 = np.array([int(s) | A.group_mask(g) for s, (_, g, _) in zip(sch, dec)],
                        np.uint64)
        pre = []
        z_s, acts = self._heads(self.theta, win, sch, pre)
        z_n, _ = self._heads(self.theta, win, sch2)
        z_t, _ = self._heads(self.theta_t, win, sch2)
        astar = np.full(B, -1, np.int64)
        y = np.zeros(B)
        q_sa = np.zeros(B)
        dz = np.zeros_like(z_s)
        live = [b for b in range(B) if not dn[b]]
        hf = {b: head_fixed(z_n[b], sp) for b in live}
        res = dict(zip(live, self._greedy_many(
            [(hf[b][3], hf[b][4], hf[b][5], int(sch2[b])) for b in live])))
        for b in range(B):
            if not dn[b]:
                v, cL, cJ, Fv, FcL, FcJ = hf[b]
                a2, q2 = res[b]
                if gpu_astar is not None:
                    a2, _ = self._adopt(a2, gpu_astar[b], Fv, FcL, FcJ, q2, int(sch2[b]))
                astar[b] = a2
                vt, aLt, aJt = QN.split_head(z_t[b], sp)
                cLt, cJt = QN.center(aLt, aJt)
                l2, g2, s2 = A.decode(sp, int(a2), self.off)
                qt = QN.q_value(vt, cLt, cJt, sp, l2, g2, s2)
                y[b] = r[b] + self.gamma * qt
            else:
                y[b] = r[b]
            v, aL, aJ = QN.split_head(z_s[b], sp)
            cL, cJ = QN.center(aL, aJ)
            l, g, sg = dec[b]
            q_sa[b] = QN.q_value(v, cL, cJ, sp, l, g, sg)
            dz[b] = QN.dq_dz(sp, l, g, sg) * self._dloss(q_sa[b] - y[b]) / b_total
        delta = q_sa - y
        loss = float(sum(self._loss_term(d) for d in delta) / B)
        masks = self._adopt_masks(pre, gpu_masks) if gpu_masks is not None else None
        grad = QN.backward(self.theta, self.dims, acts, dz, masks)
        if apply:
            self.apply(grad, sync_target)
        return {"loss": loss, "idx": idx, "astar": astar, "y": y, "q_sa": q_sa,
                "grad": grad}

    def _loss_term(self, d):
        """(1/2) delta^2, or Huber: delta^2 / 2 if |delta| <= kappa, else
        kappa (|delta| - kappa / 2)."""
        d = float(d)
        if self.loss_kind == "huber" and abs(d) > self.kappa:
            return self.kappa * (abs(d) - 0.5 * self.kappa)
        return 0.5 * d * d

    def _dloss(self, d):
        """d(loss term)/d delta: delta, or clip(delta, -kappa, kappa) for Huber."""
        if self.loss_kind == "huber":
            return float(np.clip(d, -self.kappa, self.kappa))
        return float(d)

    def apply(self, grad, sync_target):
        if self.optimizer == "adam":
            b1, b2, eps = self.adam
            self.adam_t += 1
            self.adam_m = b1 * self.adam_m + (1 - b1) * grad
            self.adam_v = b2 * self.adam_v + (1 - b2) * grad * grad
            mh = self.adam_m / (1 - b1 ** self.adam_t)
            vh = self.adam_v / (1 - b2 ** self.adam_t)
            self.theta = self.theta - self.lr * mh / (np.sqrt(vh) + eps)
        else:
            self.theta = self.theta - self.lr * grad
        if sync_target:
            self.theta_t = self.theta.copy()


def q_fixed_idx_any(space, off, Fv, FcL, FcJ, idx):
    l, g, sg = A.decode(space, int(idx), off)
    return QN.q_fixed(Fv, FcL, FcJ, space, l, g, sg)


# -- the sequential agent (reading R28) -------------------------------
# The paper's agent has V = 1 and A = 29 outputs (Table VI): one advantage per partition
# setup.  Reading: the job set is the next C unscheduled jobs of the window in queue order
# (first-come), member i on slot i; the agent chooses the setup l (C_l <= U).  The joint
# action index of that (l, g, identity) keeps the reward, transition and replay of the joint
# agent unchanged.

def seq_action(space, l, sched, off=None):
    free = [j for j in range(space.W) if not (sched >> j) & 1]
    C = space.layouts[l].C
    return A.action_index(space, l, tuple(free[:C]), tuple(range(C)), off)


def seq_valid_layouts(space, sched):
    U = space.W - bin(sched).count("1")
    return [l for l, lay in enumerate(space.layouts) if lay.C <= U]


def greedy_seq(space, Fv, FcL, sched, off=None):
    """argmax over the valid setups of Q^ = F(v) + F(cL[l]), ties to the lowest l (= the lowest
    joint index).  Returns (idx, Q^max)."""
    best, bl = None, -1
    for l in seq_valid_layouts(space, sched):
        q = Fv + FcL[l]
        if best is None or q > best:
            best, bl = q, l
    return (seq_action(space, bl, sched, off) if bl >= 0 else -1), best


def greedy_bruteforce(space, Fv, FcL, FcJ, sched):
    """Literal definition for tiny spaces: decode every index, keep the first maximum."""
    off = A.offsets(space)
    best, bi = None, -1
    for idx in range(off[-1]):
        l, g, sg = A.decode(space, idx, off)
        if A.group_mask(g) & sched:
            continue
        q = QN.q_fixed(Fv, FcL, FcJ, space, l, g, sg)
        if best is None or q > best:
            best, bi = q, idx
    return bi, best


__all__ = ["Tables", "encode", "head_fixed", "greedy_explicit", "greedy_bruteforce",
           "OracleDQN", "NEAR_TIE"]
