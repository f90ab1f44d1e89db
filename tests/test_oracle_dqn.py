"""Pins for oracle/env.py (encode, argmax, epsilon-greedy step, replay, DQN update)."""
import numpy as np
import pytest

import synth
from oracle import actions as A
from oracle import env as EV
from oracle import qnet as QN
from oracle import space as SP
from synth.configs import NetCfg


def _rand_heads(sp, rng, ties=True):
    Fv = int(rng.integers(-5, 5))
    hi = 4 if ties else 1 << 20
    FcL = [int(x) for x in rng.integers(-hi, hi, sp.L)]
    FcJ = [[int(x) for x in row] for row in rng.integers(-hi, hi, (sp.W, sp.T))]
    return Fv, FcL, FcJ


@pytest.mark.parametrize("W,cmax,S", [(4, 2, (25, 50, 75)), (5, 3, (25, 50, 75)),
                                      (4, 4, (50,))])
def test_explicit_argmax_equals_literal(W, cmax, S):
    # literal definition: decode every index, keep the first maximum over valid ones
    sp = SP.build_space(W, cmax, S)
    tab = EV.Tables(sp)
    rng = np.random.default_rng(3)
    for _ in range(40):
        Fv, FcL, FcJ = _rand_heads(sp, rng)
        sched = int(rng.integers(0, (1 << W) - 1))
        assert EV.greedy_explicit(tab, Fv, FcL, FcJ, sched) == \
            EV.greedy_bruteforce(sp, Fv, FcL, FcJ, sched)


def test_encode_layout_and_ratios():
    pool = synth.make_pool(27)
    win = [0, 9, 20, 3]
    x = EV.encode(win, 0b0101, pool, 4).reshape(4, 17)
    np.testing.assert_array_equal(x[:, :12], pool.features[win].astype(np.float64))
    c = pool.compute_pm[win].astype(float)
    np.testing.assert_allclose(x[:, 12], c / c.mean())
    assert x[:, 12].mean() == pytest.approx(1.0)   # ratio to the window mean
    assert x[:, 13].mean() == pytest.approx(1.0)
    assert x[:, 14].mean() == pytest.approx(1.0)
    assert list(x[:, 15]) == [1, 0, 1, 0]
    assert list(x[:, 16]) == [0.5] * 4


def _agent(cfgk=1, E=16, B=8, net=None, lam=0.0, gamma=0.99, lr=1e-3, W=None):
    cfg = synth.config(cfgk)
    sc = cfg.space
    sp = SP.build_space(W or sc.window, sc.cmax, sc.shares)
    pool = synth.make_pool(cfg.pool)
    net = net or cfg.net
    dims = QN.net_dims(sp, net)
    theta = synth.init_weights(dims)
    ag = EV.OracleDQN(sp, pool, net, theta, E, B, 1 << 10, gamma=gamma, lr=lr,
                      reward_lambda=lam)
    ag.reset(synth.make_windows(pool, E, sp.W))
    return ag, sp, pool


def test_episodes_schedule_every_job_exactly_once():
    # the job sets partition Q (each job exactly once), 1 <= C_i <= Cmax
    ag, sp, pool = _agent(E=24)
    W = sp.W
    used = [0] * ag.E
    finished = 0
    for t in range(12):
        st = synth.step_streams(t, ag.E, ag.B, W, pool)
        thr = synth.eps_threshold(t, 6)
        win_before = ag.windows.copy()
        a, r, d, cr, q = ag.env_step(thr, st["u_explore"], st["u_action"],
                                     st["next_windows"])
        for e in range(ag.E):
            l, g, s = A.decode(sp, int(a[e]))
            m = A.group_mask(g)
            assert used[e] & m == 0
            assert 1 <= len(g) <= sp.cmax
            used[e] |= m
            if d[e]:
                assert used[e] == (1 << W) - 1
                used[e] = 0
                finished += 1
                np.testing.assert_array_equal(ag.windows[e], st["next_windows"][e])
            else:
                np.testing.assert_array_equal(ag.windows[e], win_before[e])
    assert finished > 0


def test_epsilon_one_is_kth_valid_and_zero_is_greedy():
    ag, sp, pool = _agent(E=16)
    st = synth.step_streams(0, ag.E, ag.B, sp.W, pool)
    a1, *_ = ag.env_step(1 << 32, st["u_explore"], st["u_action"], st["next_windows"])
    for e in range(ag.E):
        nv = A.n_valid(sp, 0)
        assert a1[e] == A.kth_valid(sp, 0, A.explore_k(int(st["u_action"][e]), nv))
    # eps = 0: every action is the argmax of the online net
    ag2, sp, pool = _agent(E=16)
    z, _ = ag2._heads(ag2.theta, ag2.windows, ag2.sched)
    a0, *_ = ag2.env_step(0, st["u_explore"], st["u_action"], st["next_windows"])
    for e in range(ag2.E):
        _, _, _, Fv, FcL, FcJ = EV.head_fixed(z[e], sp)
        assert a0[e] == EV.greedy_bruteforce(sp, Fv, FcL, FcJ, 0)[0]


def test_replay_sample_index_uniform():
    ag, sp, pool = _agent(E=16)
    ag.inserted = 1000
    rng = np.random.default_rng(5)
    u = rng.integers(0, 1 << 32, 200000, dtype=np.uint64)
    idx = ag.sample(u)
    assert idx.min() >= 0 and idx.max() < 1000
    counts = np.bincount(idx, minlength=1000)
    chi2 = ((counts - 200.0) ** 2 / 200.0).sum()
    assert chi2 < 1000 + 6 * np.sqrt(2000)


def test_tabular_update_rule_special_case():
    # Q_new(s,a) = Q(s,a) + alpha (r + gamma max Q(s',.) - Q(s,a)).  With W = 1 (the
    # job-advantage terms cancel), no hidden layer, batch 1 and plain SGD on (1/2) delta^2,
    # the change of Q(s,a) is exactly alpha (y - Q) with alpha = lr (2 - 1/L) (|x|^2 + 1).
    cfg = synth.config(1)
    sp = SP.build_space(1, 1, (25, 50, 75))
    pool = synth.make_pool(27)
    net = NetCfg(0, 0)
    dims = QN.net_dims(sp, net)
    assert dims == [17, sp.H]
    rng = np.random.default_rng(7)
    theta = rng.normal(0, 0.1, QN.n_params(dims))
    for gamma in (0.0, 0.9):
        ag = EV.OracleDQN(sp, pool, net, theta, 1, 1, 64, gamma=gamma, lr=0.01)
        ag.reset([[5]])
        ag.env_step(1 << 32, [0], [123456789 << 20], [[7]])      # explore, done
        assert ag.rep_done[0] == 1
        x = EV.encode([5], 0, pool, 1)
        z0, _ = QN.forward(ag.theta, dims, x[None])
        l, g, s = A.decode(sp, int(ag.rep_act[0]))
        v, aL, aJ = QN.split_head(z0[0], sp)
        cL, cJ = QN.center(aL, aJ)
        q0 = QN.q_value(v, cL, cJ, sp, l, g, s)
        out = ag.dqn_update([0], False)
        y = ag.rep_r[0]                                # done -> y = r (no bootstrap)
        assert out["y"][0] == pytest.approx(y, abs=1e-12)
        z1, _ = QN.forward(ag.theta, dims, x[None])
        v, aL, aJ = QN.split_head(z1[0], sp)
        cL, cJ = QN.center(aL, aJ)
        q1 = QN.q_value(v, cL, cJ, sp, l, g, s)
        alpha = 0.01 * (2 - 1 / sp.L) * (x @ x + 1)
        assert q1 == pytest.approx(q0 + alpha * (y - q0), rel=1e-10, abs=1e-10)


def _hand_dqn_weights(sp, net, z_online, z_target):
    """One hidden layer of width 4 with zero weights and bias 1 (h = ReLU(1) = 1 for every
    state), a zero head matrix and the head bias set to z: the head output is exactly z,
    independent of the state, so every Q value below is a hand computation."""
    dims = QN.net_dims(sp, net)
    fin, w, H = dims
    def flat(z):
        return np.concatenate([np.zeros(w * fin), np.ones(w), np.zeros(H * w),
                               np.asarray(z, np.float64)])
    return dims, flat(z_online), flat(z_target)


# Hand-computed double-DQN case (PAPER.md:180 "double DQN", :242 "duelling double DQN",
# van Hasselt [45] at :382; update rule :178).  W = 3, Cmax = 1, MIG off: one layout (the
# whole GPU), one slot type, H = 1 + 1 + 3 = 5, z = [v, aL, aJ0, aJ1, aJ2].
#   online z = [0, 0, 0, 2, 1]   -> cJ = [-1, 1, 0]
#   target z = [0.5, 0, 0, 0, 3] -> cJ = [-1, -1, 2], v = 0.5
# Step: explore with k = 0 -> action 0 = job 0 alone; s' has jobs 1, 2 unscheduled; not done.
# A single job on the whole GPU runs at its solo time: ratio 1, r = 0.
#   a*          = argmax_a Q_online(s', a) = job 1 (Q_online = 1 vs 0)
#   y (double)  = r + gamma Q_target(s', a*) = 0 + 0.9 * (0.5 - 1)       = -0.45
#   (plain DQN  r + gamma max_a Q_target(s', a) = 0.9 * 2.5 = 2.25;
#    online-evaluated r + gamma Q_online(s', a*) = 0.9 * 1 = 0.9: both must NOT come out)
#   Q(s, a)     = 0 + 0 + cJ[0] = -1;  delta = -1 - (-0.45) = -0.55;  L = delta^2 / 2 = 0.15125
#   dQ/dz(a)    = [1, 1 - 1/L = 0, 1 - 1/3, -1/3, -1/3]  (Q4 structured gradient), B = 1,
#   so the head bias moves by -lr * delta * dQ/dz and every head-matrix column (h = 1) alike.
DDQN_Z_ONLINE = [0.0, 0.0, 0.0, 2.0, 1.0]
DDQN_Z_TARGET = [0.5, 0.0, 0.0, 0.0, 3.0]
DDQN_Y, DDQN_DELTA, DDQN_LOSS, DDQN_ASTAR = -0.45, -0.55, 0.15125, 1
DDQN_DQDZ = [1.0, 0.0, 2.0 / 3.0, -1.0 / 3.0, -1.0 / 3.0]


def test_double_dqn_target_hand_computed():
    sp = SP.build_space(3, 1, (50,), False)
    assert (sp.L, sp.T, sp.H) == (1, 1, 5)
    pool = synth.make_pool(27)
    net = NetCfg(1, 4)
    dims, th_on, th_tg = _hand_dqn_weights(sp, net, DDQN_Z_ONLINE, DDQN_Z_TARGET)
    lr = 0.01
    ag = EV.OracleDQN(sp, pool, net, th_on, 1, 1, 64, gamma=0.9, lr=lr)
    ag.theta_t = th_tg.copy()
    ag.reset([[4, 11, 20]])
    a, r, d, cr, q = ag.env_step(1 << 32, [0], [0], [[0, 0, 0]])   # explore, k = 0
    assert int(a[0]) == 0 and int(d[0]) == 0 and r[0] == 0.0
    assert q[0] == pytest.approx(-1.0, abs=1e-15)
    out = ag.dqn_update([0], False)
    assert int(out["astar"][0]) == DDQN_ASTAR
    assert out["y"][0] == pytest.approx(DDQN_Y, abs=1e-12)
    assert out["q_sa"][0] == pytest.approx(-1.0, abs=1e-12)
    assert out["loss"] == pytest.approx(DDQN_LOSS, abs=1e-12)
    H, w, fin = sp.H, 4, dims[0]
    o_head = w * fin + w
    gW = out["grad"][o_head:o_head + H * w].reshape(H, w)
    gb = out["grad"][o_head + H * w:]
    np.testing.assert_allclose(gb, DDQN_DELTA * np.array(DDQN_DQDZ), atol=1e-12)
    np.testing.assert_allclose(gW, np.repeat(gb[:, None], w, 1), atol=1e-12)
    assert not out["grad"][:o_head].any()          # zero head matrix: no hidden gradient
    np.testing.assert_allclose(ag.theta[-H:], np.array(DDQN_Z_ONLINE) - lr * gb, atol=1e-15)


def test_gamma_zero_target_is_reward():
    ag, sp, pool = _agent(E=8, B=8, gamma=0.0)
    for t in range(3):
        st = synth.step_streams(t, ag.E, ag.B, sp.W, pool)
        ag.env_step(synth.eps_threshold(t, 5), st["u_explore"], st["u_action"],
                    st["next_windows"])
    st = synth.step_streams(9, ag.E, ag.B, sp.W, pool)
    out = ag.dqn_update(st["u_replay"], False)
    np.testing.assert_allclose(out["y"], ag.rep_r[out["idx"]], atol=0)


def _hand_agent(**kw):
    sp = SP.build_space(3, 1, (50,), False)
    pool = synth.make_pool(27)
    net = NetCfg(1, 4)
    dims, th_on, th_tg = _hand_dqn_weights(sp, net, DDQN_Z_ONLINE, DDQN_Z_TARGET)
    ag = EV.OracleDQN(sp, pool, net, th_on, 1, 1, 64, gamma=0.9, lr=0.01, **kw)
    ag.theta_t = th_tg.copy()
    ag.reset([[4, 11, 20]])
    ag.env_step(1 << 32, [0], [0], [[0, 0, 0]])
    return ag, sp


def test_huber_loss_hand_computed():
    # Huber with kappa = 0.25 on the hand case above (delta = -0.55):
    # loss = kappa (|delta| - kappa/2) = 0.25 * 0.425 = 0.10625, dL/dQ = clip(delta) = -0.25;
    # with kappa >= |delta| it is the squared loss (0.15125, dL/dQ = delta)
    ag, sp = _hand_agent(loss="huber", huber_kappa=0.25)
    out = ag.dqn_update([0], False)
    assert out["loss"] == pytest.approx(0.10625, abs=1e-12)
    gb = out["grad"][-sp.H:]
    np.testing.assert_allclose(gb, -0.25 * np.array(DDQN_DQDZ), atol=1e-12)
    ag2, _ = _hand_agent(loss="huber", huber_kappa=1.0)
    out2 = ag2.dqn_update([0], False)
    assert out2["loss"] == pytest.approx(DDQN_LOSS, abs=1e-12)


def test_adam_first_step_is_lr_times_sign():
    # Adam's first bias-corrected step is m^/(sqrt(v^) + eps) = g/(|g| + eps): every parameter
    # with a nonzero gradient moves by lr * sign(-g) (Kingma & Ba, Sec. 2), zero-gradient ones
    # stay; a second identical gradient moves them by the same amount again
    ag, sp = _hand_agent(optimizer="adam", adam=(0.9, 0.999, 1e-12))
    th0 = ag.theta.copy()
    out = ag.dqn_update([0], False)
    g = out["grad"]
    step = ag.theta - th0
    np.testing.assert_allclose(step, -0.01 * np.sign(g), atol=1e-9)
    assert (step[g == 0] == 0).all()
    th1 = ag.theta.copy()
    ag.apply(g, False)
    np.testing.assert_allclose(ag.theta - th1, -0.01 * np.sign(g), atol=1e-9)


def test_sequential_agent_hand_case_and_queue_order():
    # SURVEY §8(f)2 / reading R28: flat head z = [v, a_0..a_{L-1}], the job set is the next C_l
    # jobs in queue order.  W = 3, Cmax = 2, S = {50}, MIG off: layouts [(100)], [(50, 50)];
    # v = 0, a = [1, 3] -> cL = [-1, 1]: from sched 0 the agent takes l = 1 on jobs (0, 1) --
    # joint index off[1] + rank((0, 1)) * 2! + 0 = 3 + 0 = 3 -- then only l = 0 fits: job 2,
    # index 2.
    sp = SP.build_space(3, 2, (50,), False, seq=True)
    assert sp.L == 2 and sp.H == 3
    _, _, _, Fv, FcL, FcJ = EV.head_fixed(np.array([0.0, 1.0, 3.0]), sp)
    assert EV.greedy_seq(sp, Fv, FcL, 0)[0] == 3
    assert EV.greedy_seq(sp, Fv, FcL, 0b011)[0] == 2
    # episodes take the jobs in queue order and schedule each exactly once
    cfg = synth.config(1)
    sp = SP.build_space(4, 2, (25, 50, 75), seq=True)
    pool = synth.make_pool(27)
    th = synth.init_weights(QN.net_dims(sp, cfg.net))
    ag = EV.OracleDQN(sp, pool, cfg.net, th, 8, 8, 256)
    ag.reset(synth.make_windows(pool, 8, 4))
    order = [[] for _ in range(8)]
    for t in range(8):
        st = synth.step_streams(t, 8, 8, 4, pool)
        a, r, d, cr, q = ag.env_step(synth.eps_threshold(t, 6), st["u_explore"], st["u_action"],
                                     st["next_windows"])
        for e in range(8):
            l, g, s = A.decode(sp, int(a[e]))
            assert s == tuple(range(len(g)))
            order[e] += list(g)
            if d[e]:
                assert order[e] == [0, 1, 2, 3]
                order[e] = []
    out = ag.dqn_update(st["u_replay"], False)
    assert np.isfinite(out["loss"]) and out["grad"].shape == th.shape
