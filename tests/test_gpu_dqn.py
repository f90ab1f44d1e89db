"""GPU parity of the DQN step (hrp_env_step + hrp_dqn_update) and inference (hrp_q_forward)
against the float64 oracle, in lockstep over seeded steps (tests/dqn_harness.py).

Sizes follow SURVEY §8(c) "Parity protocol": config 1 in full (E = B = 64, 100 steps);
config 2 at E = B = 256 for 100 steps (the weight-gradient GEMM runs split-K with S >= 8, the
reduce's 8-wide path) and in the bench's launch configuration E = B = 4096 for 3 steps;
config 4 (W = 64, Cmax = 4, 4 x 512, P = 256, pruned argmax) at E = B = 64 for 20 steps."""
import numpy as np
import pytest
import torch

import synth
from oracle import env as EV
from oracle import pruned as PR
from oracle import qnet as QN
from oracle import space as SP
from dqn_harness import close, check_near_ties, log_stats, make_pair, run_lockstep

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("argmax_mode", [1, 2])
def test_config1_100_steps(argmax_mode):
    # BASELINE config 1: W=4, Cmax=2, S={25,50,75}, MLP 2x64, 64 envs, 100 steps
    st = run_lockstep(1, 64, 64, 100, argmax_mode=argmax_mode, check_weights_every=1,
                      oracle_argmax="explicit")
    print(st)


def test_config1_intermediate_reward():
    # r = r_f + lambda * sum r_i (Table VI, R9) with lambda = 1
    st = run_lockstep(1, 32, 32, 20, lam=1.0)
    print(st)


def test_ragged_sizes():
    # E, B not multiples of any tile size; W = 5 ragged rows of the encoder
    st = run_lockstep(1, 37, 23, 12, W=5)
    print(st)


def test_config2_explicit_vs_explicit_oracle():
    # config 2 space + net, explicit GPU enumeration against the oracle's explicit enumeration
    st = run_lockstep(2, 48, 48, 8, argmax_mode=1, check_weights_every=2,
                      oracle_argmax="explicit")
    print(st)


def test_config2_256_envs_100_steps():
    # SURVEY protocol: config 2 at E = B = 256 for 100 seeded steps (split-K S >= 8 in every
    # weight-gradient GEMM, target syncs at steps 25/50/75/100), each step compared from a
    # common state (R16b: the oracle adopts the GPU's weights after every step's comparison)
    st = run_lockstep(2, 256, 256, 100, resync=True)
    print(st)


def test_config2_256_envs_free_running_drift():
    # the same run without re-synchronisation: fp32 vs fp64 differences are amplified by the
    # training dynamics (large TD errors, lr 1e-3); the run must stay within 1e-4 for at least
    # 15 steps; the step where it first leaves is logged (R16b)
    st = run_lockstep(2, 256, 256, 100, check_weights_every=1, drift_min_steps=15,
                      name="drift_cfg2_E256_B256")
    print(st)


def test_config2_full_size_3_steps():
    # the bench's launch configuration: E = B = 4096, every output and the weights compared
    # element by element after each of 3 steps
    st = run_lockstep(2, 4096, 4096, 3)
    print(st)


def test_config4_64_envs_20_steps():
    # config 4: W = 64, Cmax = 4, 4 x 512, H = 5379, pool of 256, pruned exact argmax
    st = run_lockstep(4, 64, 64, 20, resync=True)
    print(st)


def test_config4_64_envs_free_running_drift():
    st = run_lockstep(4, 64, 64, 20, check_weights_every=1, drift_min_steps=1,
                      name="drift_cfg4_E64_B64")
    print(st)


def _states(pool, n, W, seed):
    wins = synth.make_windows(pool, n, W, step=seed)
    sched = synth.sched_states(n, W, step=seed)
    return wins, sched


@pytest.mark.parametrize("cfgk,n,mode", [(1, 200, 1), (2, 96, 1), (2, 96, 2)])
def test_q_forward_parity(cfgk, n, mode):
    cfg, pool, osp, sess, orc = make_pair(cfgk, 64, 64, argmax_mode=mode, workers=0)
    wins, sched = _states(pool, n, osp.W, 5)
    dw = torch.from_numpy(wins).to(sess.dev)
    ds = torch.from_numpy(sched.view(np.int64)).to(sess.dev)
    from paper_2405_08754_b200 import hrp
    from oracle import actions as A
    c0 = hrp.hrp_covered_counts(sess.ctx)
    am, qm, hd = sess.q_forward(dw, ds, head=True)
    torch.cuda.synchronize()
    c1 = hrp.hrp_covered_counts(sess.ctx)
    # the covered-actions counter is the number of valid actions of the scored states
    assert c1[0] - c0[0] == sum(A.n_valid(osp, int(x)) for x in sched)
    a_o, q_o, z_o = orc.q_forward(wins, sched, gpu_argmax=am.cpu().numpy())
    np.testing.assert_array_equal(am.cpu().numpy(), a_o)
    close(qm.cpu().numpy(), q_o, what="qmax")
    close(hd.cpu().numpy().ravel(), z_o.ravel(), what="head")
    stats = {}
    check_near_ties(orc, stats)
    log_stats(f"q_forward_cfg{cfgk}_mode{mode}", stats)


def test_explicit_equals_pruned_full_size():
    # config 2 at the bench's E=4096: the two exact argmax kernels agree bit for bit
    from paper_2405_08754_b200.session import Session
    cfg = synth.config(2)
    pool = synth.make_pool(27)
    osp = SP.build_space(16, 3, cfg.space.shares)
    th = synth.init_weights(QN.net_dims(osp, cfg.net))
    s1 = Session(cfg, pool, init_weights=th, argmax_mode=1)
    s2 = Session(cfg, pool, init_weights=th, argmax_mode=2)
    wins, sched = _states(pool, 4096, 16, 9)
    dw = torch.from_numpy(wins).to(s1.dev)
    ds = torch.from_numpy(sched.view(np.int64)).to(s1.dev)
    a1, q1, _ = s1.q_forward(dw, ds)
    a2, q2, _ = s2.q_forward(dw, ds)
    torch.cuda.synchronize()
    # argmax bit-exact; Q^max agrees to fp32 rounding of the (differently ordered) mean sums
    assert torch.equal(a1, a2)
    assert torch.allclose(q1, q2, rtol=1e-6, atol=1e-6)


def test_config4_pruned_q_forward_sampled():
    # config 4 space + net (W=64, Cmax=4, 4x512, P=256): pruned exact argmax vs the oracle's
    # pruned argmax on oracle-computed heads
    cfg, pool, osp, sess, orc = make_pair(4, 64, 64, argmax_mode=2)
    wins, sched = _states(pool, 24, 64, 3)
    dw = torch.from_numpy(wins).to(sess.dev)
    ds = torch.from_numpy(sched.view(np.int64)).to(sess.dev)
    am, qm, hd = sess.q_forward(dw, ds, head=True)
    torch.cuda.synchronize()
    a_o, q_o, z_o = orc.q_forward(wins, sched, gpu_argmax=am.cpu().numpy())
    orc.close()
    np.testing.assert_array_equal(am.cpu().numpy(), a_o)
    close(qm.cpu().numpy(), q_o, what="qmax")
    close(hd.cpu().numpy().ravel(), z_o.ravel(), what="head")


@pytest.mark.parametrize("period", [1, 3, 20])
def test_pruned_top_lists_with_tied_job_rows(period):
    # config 4 (W = 64): the head's job-advantage rows (and biases) of position j are copies of
    # position j mod period's, so every slot type has exact ties across positions.  period 1:
    # all U free positions tie (longer candidate lists than kPCap -> the full-scan fallback);
    # 3 and 20: mixed lists.  Ties must go to the lowest position (R15), as in the oracle.
    from paper_2405_08754_b200.session import Session
    cfg = synth.config(4)
    pool = synth.make_pool(cfg.pool)
    sc = cfg.space
    osp = SP.build_space(sc.window, sc.cmax, sc.shares, sc.mig)
    dims = QN.net_dims(osp, cfg.net)
    th = synth.init_weights(dims).copy()
    fi, H = dims[-2], dims[-1]
    o = sum(dims[i] * dims[i + 1] + dims[i + 1] for i in range(len(dims) - 2))
    Wh = th[o:o + fi * H].reshape(H, fi)
    bh = th[o + fi * H:o + fi * H + H]
    L, T, W = osp.L, osp.T, osp.W
    for j in range(period, W):
        src = 1 + L + (j % period) * T
        dst = 1 + L + j * T
        Wh[dst:dst + T] = Wh[src:src + T]
        bh[dst:dst + T] = bh[src:src + T]
    sess = Session(cfg, pool, n_envs=64, batch=64, init_weights=th, argmax_mode=2, replay=1024)
    orc = EV.OracleDQN(osp, pool, cfg.net, th, 64, 64, 1024, gamma=cfg.gamma, lr=cfg.lr,
                       argmax="pruned", workers=0)
    wins, sched = _states(pool, 24, W, 11)
    sched = sched.copy()
    sched[:4] = 0                       # all 64 positions free
    dw = torch.from_numpy(wins).to(sess.dev)
    ds = torch.from_numpy(sched.view(np.int64)).to(sess.dev)
    am, qm, hd = sess.q_forward(dw, ds, head=True)
    torch.cuda.synchronize()
    h = hd.cpu().numpy()
    aj = h[:, 1 + L:].reshape(len(wins), W, T)
    assert (aj[:, period:] == aj[:, [j % period for j in range(period, W)]]).all(), \
        "tied rows must give bit-identical head outputs"
    a_o, q_o, _ = orc.q_forward(wins, sched, gpu_argmax=am.cpu().numpy())
    orc.close()
    np.testing.assert_array_equal(am.cpu().numpy(), a_o)
    close(qm.cpu().numpy(), q_o, what="qmax")
    assert orc.near_ties == 0


def test_double_dqn_hand_computed_through_libhrp():
    # the hand-computed double-DQN case of tests/test_oracle_dqn.py
    # through the C ABI: online and target heads differ, gamma = 0.9, s' not terminal
    from test_oracle_dqn import (DDQN_ASTAR, DDQN_DELTA, DDQN_DQDZ, DDQN_LOSS,
                                 DDQN_Z_ONLINE, DDQN_Z_TARGET, _hand_dqn_weights)
    from paper_2405_08754_b200.session import Session
    cfg = synth.config(1).with_(space=synth.SpaceCfg(3, 1, (50,), mig=False),
                                net=synth.NetCfg(1, 4), gamma=0.9, lr=0.01)
    pool = synth.make_pool(27)
    osp = SP.build_space(3, 1, (50,), False)
    dims, th_on, th_tg = _hand_dqn_weights(osp, cfg.net, DDQN_Z_ONLINE, DDQN_Z_TARGET)
    sess = Session(cfg, pool, n_envs=1, batch=1, init_weights=th_on.astype(np.float32),
                   replay=64)
    from paper_2405_08754_b200 import hrp
    hrp.hrp_set_weights(sess.ctx, np.concatenate([th_on, th_tg]).astype(np.float32))
    d = sess.dev
    sess.reset(np.array([[4, 11, 20]], np.uint8))
    sess.step(1 << 32, torch.zeros(1, dtype=torch.int32, device=d),
              torch.zeros(1, dtype=torch.int64, device=d), torch.zeros((1, 3), dtype=torch.uint8,
                                                                       device=d))
    sess.update(torch.zeros(1, dtype=torch.int32, device=d), False)
    sess.sync()
    assert int(sess.actions.item()) == 0 and int(sess.done.item()) == 0
    assert float(sess.rewards.item()) == 0.0
    assert int(sess.astar.item()) == DDQN_ASTAR
    assert abs(sess.loss.item() - DDQN_LOSS) <= 1e-6
    w = sess.weights()
    n = sess.n_params
    H = osp.H
    gb = DDQN_DELTA * np.array(DDQN_DQDZ)
    np.testing.assert_allclose(w[n - H:n], np.array(DDQN_Z_ONLINE) - 0.01 * gb, atol=1e-6)
    np.testing.assert_allclose(w[2 * n - H:], DDQN_Z_TARGET, atol=0)   # target untouched
    sess.close()


def test_sharded_update_two_contexts_matches_oracle_simulation():
    # E_local envs per rank, gradient = (sum over ranks of the local sums) /
    # B_global.  Two world-1 contexts stand in for two ranks on one GPU: each exports its shard's
    # gradient (hrp_dqn_grad, scale 1/B_local), the test averages them (the allreduce) and both
    # apply it (hrp_apply_grad); the oracle simulates the same two shards (as in
    # tests/test_parallel_gloo.py).  Replicas must stay identical and match the oracle.
    from paper_2405_08754_b200.parallel import env_shard
    from paper_2405_08754_b200.session import Session, streams_to_dev
    cfg = synth.config(1)
    pool = synth.make_pool(27)
    osp = SP.build_space(4, 2, cfg.space.shares)
    th = synth.init_weights(QN.net_dims(osp, cfg.net))
    EL, WORLD, STEPS = 24, 2, 6
    sess = [Session(cfg, pool, n_envs=EL, batch=EL, init_weights=th, replay=1024)
            for _ in range(WORLD)]
    orcs = [EV.OracleDQN(osp, pool, cfg.net, th, EL, EL, 1024, gamma=cfg.gamma, lr=cfg.lr)
            for _ in range(WORLD)]
    for r in range(WORLD):
        w0 = synth.make_windows(pool, EL, 4, rank=r, first_env=env_shard(EL, r))
        sess[r].reset(w0)
        orcs[r].reset(w0)
    n = sess[0].n_params
    grads = [torch.empty(n, dtype=torch.float32, device=sess[0].dev) for _ in range(WORLD)]
    for t in range(STEPS):
        thr = synth.eps_threshold(t, cfg.n_decay)
        sync_t = (t + 1) % 3 == 0
        g_orc = 0
        for r in range(WORLD):
            st = synth.step_streams(t, EL, EL, 4, pool, rank=r, first_env=env_shard(EL, r))
            d = streams_to_dev(st, sess[r].dev)
            sess[r].step(thr, d["u_explore"], d["u_action"], d["next_windows"])
            sess[r].grad(d["u_replay"], grads[r])
            sess[r].sync()
            a, *_ = orcs[r].env_step(thr, st["u_explore"], st["u_action"], st["next_windows"],
                                     gpu_actions=sess[r].greedy.cpu().numpy())
            np.testing.assert_array_equal(sess[r].actions.cpu().numpy(), a)
            out = orcs[r].dqn_update(st["u_replay"], False, gpu_astar=sess[r].astar.cpu().numpy(),
                                     b_total=EL * WORLD, apply=False,
                                     gpu_masks=sess[r].relu_masks())
            close([sess[r].loss.item()], [out["loss"]], what=f"loss r={r} t={t}")
            # this rank's exported gradient is its local sum / B_local
            close(grads[r].cpu().numpy(), out["grad"] * WORLD, what=f"grad r={r} t={t}")
            g_orc = g_orc + out["grad"]
        g = (grads[0] + grads[1]) / WORLD          # the allreduce-sum scaled to 1 / B_global
        for r in range(WORLD):
            sess[r].apply_grad(g, sync_t)
            orcs[r].apply(g_orc, sync_t)
    w0, w1 = sess[0].weights(), sess[1].weights()
    assert np.array_equal(w0, w1), "replicas diverged"
    close(w0[:n], orcs[0].theta, what="online weights")
    close(w0[n:], orcs[0].theta_t, what="target weights")
    assert not np.allclose(w0[:n], th), "weights did not move"
    for s in sess:
        s.close()


def test_non_finite_weights_are_reported_not_followed():
    # NaN head outputs must not drive the env off its valid actions; hrp_sync reports
    from paper_2405_08754_b200 import hrp
    from paper_2405_08754_b200.session import streams_to_dev
    cfg, pool, osp, sess, orc = make_pair(1, 16, 16, argmax_mode=1, workers=0)
    orc.close()
    w = sess.weights()
    w[:] = np.nan
    hrp.hrp_set_weights(sess.ctx, w)
    sess.reset(synth.make_windows(pool, 16, 4))
    st = streams_to_dev(synth.step_streams(0, 16, 16, 4, pool), sess.dev)
    sess.step(0, st["u_explore"], st["u_action"], st["next_windows"])   # greedy only
    with pytest.raises(hrp.HrpError) as ei:
        sess.sync()
    assert ei.value.status == hrp.HRP_ENUMERIC
    a = sess.actions.cpu().numpy()
    from oracle import actions as A
    assert (a >= 0).all() and (a < A.n_actions(osp)).all()
    sess.sync()                                   # the flag is cleared once reported
    sess.close()


def test_cuda_graph_replay_equals_eager():
    # bench.py times per-step CUDA graphs: steps recorded into graphs (host counters advancing
    # at capture) and replayed in order must reproduce eager launches bit for bit, on two
    # streams (fork/join events) and the tensor-core path
    from paper_2405_08754_b200.session import Session, streams_to_dev
    cfg = synth.config(2)
    pool = synth.make_pool(27)
    osp = SP.build_space(16, 3, cfg.space.shares)
    th = synth.init_weights(QN.net_dims(osp, cfg.net))
    E = B = 256
    outs = []
    for use_graph in (False, True):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            sess = Session(cfg, pool, n_envs=E, batch=B, init_weights=th, replay=4096,
                           stream=stream)
            sess.reset(synth.make_windows(pool, E, 16))
            steps = [streams_to_dev(synth.step_streams(t, E, B, 16, pool), sess.dev)
                     for t in range(6)]
            rec, graphs = [], []
            for t, d in enumerate(steps):
                thr = synth.eps_threshold(t, cfg.n_decay)

                def one(t=t, d=d, thr=thr):
                    sess.step(thr, d["u_explore"], d["u_action"], d["next_windows"], extras=False)
                    sess.update(d["u_replay"], t % 3 == 2, extras=False)
                if use_graph and t >= 2:
                    # as bench.py: capture every remaining step first, then replay in order
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=stream):
                        one()
                    graphs.append(g)
                    continue
                one()
                stream.synchronize()
                rec.append((sess.actions.clone(), sess.rewards.clone(), sess.loss.clone()))
            for g in graphs:
                g.replay()
                stream.synchronize()
                rec.append((sess.actions.clone(), sess.rewards.clone(), sess.loss.clone()))
            rec.append(torch.from_numpy(sess.weights()))
            outs.append(rec)
            sess.close()
    for x, y in zip(outs[0][:-1], outs[1][:-1]):
        for u, v in zip(x, y):
            assert torch.equal(u, v)
    assert torch.equal(outs[0][-1], outs[1][-1])


def test_nccl_bucketed_allreduce_path_on_one_gpu():
    # the per-layer allreduce buckets (side stream, NCCL calls captured in the
    # per-step CUDA graphs) run on one GPU through a one-rank communicator; a sum over one rank
    # is the identity, so the weights must equal the no-communicator context's bit for bit
    from paper_2405_08754_b200 import hrp
    from paper_2405_08754_b200.session import Session, streams_to_dev
    cfg = synth.config(2)
    pool = synth.make_pool(27)
    osp = SP.build_space(16, 3, cfg.space.shares)
    th = synth.init_weights(QN.net_dims(osp, cfg.net))
    E = B = 256
    outs = []
    for nccl in (False, True):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            sess = Session(cfg, pool, n_envs=E, batch=B, init_weights=th, replay=4096,
                           stream=stream, nccl_id=hrp.hrp_nccl_unique_id() if nccl else None)
            sess.reset(synth.make_windows(pool, E, 16))
            steps = [streams_to_dev(synth.step_streams(t, E, B, 16, pool), sess.dev)
                     for t in range(5)]
            graphs = []
            for t, d in enumerate(steps):
                thr = synth.eps_threshold(t, cfg.n_decay)

                def one(t=t, d=d, thr=thr):
                    sess.step(thr, d["u_explore"], d["u_action"], d["next_windows"], extras=False)
                    sess.update(d["u_replay"], t == 3, extras=False)
                if t < 2:
                    one()
                    continue
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    one()
                graphs.append(g)
            for g in graphs:
                g.replay()
            stream.synchronize()
            sess.sync()
            outs.append(sess.weights())
            sess.close()
    assert np.array_equal(outs[0], outs[1])
