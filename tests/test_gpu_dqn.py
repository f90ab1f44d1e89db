"""GPU parity of the DQN step (hrp_env_step + hrp_dqn_update) and inference (hrp_q_forward)
against the float64 oracle, in lockstep over seeded steps (tests/dqn_harness.py)."""
import numpy as np
import pytest
import torch

import synth
from oracle import env as EV
from oracle import pruned as PR
from oracle import qnet as QN
from oracle import space as SP
from dqn_harness import close, make_pair, run_lockstep

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("gemm_mode", [1, 2])
def test_config1_100_steps(gemm_mode):
    # BASELINE config 1: W=4, Cmax=2, S={25,50,75}, MLP 2x64, 64 envs, 100 steps
    st = run_lockstep(1, 64, 64, 100, gemm_mode=gemm_mode, argmax_mode=1,
                      check_weights_every=1)
    print(st)


def test_config1_pruned_argmax():
    st = run_lockstep(1, 64, 64, 30, argmax_mode=2)
    print(st)


def test_config1_intermediate_reward():
    # r = r_f + lambda * sum r_i (Table VI, R9) with lambda = 1
    st = run_lockstep(1, 32, 32, 20, lam=1.0)
    print(st)


def test_ragged_sizes():
    # E, B not multiples of any tile size; W = 5 ragged rows of the encoder
    st = run_lockstep(1, 37, 23, 12, W=5)
    print(st)


@pytest.mark.parametrize("gemm_mode", [1, 2])
def test_config2_reduced(gemm_mode):
    # BASELINE config 2 space + net (W=16, Cmax=3, S={10..90}, 3x256) at E=B=48
    st = run_lockstep(2, 48, 48, 8, gemm_mode=gemm_mode, argmax_mode=1,
                      check_weights_every=2)
    print(st)


def _states(pool, n, W, seed):
    wins = synth.make_windows(pool, n, W, step=seed)
    sched = synth.sched_states(n, W, step=seed)
    return wins, sched


@pytest.mark.parametrize("cfgk,n,mode", [(1, 200, 1), (2, 96, 1), (2, 96, 2)])
def test_q_forward_parity(cfgk, n, mode):
    cfg, pool, osp, sess, orc = make_pair(cfgk, 64, 64, argmax_mode=mode)
    wins, sched = _states(pool, n, osp.W, 5)
    dw = torch.from_numpy(wins).to(sess.dev)
    ds = torch.from_numpy(sched.view(np.int64)).to(sess.dev)
    am, qm, hd = sess.q_forward(dw, ds, head=True)
    torch.cuda.synchronize()
    a_o, q_o, z_o = orc.q_forward(wins, sched, gpu_argmax=am.cpu().numpy())
    np.testing.assert_array_equal(am.cpu().numpy(), a_o)
    close(qm.cpu().numpy(), q_o, what="qmax")
    close(hd.cpu().numpy().ravel(), z_o.ravel(), what="head")
    print("near ties", orc.near_ties)


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
    orc.greedy_fn = lambda Fv, FcL, FcJ, s: PR.greedy_pruned(osp, Fv, FcL, FcJ, s, orc.off)
    wins, sched = _states(pool, 24, 64, 3)
    dw = torch.from_numpy(wins).to(sess.dev)
    ds = torch.from_numpy(sched.view(np.int64)).to(sess.dev)
    am, qm, hd = sess.q_forward(dw, ds, head=True)
    torch.cuda.synchronize()
    a_o, q_o, z_o = orc.q_forward(wins, sched, gpu_argmax=am.cpu().numpy())
    np.testing.assert_array_equal(am.cpu().numpy(), a_o)
    close(qm.cpu().numpy(), q_o, what="qmax")
    close(hd.cpu().numpy().ravel(), z_o.ravel(), what="head")


def test_config2_full_size_step_sampled():
    # BASELINE config 2 in the bench's launch configuration (E = B = 4096): one step + one
    # update; a sample of envs is replayed through the oracle (per-env outputs depend only on
    # that env's state and the shared weights)
    from paper_2405_08754_b200.session import Session, streams_to_dev
    cfg = synth.config(2)
    pool = synth.make_pool(27)
    osp = SP.build_space(16, 3, cfg.space.shares)
    th = synth.init_weights(QN.net_dims(osp, cfg.net))
    E = cfg.n_envs
    sess = Session(cfg, pool, init_weights=th)
    win0 = synth.make_windows(pool, E, 16)
    sess.reset(win0)
    st = synth.step_streams(0, E, E, 16, pool)
    thr = synth.eps_threshold(60, cfg.n_decay)   # late schedule: mostly greedy
    dst = streams_to_dev(st, sess.dev)
    sess.step(thr, dst["u_explore"], dst["u_action"], dst["next_windows"])
    sess.update(dst["u_replay"], False)
    sess.sync()
    loss = sess.loss.item()
    assert np.isfinite(loss)
    pick = np.array([0, 1, 2, 777, 2048, 4095])
    orc = EV.OracleDQN(osp, pool, cfg.net, th, len(pick), 1, 1 << 10, gamma=cfg.gamma,
                       lr=cfg.lr)
    orc.reset(win0[pick])
    g = sess.greedy.cpu().numpy()[pick]
    a, r, d, cr, q = orc.env_step(thr, st["u_explore"][pick], st["u_action"][pick],
                                  st["next_windows"][pick], gpu_actions=g)
    np.testing.assert_array_equal(sess.actions.cpu().numpy()[pick], a)
    np.testing.assert_array_equal(sess.corun.cpu().numpy()[pick], cr)
    close(sess.rewards.cpu().numpy()[pick], r, what="rewards")
    close(sess.qsel.cpu().numpy()[pick], q, what="qsel")


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
