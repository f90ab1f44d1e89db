"""Lockstep GPU-vs-oracle driver for the DQN parity tests (test infrastructure).

Protocol (SURVEY §8(c) "Parity protocol", R15/R16): integers bit-exact (actions,
done, CoRun, replay sample indices, a*); floats within 1e-4 * max(|oracle|, rms(tensor))
(rewards, Q^ of the taken action, loss, weights after every step).  The oracle runs free
(its fp64 weights are never re-synchronised); only argmax near-ties (oracle Q^ gap <= 1e-4)
adopt the GPU's choice and are counted.
"""
from __future__ import annotations

import numpy as np
import torch

import synth
from oracle import env as EV
from oracle import pruned as PR
from oracle import qnet as QN
from oracle import space as SP

TOL = 1e-4


def close(gpu, orc, tol=TOL, what=""):
    gpu = np.asarray(gpu, np.float64)
    orc = np.asarray(orc, np.float64)
    scale = np.maximum(np.abs(orc), np.sqrt(np.mean(orc ** 2)) if orc.size else 0.0)
    scale = np.maximum(scale, 1e-30)
    err = np.abs(gpu - orc) / scale
    bad = np.nonzero(err > tol)[0]
    assert bad.size == 0, f"{what}: {bad.size} outside tol, worst {err.max():.3e} at " \
                          f"{int(np.argmax(err))}: gpu {gpu.ravel()[np.argmax(err)]} " \
                          f"orc {orc.ravel()[np.argmax(err)]}"
    return float(err.max()) if err.size else 0.0


def make_pair(cfgk, E, B, gemm_mode=1, argmax_mode=1, lam=0.0, W=None, replay=None):
    from paper_2405_08754_b200.session import Session
    cfg = synth.config(cfgk)
    if W is not None:
        cfg = cfg.with_(space=cfg.space.__class__(W, cfg.space.cmax, cfg.space.shares,
                                                  cfg.space.mig, cfg.space.interference_q3,
                                                  lam))
    pool = synth.make_pool(cfg.pool)
    sc = cfg.space
    osp = SP.build_space(sc.window, sc.cmax, sc.shares, sc.mig)
    dims = QN.net_dims(osp, cfg.net)
    theta0 = synth.init_weights(dims)
    N = replay or max(1 << 10, 4 * E)
    sess = Session(cfg, pool, n_envs=E, batch=B, init_weights=theta0, argmax_mode=argmax_mode,
                   gemm_mode=gemm_mode, replay=N, reward_lambda=lam)
    assert sess.n_params == len(theta0)
    greedy = None
    if argmax_mode == 2:
        off = None
        greedy = lambda Fv, FcL, FcJ, s: PR.greedy_pruned(osp, Fv, FcL, FcJ, s, off)
    orc = EV.OracleDQN(osp, pool, cfg.net, theta0, E, B, N, gamma=cfg.gamma, lr=cfg.lr,
                       reward_lambda=lam, greedy=greedy)
    return cfg, pool, osp, sess, orc


def run_lockstep(cfgk, E, B, steps, gemm_mode=1, argmax_mode=1, lam=0.0, W=None, seed_step=0,
                 check_weights_every=1):
    from paper_2405_08754_b200.session import streams_to_dev
    cfg, pool, osp, sess, orc = make_pair(cfgk, E, B, gemm_mode, argmax_mode, lam, W)
    Wn = osp.W
    win0 = synth.make_windows(pool, E, Wn, step=seed_step)
    sess.reset(win0)
    orc.reset(win0)
    stats = {"near_ties": 0, "max_err": {}}
    for t in range(steps):
        st = synth.step_streams(seed_step + t, E, B, Wn, pool)
        dst = streams_to_dev(st, sess.dev)
        thr = synth.eps_threshold(t, cfg.n_decay)
        sess.step(thr, dst["u_explore"], dst["u_action"], dst["next_windows"])
        sess.sync()
        g_greedy = sess.greedy.cpu().numpy()
        a, r, d, cr, q = orc.env_step(thr, st["u_explore"], st["u_action"], st["next_windows"],
                                      gpu_actions=g_greedy)
        np.testing.assert_array_equal(sess.actions.cpu().numpy(), a, err_msg=f"actions t={t}")
        np.testing.assert_array_equal(sess.done.cpu().numpy(), d, err_msg=f"done t={t}")
        np.testing.assert_array_equal(sess.corun.cpu().numpy(), cr, err_msg=f"corun t={t}")
        e1 = close(sess.rewards.cpu().numpy(), r, what=f"rewards t={t}")
        e2 = close(sess.qsel.cpu().numpy(), q, what=f"qsel t={t}")
        sync_t = (t + 1) % cfg.target_sync == 0
        sess.update(dst["u_replay"], sync_t)
        sess.sync()
        g_astar = sess.astar.cpu().numpy()
        out = orc.dqn_update(st["u_replay"], sync_t, gpu_astar=g_astar)
        np.testing.assert_array_equal(sess.sidx.cpu().numpy(), out["idx"], err_msg=f"idx t={t}")
        np.testing.assert_array_equal(g_astar, out["astar"], err_msg=f"astar t={t}")
        e3 = close([sess.loss.item()], [out["loss"]], what=f"loss t={t}")
        if (t + 1) % check_weights_every == 0 or t == steps - 1:
            w = sess.weights()
            n = sess.n_params
            e4 = close(w[:n], orc.theta, what=f"online weights t={t}")
            e5 = close(w[n:], orc.theta_t, what=f"target weights t={t}")
        else:
            e4 = e5 = 0.0
        for k, v in (("reward", e1), ("qsel", e2), ("loss", e3), ("theta", e4),
                     ("theta_t", e5)):
            stats["max_err"][k] = max(stats["max_err"].get(k, 0.0), v)
    stats["near_ties"] = orc.near_ties
    sess.close()
    return stats
