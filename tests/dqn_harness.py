"""Lockstep GPU-vs-oracle driver for the DQN parity tests (test infrastructure).

Protocol (SURVEY §8(c) "Parity protocol", R15/R16): integers bit-exact (actions,
done, CoRun, replay sample indices, a*); floats within 1e-4 * max(|oracle|, rms(tensor))
(rewards, Q^ of the taken action, loss, weights after every checked step).  The oracle runs
free (its fp64 weights are never re-synchronised) unless `resync` is set: then every step
starts from a common state -- after each step's comparison the oracle adopts the GPU's fp32
weights -- so each step's outputs are compared for that step's arithmetic alone ("1e-4 relative
per step", BASELINE north star; R16b).  Only argmax near-ties (oracle Q^ gap
<= 1e-4 max(1, |Q|)) adopt the GPU's choice.  They are counted against the number of greedy
argmaxes and bounded (NEAR_TIE_FRAC); every run's counts and worst errors are appended to
$HRP_PARITY_LOG (JSON lines) when that variable is set.
"""
from __future__ import annotations

import json
import os
import time

import numpy as np
import torch

import synth
from oracle import env as EV
from oracle import qnet as QN
from oracle import space as SP

TOL = 1e-4
NEAR_TIE_FRAC = 1e-3      # at most 0.1 % of the greedy argmaxes may be R15 adoptions (+1)
WORKERS = max(1, min(16, (os.cpu_count() or 1)))


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


def log_stats(name, stats):
    path = os.environ.get("HRP_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"test": name, **stats}) + "\n")


def check_near_ties(orc, stats):
    stats["near_ties"] = orc.near_ties
    stats["greedy_argmaxes"] = orc.greedy_calls
    stats["near_tie_worst_rel_gap"] = orc.near_tie_gap
    stats["relu_near_zero_adopted"] = orc.relu_near
    stats["relu_decisions"] = orc.relu_decisions
    # R25 adoptions must stay rare too (units within 1e-4 rms of zero)
    assert orc.relu_near <= 1e-5 * orc.relu_decisions + 4, \
        f"{orc.relu_near} ReLU' adoptions out of {orc.relu_decisions} decisions"
    assert orc.near_ties <= NEAR_TIE_FRAC * orc.greedy_calls + 1, \
        f"{orc.near_ties} R15 near-tie adoptions out of {orc.greedy_calls} argmaxes"


def make_pair(cfgk, E, B, argmax_mode=2, lam=0.0, W=None, replay=None, workers=None,
              oracle_argmax=None, variant=None, cmax=None):
    """variant: SURVEY §8(f)4 options for both sides, e.g. {"optimizer": "adam",
    "loss": "huber", "huber_kappa": 10.0}."""
    variant = dict(variant or {})
    from paper_2405_08754_b200.session import Session
    cfg = synth.config(cfgk)
    if W is not None or cmax is not None:
        cfg = cfg.with_(space=cfg.space.__class__(W or cfg.space.window, cmax or cfg.space.cmax,
                                                  cfg.space.shares, cfg.space.mig,
                                                  cfg.space.interference_q3, lam))
    pool = synth.make_pool(cfg.pool)
    sc = cfg.space
    osp = SP.build_space(sc.window, sc.cmax, sc.shares, sc.mig,
                         seq=variant.get("agent") == "sequential")
    dims = QN.net_dims(osp, cfg.net)
    theta0 = synth.init_weights(dims)
    N = replay or max(1 << 10, 4 * E)
    sess = Session(cfg, pool, n_envs=E, batch=B, init_weights=theta0, argmax_mode=argmax_mode,
                   replay=N, reward_lambda=lam, **variant)
    variant.pop("precision", None)
    variant.pop("agent", None)
    assert sess.n_params == len(theta0)
    # the oracle's argmax: explicit enumeration where it is cheap, else the exact top-C search
    # (oracle/pruned.py, pinned against explicit enumeration); both give the same index
    argmax = oracle_argmax or ("explicit" if (osp.W <= 8 and argmax_mode == 1) else "pruned")
    nw = WORKERS if workers is None else workers
    orc = EV.OracleDQN(osp, pool, cfg.net, theta0, E, B, N, gamma=cfg.gamma, lr=cfg.lr,
                       reward_lambda=lam, argmax=argmax,
                       workers=nw if (E > 64 or osp.W >= 16) else 0, **variant)
    return cfg, pool, osp, sess, orc


def run_lockstep(cfgk, E, B, steps, argmax_mode=2, lam=0.0, W=None, seed_step=0,
                 check_weights_every=1, name=None, workers=None, oracle_argmax=None,
                 resync=False, drift_min_steps=None, variant=None, cmax=None):
    """drift_min_steps: free-running drift probe -- instead of failing, stop at the first step
    whose float outputs leave the tolerance, record it, and assert it is >= drift_min_steps."""
    from paper_2405_08754_b200.session import streams_to_dev
    t_start = time.time()
    cfg, pool, osp, sess, orc = make_pair(cfgk, E, B, argmax_mode, lam, W, workers=workers,
                                          oracle_argmax=oracle_argmax, variant=variant,
                                          cmax=cmax)
    Wn = osp.W
    win0 = synth.make_windows(pool, E, Wn, step=seed_step)
    sess.reset(win0)
    orc.reset(win0)
    stats = {"cfg": cfgk, "E": E, "B": B, "steps": steps, "argmax_mode": argmax_mode,
             "oracle_argmax": orc.argmax, "resync": resync, "variant": variant, "max_err": {}}
    if resync:
        check_weights_every = 1
    n = sess.n_params

    def one(t):
        st = synth.step_streams(seed_step + t, E, B, Wn, pool)
        dst = streams_to_dev(st, sess.dev)
        thr = synth.eps_threshold(t, cfg.n_decay)
        sess.step(thr, dst["u_explore"], dst["u_action"], dst["next_windows"])
        sess.sync()
        g_greedy = sess.greedy.cpu().numpy()
        a, r, d, cr, q = orc.env_step(thr, st["u_explore"], st["u_action"],
                                      st["next_windows"], gpu_actions=g_greedy)
        np.testing.assert_array_equal(sess.actions.cpu().numpy(), a, err_msg=f"actions t={t}")
        np.testing.assert_array_equal(sess.done.cpu().numpy(), d, err_msg=f"done t={t}")
        np.testing.assert_array_equal(sess.corun.cpu().numpy(), cr, err_msg=f"corun t={t}")
        e1 = close(sess.rewards.cpu().numpy(), r, what=f"rewards t={t}")
        e2 = close(sess.qsel.cpu().numpy(), q, what=f"qsel t={t}")
        sync_t = (t + 1) % cfg.target_sync == 0
        sess.update(dst["u_replay"], sync_t)
        sess.sync()
        g_astar = sess.astar.cpu().numpy()
        out = orc.dqn_update(st["u_replay"], sync_t, gpu_astar=g_astar,
                             gpu_masks=sess.relu_masks())
        np.testing.assert_array_equal(sess.sidx.cpu().numpy(), out["idx"], err_msg=f"idx t={t}")
        np.testing.assert_array_equal(g_astar, out["astar"], err_msg=f"astar t={t}")
        e3 = close([sess.loss.item()], [out["loss"]], what=f"loss t={t}")
        e4 = e5 = 0.0
        if (t + 1) % check_weights_every == 0 or t == steps - 1:
            w = sess.weights()
            e4 = close(w[:n], orc.theta, what=f"online weights t={t}")
            e5 = close(w[n:], orc.theta_t, what=f"target weights t={t}")
            if resync:
                orc.theta = w[:n].astype(np.float64)
                orc.theta_t = w[n:].astype(np.float64)
        for k, v in (("reward", e1), ("qsel", e2), ("loss", e3), ("theta", e4),
                     ("theta_t", e5)):
            stats["max_err"][k] = max(stats["max_err"].get(k, 0.0), v)

    try:
        for t in range(steps):
            try:
                one(t)
            except AssertionError as ex:
                if drift_min_steps is None:
                    raise
                stats["first_excursion_step"] = t
                stats["excursion"] = str(ex).split("\n")[0][:200]
                assert t >= drift_min_steps, f"free-running drift left 1e-4 at step {t}: {ex}"
                break
        check_near_ties(orc, stats)
    finally:
        stats["seconds"] = round(time.time() - t_start, 1)
        stats.setdefault("near_ties", orc.near_ties)
        stats.setdefault("greedy_argmaxes", orc.greedy_calls)
        stats.setdefault("relu_near_zero_adopted", orc.relu_near)
        log_stats(name or f"lockstep_cfg{cfgk}_E{E}_B{B}_x{steps}", stats)
        orc.close()
        sess.close()
    return stats
