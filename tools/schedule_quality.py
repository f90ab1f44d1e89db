"""Schedule-quality report (Fig. 8, Fig. 11 AppSlowdown
P:291-305, Fig. 12 Fairness P:307-313) on Q1-Q12 (Table V, W = 12, Cmax = 4):

* Time Sharing, MIG Only (C = 2), MPS Only (C <= 4), MIG+MPS (C <= 4): the exhaustive optimum
  of each method's search space -- hrp_brute_run;
* MIG+MPS Default (C <= 4): one MIG partition for all queues (the one with the best average
  optimum throughput over Q1-Q12), MPS in its default mode modelled as equal shares (R27);
* MIG+MPS w/ RL: the duelling double-DQN agent trained with libhrp on config 3's space
  (class-stratified random windows, R18) and run greedily (epsilon = 0) on Q1-Q12 --
  hrp_env_step;
then per queue the relative throughput Solo / CoRun, the mean AppSlowdown and the Fairness,
every co-run time from hrp_job_times.  The co-run model is R8's synthetic one: the numbers are
the synthetic analogue of the figures, not a reproduction.

usage: python tools/schedule_quality.py [--steps 3000] [--out profiles/r2_schedule_quality.md]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def train_policy(pool, steps, E, lr, seed_step=1000, log_every=250, agent="joint"):
    """Train on config 3's space (W = 12, Cmax = 4, S = {10..90}) with a 3 x 256 Q-MLP, Adam +
    Huber (plain SGD on (1/2) delta^2 diverges at these reward scales), epsilon
    1 -> 0.01 over the first half.  Returns (online weights, training log)."""
    import torch
    from paper_2405_08754_b200 import hrp
    from paper_2405_08754_b200.session import Session, space_of, streams_to_dev
    sc = synth.SpaceCfg(12, 4, tuple(range(10, 100, 10)))
    cfg = synth.config(2).with_(space=sc, n_decay=max(1, steps // 2), lr=lr, target_sync=100)
    tab = hrp.hrp_layout_table(space_of(sc))
    H = 1 + tab["n_layouts"] + (12 * tab["n_types"] if agent == "joint" else 0)
    dims = [12 * 17] + [256] * 3 + [H]
    th = synth.init_weights(dims)
    sess = Session(cfg, pool, n_envs=E, batch=E, init_weights=th, replay=max(1 << 16, 16 * E),
                   optimizer="adam", loss="huber", huber_kappa=10.0, agent=agent)
    sess.reset(synth.make_windows(pool, E, 12, step=seed_step))
    log = []
    t0 = time.time()
    rsum = 0.0
    for t in range(steps):
        st = streams_to_dev(synth.step_streams(seed_step + t, E, E, 12, pool), sess.dev)
        sess.step(synth.eps_threshold(t, cfg.n_decay), st["u_explore"], st["u_action"],
                  st["next_windows"], extras=False)
        sess.update(st["u_replay"], (t + 1) % cfg.target_sync == 0, extras=False)
        if (t + 1) % log_every == 0:
            sess.sync()
            r = float(sess.rewards.mean().item())
            log.append({"step": t + 1, "loss": float(sess.loss.item()), "mean_reward": r,
                        "seconds": round(time.time() - t0, 1)})
            print(json.dumps(log[-1]), flush=True)
    w = sess.weights()[:sess.n_params].copy()
    sess.close()
    return w, log, cfg.with_(extra={"agent": agent})


def rl_schedules(pool, Q, weights, cfg):
    from paper_2405_08754_b200.schedule import greedy_rollout
    from paper_2405_08754_b200.session import Session
    sess = Session(cfg, pool, n_envs=len(Q), batch=len(Q), init_weights=weights, replay=1024,
                   agent=cfg.extra.get("agent", "joint"))
    out = greedy_rollout(sess, Q)
    sess.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--envs", type=int, default=4096)
    ap.add_argument("--lr", type=float, default=1e-4)
    args = ap.parse_args()
    import torch
    from paper_2405_08754_b200 import hrp
    from paper_2405_08754_b200.schedule import (job_metrics, make_plan, optimum_schedules,
                                                time_sharing_schedules)
    from paper_2405_08754_b200.session import space_of
    pool = synth.make_pool(27)
    prof = hrp.make_profiles(pool)
    Q = synth.table_v_windows(pool)
    full = synth.BASELINE_SPACES["mig_mps"][0]
    full_space = space_of(full)
    full_plan = make_plan(full_space, prof)
    methods, timing = {}, {}
    methods["Time Sharing"] = job_metrics(full_plan, pool, Q, time_sharing_schedules(full_space, Q))
    for name, key in (("MIG Only (C=2)", "mig_only"), ("MPS Only (C<=4)", "mps_only"),
                      ("MIG+MPS optimum (C<=4)", "mig_mps")):
        scfg, lay = synth.BASELINE_SPACES[key]
        plan = make_plan(space_of(scfg, lay), prof) if key != "mig_mps" else full_plan
        optimum_schedules(plan, Q)                      # warm-up
        torch.cuda.synchronize()
        t = time.perf_counter()
        sch, best = optimum_schedules(plan, Q)
        timing[key] = time.perf_counter() - t
        methods[name] = job_metrics(plan, pool, Q, sch)
        assert all(m["corun"] == b for m, b in zip(methods[name], best)), "optimum mismatch"
    # MIG+MPS Default (R27): one MIG partition for all queues, chosen by the average
    # throughput over Q1-Q12 of the exhaustive optimum under it with equal (default) MPS shares
    from paper_2405_08754_b200.schedule import default_mps_table, mig_partitions
    best_p, best_am, per_p = None, -1.0, []
    for part in mig_partitions(12, 4):
        table = default_mps_table(part, 4)
        plan = make_plan(space_of(full, table), prof)
        sch, best = optimum_schedules(plan, Q)
        am = float(np.mean(np.asarray(pool.solo_ticks, np.int64)[Q].sum(1) / best))
        per_p.append((part, am))
        if am > best_am:
            best_p, best_am, best_plan, best_sch = part, am, plan, sch
    methods["MIG+MPS Default (C<=4)"] = job_metrics(best_plan, pool, Q, best_sch)
    t = time.time()
    w, log, cfg = train_policy(pool, args.steps, args.envs, args.lr)
    train_s = time.time() - t
    rl = rl_schedules(pool, Q, w, cfg)
    methods["MIG+MPS w/ RL (C<=4)"] = job_metrics(full_plan, pool, Q, rl)
    # the paper-literal sequential agent: flat head over the setups, job
    # sets in queue order
    ws, log_s, cfg_s = train_policy(pool, args.steps, args.envs, args.lr, agent="sequential")
    rl_s = rl_schedules(pool, Q, ws, cfg_s)
    methods["RL sequential (C<=4)"] = job_metrics(full_plan, pool, Q, rl_s)
    names = list(methods)
    lines = []
    for metric, key, fmt in (("Relative throughput (Solo / CoRun, Fig. 8)", "throughput", "{:.3f}"),
                             ("Mean AppSlowdown (Fig. 11)", "mean_slowdown", "{:.3f}"),
                             ("Fairness min/max AppSlowdown (Fig. 12)", "fairness", "{:.3f}")):
        lines.append(f"\n### {metric}\n")
        lines.append("| mix | " + " | ".join(names) + " |")
        lines.append("|" + "---|" * (len(names) + 1))
        for i in range(len(Q)):
            lines.append(f"| Q{i + 1} | " + " | ".join(fmt.format(methods[n][i][key])
                                                       for n in names) + " |")
        lines.append("| AM | " + " | ".join(fmt.format(np.mean([m[key] for m in methods[n]]))
                                            for n in names) + " |")
    rl_vs_opt = [methods["MIG+MPS w/ RL (C<=4)"][i]["throughput"] /
                 methods["MIG+MPS optimum (C<=4)"][i]["throughput"] for i in range(len(Q))]
    txt = "\n".join(lines)
    meta = {"device": torch.cuda.get_device_name(0), "train_steps": args.steps,
            "train_envs": args.envs, "lr": args.lr, "train_seconds": round(train_s, 1),
            "optimizer": "adam + huber(10)", "rl_throughput_fraction_of_optimum": rl_vs_opt,
            "rl_fraction_of_optimum_am": float(np.mean(rl_vs_opt)),
            "rl_job_sets": rl, "rl_sequential_job_sets": rl_s,
            "mig_mps_default_partition": best_p,
            "mig_mps_default_am_per_partition": [[list(p), a] for p, a in per_p],
            "optimum_seconds_per_call_12_windows":
                {k: round(v, 4) for k, v in timing.items()}, "train_log": log}
    print(txt)
    print(json.dumps({k: v for k, v in meta.items() if k != "train_log"}))
    if args.out:
        with open(args.out, "w") as f:
            f.write("# Schedule quality of the compared methods on Q1-Q12 (synthetic co-run "
                    "model R8)\n\nProduced by `tools/schedule_quality.py` on one B200: exhaustive "
                    "optima per method's search space (hrp_brute_run, P:245-248), the trained "
                    "agent's greedy episodes (hrp_env_step, epsilon = 0), per-job co-run times "
                    "(hrp_job_times).  AppSlowdown = CoRunAppTime / SoloRunAppTime (P:293); "
                    "Fairness = min / max AppSlowdown over the queue (P:309).\n"
                    + txt + "\n\n```\n" + json.dumps(meta, indent=1) + "\n```\n")


if __name__ == "__main__":
    main()
