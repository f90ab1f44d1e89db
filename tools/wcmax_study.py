"""W / Cmax scaling study (Fig. 9-10) on one B200.

Part A -- schedule quality: the queue's relative throughput (sum of solo times / sum of co-run
times) of the exhaustive MIG+MPS optimum when the scheduler sees W jobs at a time (each 12-job
Table V queue cut into consecutive windows of W jobs, the last one shorter), for W in
{2, 3, 4, 6, 8, 10, 12} at Cmax = 4 (Fig. 9) and Cmax in {1, 2, 3, 4} at W = 12 (Fig. 10).
Part B -- hot-path cost: the action-space size, libhrp's DQN step throughput (env step + DQN
update, E = B = 4096, 3 x 256 MLP, exact pruned argmax) and the exhaustive search's windows/s
over the same grid, plus the DQN step at W = 16, 32, 64.
Parity of every grid point: tests/test_gpu_wcmax.py.

usage: python tools/wcmax_study.py [--out profiles/r2_wcmax_study.md]
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

S10 = tuple(range(10, 100, 10))


def queue_throughput(pool, Q, W, cmax, plans):
    """Per queue: sum solo / sum optimum co-run over consecutive windows of W jobs."""
    from paper_2405_08754_b200 import hrp
    from paper_2405_08754_b200.schedule import make_plan, optimum_schedules
    from paper_2405_08754_b200.session import space_of
    prof = hrp.make_profiles(pool)
    tot_solo = np.zeros(len(Q), np.int64)
    tot_co = np.zeros(len(Q), np.int64)
    for s in range(0, Q.shape[1], W):
        chunk = np.ascontiguousarray(Q[:, s:s + W])
        w = chunk.shape[1]
        key = (w, min(cmax, w))
        if key not in plans:
            plans[key] = make_plan(space_of(synth.SpaceCfg(w, min(cmax, w), S10)), prof)
        _, best = optimum_schedules(plans[key], chunk)
        tot_co += best
        tot_solo += np.asarray(pool.solo_ticks, np.int64)[chunk].sum(1)
    return tot_solo / tot_co


def dqn_rate(pool, W, cmax, E=4096, steps=10, warmup=3):
    """env-steps/s of hrp_env_step + hrp_dqn_update (device time, CUDA events)."""
    import torch
    from paper_2405_08754_b200 import hrp
    from paper_2405_08754_b200.session import Session, space_of, streams_to_dev
    sc = synth.SpaceCfg(W, cmax, S10)
    cfg = synth.config(2).with_(space=sc)
    tab = hrp.hrp_layout_table(space_of(sc))
    H = 1 + tab["n_layouts"] + W * tab["n_types"]
    th = synth.init_weights([W * 17, 256, 256, 256, H])
    sess = Session(cfg, pool, n_envs=E, batch=E, init_weights=th)
    sess.reset(synth.make_windows(pool, E, W))
    st = [streams_to_dev(synth.step_streams(t, E, E, W, pool), sess.dev)
          for t in range(steps + warmup)]
    for t in range(warmup):
        sess.step(synth.eps_threshold(40 + t, 50), st[t]["u_explore"], st[t]["u_action"],
                  st[t]["next_windows"], extras=False)
        sess.update(st[t]["u_replay"], False, extras=False)
    torch.cuda.synchronize()
    e0 = hrp.hrp_eval_counts(sess.ctx)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for t in range(warmup, warmup + steps):
        sess.step(synth.eps_threshold(40 + t, 50), st[t]["u_explore"], st[t]["u_action"],
                  st[t]["next_windows"], extras=False)
        sess.update(st[t]["u_replay"], False, extras=False)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    e1 = hrp.hrp_eval_counts(sess.ctx)
    sess.close()
    return {"env_steps_per_s": E * steps / (ms / 1e3), "ms_per_step": ms / steps,
            "candidates_per_s": (sum(e1) - sum(e0)) / (ms / 1e3), "n_actions": tab["n_actions"],
            "layouts": tab["n_layouts"], "slot_types": tab["n_types"], "head_width": H}


def brute_rate(pool, W, cmax, n=4096, reps=3):
    import torch
    from paper_2405_08754_b200 import hrp
    from paper_2405_08754_b200.session import space_of
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    plan = hrp.hrp_brute_create(space_of(synth.SpaceCfg(W, cmax, S10)), hrp.make_profiles(pool),
                                0, st.cuda_stream)
    w = torch.from_numpy(synth.make_windows(pool, n, W, step=5)).to(dev)
    outs = [torch.empty(n, dtype=torch.int64, device=dev), torch.empty(n, dtype=torch.int64,
                                                                       device=dev),
            torch.empty((n, W), dtype=torch.uint8, device=dev),
            torch.empty((n, W), dtype=torch.int64, device=dev)]
    hrp.hrp_brute_run(plan, n, w, *outs, st.cuda_stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        hrp.hrp_brute_run(plan, n, w, *outs, st.cuda_stream)
    b.record()
    torch.cuda.synchronize()
    hrp.hrp_brute_destroy(plan)
    return n * reps / (a.elapsed_time(b) / 1e3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    pool = synth.make_pool(27)
    Q = synth.table_v_windows(pool)
    plans = {}
    rows_w, rows_c = [], []
    for W in (2, 3, 4, 6, 8, 10, 12):
        tp = queue_throughput(pool, Q, W, 4, plans)
        r = {"W": W, "cmax": min(4, W), "throughput_am": float(tp.mean()),
             "throughput_max": float(tp.max()), "brute_windows_per_s": brute_rate(pool, W, min(4, W))}
        if W >= 4:
            r.update(dqn_rate(pool, W, 4))
        rows_w.append(r)
        print(json.dumps(r), flush=True)
    for cmax in (1, 2, 3, 4):
        tp = queue_throughput(pool, Q, 12, cmax, plans)
        r = {"W": 12, "cmax": cmax, "throughput_am": float(tp.mean()),
             "throughput_max": float(tp.max()), "brute_windows_per_s": brute_rate(pool, 12, cmax)}
        r.update(dqn_rate(pool, 12, cmax))
        rows_c.append(r)
        print(json.dumps(r), flush=True)
    big = []
    for W, cmax in ((16, 3), (16, 4), (32, 3), (32, 4), (64, 3), (64, 4)):
        r = {"W": W, "cmax": cmax}
        r.update(dqn_rate(pool, W, cmax))
        big.append(r)
        print(json.dumps(r), flush=True)

    def table(rows, keys):
        hdr = "| " + " | ".join(k for k, _ in keys) + " |"
        out = [hdr, "|" + "---|" * len(keys)]
        for r in rows:
            out.append("| " + " | ".join(f.format(r[k]) if k in r else "-" for k, f in keys) + " |")
        return "\n".join(out)
    keys = [("W", "{}"), ("cmax", "{}"), ("throughput_am", "{:.3f}"), ("throughput_max", "{:.3f}"),
            ("n_actions", "{:,}"), ("brute_windows_per_s", "{:,.0f}"),
            ("env_steps_per_s", "{:,.0f}"), ("ms_per_step", "{:.3f}")]
    keys2 = [("W", "{}"), ("cmax", "{}"), ("n_actions", "{:,}"), ("layouts", "{}"),
             ("head_width", "{}"), ("env_steps_per_s", "{:,.0f}"), ("ms_per_step", "{:.3f}"),
             ("candidates_per_s", "{:.3g}")]
    txt = ("## Fig. 9 analogue: window size W (Cmax = 4)\n\n" + table(rows_w, keys) +
           "\n\n## Fig. 10 analogue: Cmax (W = 12)\n\n" + table(rows_c, keys) +
           "\n\n## DQN step beyond the paper's window (E = B = 4096, 3 x 256, pruned argmax)\n\n"
           + table(big, keys2) + "\n")
    print(txt)
    if args.out:
        with open(args.out, "w") as f:
            f.write("# W / Cmax scaling study (synthetic co-run model R8, one B200)\n\n"
                    "Produced by `tools/wcmax_study.py`.  throughput = sum of solo times / sum of "
                    "the exhaustive MIG+MPS optimum's co-run times over the 12-job Table V queues "
                    "cut into consecutive windows of W jobs (AM and max over Q1-Q12); "
                    "brute_windows_per_s = hrp_brute_run on 4,096 random windows; "
                    "env_steps_per_s = hrp_env_step + hrp_dqn_update at E = B = 4,096 "
                    f"(device: {torch.cuda.get_device_name(0)}).\n\n" + txt)


if __name__ == "__main__":
    main()
