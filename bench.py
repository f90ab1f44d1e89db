#!/usr/bin/env python
"""Benchmark of the hot path (BASELINE.json metric: DQN env-steps/s + Q-evals/s, fraction of
roofline) on BASELINE config 2: W=16 jobs, Cmax=3, full MIG GI/CI x MPS {10..90}% action space
(191,312 joint actions), Q-MLP 3x256, E=4096 envs, B=4096 replay batch per GPU.

One step = hrp_env_step (encode, Q forward, score every valid action + argmax, epsilon-greedy,
reward, transition, replay insert) + hrp_dqn_update (replay sample, online/target forward,
double-DQN argmax on s', TD loss, backward, [NCCL allreduce], SGD, target sync every 25).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 2]
Under torchrun each rank runs E envs (weak scaling, one process per GPU).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "DQN env-steps/sec + Q-evals/sec at 1/2/4/8 B200; fraction of roofline"
UNIT = "env-steps/s"


def workload_name(cfg):
    s = cfg.space
    return (f"cfg{cfg.name[-1]}: W={s.window} jobs, Cmax={s.cmax}, MIG GI/CI x MPS "
            f"{{{min(s.shares)}..{max(s.shares)}}}%, Q-MLP {cfg.net.hidden_layers}x"
            f"{cfg.net.hidden_width}, E={cfg.n_envs} envs, B={cfg.batch} per GPU")


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------------------------------
def cpu_baseline(cfg, seconds=15.0):
    """The oracle as it stands, single-threaded, on a bounded sample of the workload."""
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(1)
    except Exception:
        lim = None
    from oracle import env as EV
    from oracle import qnet as QN
    from oracle import space as SP
    pool = synth.make_pool(cfg.pool)
    sc = cfg.space
    osp = SP.build_space(sc.window, sc.cmax, sc.shares, sc.mig)
    th = synth.init_weights(QN.net_dims(osp, cfg.net))
    E = 32
    orc = EV.OracleDQN(osp, pool, cfg.net, th, E, E, 1 << 12, gamma=cfg.gamma, lr=cfg.lr)
    orc.reset(synth.make_windows(pool, E, sc.window))
    t0 = time.perf_counter()
    steps = 0
    while True:
        st = synth.step_streams(steps, E, E, sc.window, pool)
        orc.env_step(synth.eps_threshold(60, cfg.n_decay), st["u_explore"], st["u_action"],
                     st["next_windows"])
        orc.dqn_update(st["u_replay"], (steps + 1) % cfg.target_sync == 0)
        steps += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    if lim is not None:
        lim.unregister() if hasattr(lim, "unregister") else None
    return {"value": E * steps / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{steps} oracle steps of cfg{cfg.name[-1]} at E=B={E} (env step + DQN "
                      f"update, explicit argmax over every valid action), 1 thread, {dt:.1f} s"}


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import env as EV
    from oracle import qnet as QN
    from oracle import space as SP
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    pool = synth.make_pool(cfg.pool)
    sc = cfg.space
    osp = SP.build_space(sc.window, sc.cmax, sc.shares, sc.mig)
    th = synth.init_weights(QN.net_dims(osp, cfg.net))
    E = 16
    orc = EV.OracleDQN(osp, pool, cfg.net, th, E, E, 1 << 12, gamma=cfg.gamma, lr=cfg.lr)
    orc.reset(synth.make_windows(pool, E, sc.window))

    def step(t):
        st = synth.step_streams(t, E, E, sc.window, pool)
        orc.env_step(synth.eps_threshold(t, cfg.n_decay), st["u_explore"], st["u_action"],
                     st["next_windows"])
        orc.dqn_update(st["u_replay"], (t + 1) % cfg.target_sync == 0)

    for t in range(args.warmup):
        step(t)
    t0 = time.perf_counter()
    for t in range(args.steps):
        step(args.warmup + t)
    dt = time.perf_counter() - t0
    v = E * args.steps / dt
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": workload_name(cfg),
                                           "sample": f"E=B={E} envs per step (oracle)"},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": f"E=B={E} per step, {args.steps} steps, 1 thread"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, dev):
        self.p = None
        self.path = f"/tmp/hrp_clocks_{os.getpid()}.csv"
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(dev), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.15)
        self.p.terminate()
        self.p.wait()
        rows = []
        for ln in open(self.path):
            f = [x.strip() for x in ln.split(",")]
            if len(f) >= 7 and f[0].isdigit():
                rows.append(f)
        if not rows:
            return None
        sm = [int(r[0]) for r in rows]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, n in enumerate(names):
                if r[3 + k].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": int(rows[0][1]),
                "reasons": sorted(reasons), "samples": len(rows)}


def run_gpu(args, cfg):
    import torch
    import torch.distributed as dist
    from paper_2405_08754_b200 import hrp
    from paper_2405_08754_b200.session import Session, streams_to_dev

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    nccl_id = None
    if world > 1:
        buf = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(hrp.hrp_nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, 0)
        nccl_id = bytes(buf.cpu().numpy().tobytes())
    pool = synth.make_pool(cfg.pool)
    sc = cfg.space
    stream = torch.cuda.Stream(dev)
    from paper_2405_08754_b200.session import space_of
    tab = hrp.hrp_layout_table(space_of(sc))           # host tables from libhrp
    osp = TableInfo(sc, tab)
    th = synth.init_weights(osp.dims(cfg.net))
    E, B = cfg.n_envs, cfg.batch
    with torch.cuda.stream(stream):
        sess = Session(cfg, pool, init_weights=th, device=local, rank=rank, world=world,
                       nccl_id=nccl_id, argmax_mode=args.argmax, gemm_mode=args.gemm,
                       stream=stream)
        sess.reset(synth.make_windows(pool, E, sc.window, rank=rank, first_env=rank * E))
    total = args.warmup + args.steps
    # per-step host streams, resident in HBM before the timed region
    streams_h = [synth.step_streams(t, E, B, sc.window, pool, rank=rank, first_env=rank * E)
                 for t in range(total)]
    streams_d = [streams_to_dev(s, dev) for s in streams_h]
    thr = [synth.eps_threshold(t, cfg.n_decay) for t in range(total)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def one_step(t, d):
        sess.step(thr[t], d["u_explore"], d["u_action"], d["next_windows"], extras=False)
        sess.update(d["u_replay"], (t + 1) % cfg.target_sync == 0, extras=False)

    with torch.cuda.stream(stream):
        for t in range(args.warmup):
            one_step(t, streams_d[t])
        stream.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        n_launch0 = sess.launches()
        evals0 = hrp.hrp_eval_count(sess.ctx)
        clocks = Clocks(local)
        hrp.hrp_profile(sess.ctx, True)
        for k in range(args.steps):
            t = args.warmup + k
            flush.zero_()                       # L2 flushed between timed steps
            ev0[k].record(stream)
            one_step(t, streams_d[t])
            ev1[k].record(stream)
        stream.synchronize()
        clk = clocks.stop()
        prof = hrp.hrp_profile_read(sess.ctx)
        hrp.hrp_profile(sess.ctx, False)
        n_launch = sess.launches() - n_launch0
        evals = hrp.hrp_eval_count(sess.ctx) - evals0
        ms = sum(a.elapsed_time(b) for a, b in zip(ev0, ev1))
    # max over ranks
    t_all = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_all, op=dist.ReduceOp.MAX)
    ms = float(t_all.item())
    value = world * E * args.steps / (ms / 1e3)

    # ---- e2e: host pinned streams copied in, results copied out, inside the timed region
    with torch.cuda.stream(stream):
        pinned = []
        for t in range(args.steps):
            s = streams_h[args.warmup + t]
            pinned.append({k: torch.from_numpy(np.ascontiguousarray(
                v.view(np.int32) if v.dtype == np.uint32 else
                (v.view(np.int64) if v.dtype == np.uint64 else v))).pin_memory()
                for k, v in s.items()})
        bufs = {k: torch.empty_like(v, device=dev) for k, v in pinned[0].items()}
        out_h = {"actions": torch.empty(E, dtype=torch.int64).pin_memory(),
                 "rewards": torch.empty(E, dtype=torch.float32).pin_memory(),
                 "loss": torch.empty(1, dtype=torch.float32).pin_memory()}
        h2d = sum(v.numel() * v.element_size() for v in pinned[0].values())
        d2h = sum(v.numel() * v.element_size() for v in out_h.values())
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(args.steps):
            t = args.warmup + k
            for key, v in pinned[k].items():
                bufs[key].copy_(v, non_blocking=True)
            one_step(t, bufs)
            out_h["actions"].copy_(sess.actions, non_blocking=True)
            out_h["rewards"].copy_(sess.rewards, non_blocking=True)
            out_h["loss"].copy_(sess.loss, non_blocking=True)
        e1.record(stream)
        stream.synchronize()
        ms_e2e = e0.elapsed_time(e1)
    te = torch.tensor([ms_e2e], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * E * args.steps / (float(te.item()) / 1e3)

    if rank == 0:
        res = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
               "dtype": "f32+i64", "data": "synthetic",
               "config": {"workload": workload_name(cfg), "global_envs": world * E,
                          "actions_per_state": int(sess_actions(osp)),
                          "argmax": "explicit" if sess_explicit(args, sc) else "pruned-exact",
                          "gemm": {0: "auto", 1: "fp32 CUDA-core", 2: "tcgen05 3xTF32"}[args.gemm],
                          "l2": "flushed (256 MiB memset) between timed steps",
                          "parallelism": f"dp{world} (env sharding + NCCL grad allreduce)"},
               "q_evals_per_s": evals * world / (ms / 1e3),
               "q_evals_per_step": evals / args.steps,
               "gpu_launches": int(n_launch),
               "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                       "d2h_bytes_per_step": int(d2h)},
               "clocks": clk,
               "kernels_ms_per_step": {k: v[0] / args.steps for k, v in prof.items() if v[1]}}
        res["roofline"] = roofline(prof, args.steps, evals, cfg, osp, world)
        if not args.no_cpu_baseline and world == 1:
            res["cpu_baseline"] = cpu_baseline(cfg, args.cpu_seconds)
        print(json.dumps(res), flush=True)
    sess.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


class TableInfo:
    def __init__(self, sc, tab):
        self.W, self.cmax = sc.window, sc.cmax
        self.L, self.T, self.n_actions = tab["n_layouts"], tab["n_types"], tab["n_actions"]
        self.H = 1 + self.L + self.W * self.T

    def dims(self, net):
        return [self.W * 17] + [net.hidden_width] * net.hidden_layers + [self.H]


def sess_actions(osp):
    return osp.n_actions


def sess_explicit(args, sc):
    return args.argmax == 1 or (args.argmax == 0 and sc.window <= 16)


def roofline(prof, steps, evals, cfg, osp, world):
    """Dominant kernel's achieved vs peak."""
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    top = max(prof.items(), key=lambda kv: kv[1][0])
    name, (ms, cnt) = top
    sec = ms / 1e3
    clock = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    if name in ("select", "td"):
        # ALU bound: algorithmic int32-lane ops = explicit Q^ evals x (2C + 2)
        C = osp.cmax
        ops = (evals / 2.0) * (2 * C + 2)   # select + td each hold ~half of the evals
        peak = 148 * 128 * clock / 1e12    # Tops/s (lane-ops), 148 SMs x 128 lanes x f_max
        ach = ops / sec / 1e12
        return {"kernel": name, "bound": "alu", "achieved": ach, "peak": peak, "unit": "Tops/s",
                "frac": ach / peak, "traffic": None,
                "peak_src": "derived: 148 SM x 128 int32 lanes x sm_max_mhz (MEASURED_PEAKS)"}
    if name.startswith("gemm"):
        dims = [osp.W * 17] + [cfg.net.hidden_width] * cfg.net.hidden_layers + [osp.H]
        F = sum(2 * dims[i] * dims[i + 1] for i in range(len(dims) - 1))
        if name == "gemm_fwd":
            flops = (cfg.n_envs + 3 * cfg.batch) * F * steps
        else:
            flops = cfg.batch * (2 * F - 2 * dims[0] * dims[1]) * steps
        ach = flops / sec / 1e12
        peak = float(peaks.get("bf16_tflops_sustained", 1407.2)) / 2.0  # tf32 = bf16 / 2
        return {"kernel": name, "bound": "tensor", "achieved": ach, "peak": peak,
                "unit": "TFLOP/s", "frac": ach / peak, "traffic": None,
                "peak_src": "MEASURED_PEAKS bf16_tflops_sustained x 1/2 (tf32 nominal ratio)"}
    return {"kernel": name, "bound": "hbm", "achieved": None,
            "peak": float(peaks.get("hbm_gbs", 6453.7)), "unit": "GB/s", "frac": None,
            "traffic": None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--argmax", type=int, default=0, help="0 auto, 1 explicit, 2 pruned")
    ap.add_argument("--gemm", type=int, default=0, help="0 auto, 1 CUDA-core fp32, 2 tcgen05")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = synth.config(args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_gpu(args, cfg)


if __name__ == "__main__":
    main()
