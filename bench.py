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
# one JSON line on stdout: keep NCCL's banner off it (HRP_NCCL_DEBUG overrides)
os.environ["NCCL_DEBUG"] = os.environ.get("HRP_NCCL_DEBUG", "WARN")

import synth  # noqa: E402

METRIC = "DQN env-steps/sec + Q-evals/sec at 1/2/4/8 B200; fraction of roofline"
UNIT = "env-steps/s"


def workload_name(cfg, E=None, B=None, scaling="weak"):
    s = cfg.space
    E = cfg.n_envs if E is None else E
    B = cfg.batch if B is None else B
    shard = (f"E={cfg.n_envs} envs, B={cfg.batch} global, sharded ({E} / {B} per GPU)"
             if scaling == "strong" else f"E={E} envs, B={B} per GPU")
    return (f"cfg{cfg.name[-1]}: W={s.window} jobs, Cmax={s.cmax}, MIG GI/CI x MPS "
            f"{{{min(s.shares)}..{max(s.shares)}}}%, Q-MLP {cfg.net.hidden_layers}x"
            f"{cfg.net.hidden_width}, {shard}")


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------------------------------
def host_cores():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def _oracle_rate(cfg, E, seconds, workers):
    """env-steps/s of the oracle (env step + DQN update, explicit argmax over every valid
    action, eps late in the schedule) on E envs, BLAS on one thread per process."""
    from oracle import env as EV
    from oracle import qnet as QN
    from oracle import space as SP
    pool = synth.make_pool(cfg.pool)
    sc = cfg.space
    osp = SP.build_space(sc.window, sc.cmax, sc.shares, sc.mig)
    th = synth.init_weights(QN.net_dims(osp, cfg.net))
    orc = EV.OracleDQN(osp, pool, cfg.net, th, E, E, 1 << 12, gamma=cfg.gamma, lr=cfg.lr,
                       workers=workers)
    orc.reset(synth.make_windows(pool, E, sc.window))
    if workers > 1:
        orc.q_forward(orc.windows[:2], orc.sched[:2])     # start the worker processes untimed
    steps = 0
    t0 = time.perf_counter()
    while True:
        st = synth.step_streams(steps, E, E, sc.window, pool)
        orc.env_step(synth.eps_threshold(60, cfg.n_decay), st["u_explore"], st["u_action"],
                     st["next_windows"])
        orc.dqn_update(st["u_replay"], (steps + 1) % cfg.target_sync == 0)
        steps += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    orc.close()
    return E * steps / dt, steps, dt


def cpu_baseline(cfg, seconds=15.0):
    """The oracle as it stands on a bounded sample of the workload, on this box's host cores:
    all-core mode (the per-state argmax mapped over one process per core, BLAS 1 thread) as the
    reported value, single-thread mode beside it."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    cores = host_cores()
    v1, n1, t1 = _oracle_rate(cfg, 32, seconds / 2, 0)
    Ea = max(32, 8 * cores)
    va, na, ta = _oracle_rate(cfg, Ea, seconds / 2, cores)
    name = f"cfg{cfg.name[-1]}"
    return {"value": va, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{na} oracle steps of {name} at E=B={Ea} (env step + DQN update, explicit "
                      f"argmax over every valid action mapped over {cores} processes), "
                      f"{ta:.1f} s",
            "single_thread": {"value": v1, "unit": UNIT, "cores": 1,
                              "sample": f"{n1} oracle steps at E=B=32, 1 thread, {t1:.1f} s"}}


def run_reference(args, cfg):
    """The reference arm: the oracle as it stands (there is no reference implementation to
    install, /root/reference holds only the paper) on this box's host cores, each step a
    bounded sample (E = B = 16 envs) of the workload."""
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
    cores = host_cores()
    pool = synth.make_pool(cfg.pool)
    sc = cfg.space
    osp = SP.build_space(sc.window, sc.cmax, sc.shares, sc.mig)
    th = synth.init_weights(QN.net_dims(osp, cfg.net))
    E = 16
    orc = EV.OracleDQN(osp, pool, cfg.net, th, E, E, 1 << 12, gamma=cfg.gamma, lr=cfg.lr,
                       workers=cores)
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
    orc.close()
    v = E * args.steps / dt
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": workload_name(cfg),
                                           "sample": f"E=B={E} envs per step (oracle)"},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                            "sample": f"E=B={E} per step, {args.steps} steps, argmax mapped over "
                                      f"{cores} processes"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------------------
class Clocks:
    """SM clock + throttle-reason sampling DURING the timed region (B200_PROFILING.md clocks
    line). A timed region here is ~10 ms of GPU work, shorter than nvidia-smi's 100 ms
    sampling period, so NVML is polled from a thread every ~5 ms while the host waits on the
    stream (a 0.5 ms period perturbed the GPU: cfg 3 ran 42-57 k instead of 80 k windows/s,
    profiles/r1zp_cfg3_nvml_period.txt); one sample is always taken at stop(). Falls back to nvidia-smi if NVML is
    unavailable."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, dev):
        import threading
        self.rows = []
        self.src = None
        self.p = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            ids = [x.strip() for x in vis.split(",") if x.strip()]
            if ids and len(ids) > dev:
                tok = ids[dev]
                h = (nv.nvmlDeviceGetHandleByIndex(int(tok)) if tok.isdigit()
                     else nv.nvmlDeviceGetHandleByUUID(tok))
            else:
                h = nv.nvmlDeviceGetHandleByIndex(dev)
            self.nv, self.h = nv, h
            self.smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.bits = (nv.nvmlClocksEventReasonHwSlowdown,
                         nv.nvmlClocksEventReasonHwThermalSlowdown,
                         nv.nvmlClocksEventReasonSwThermalSlowdown,
                         nv.nvmlClocksEventReasonSwPowerCap)
            self._sample()
            self.rows.clear()
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()
            self.src = "nvml"
        except Exception:
            self._smi(dev)

    def _sample(self):
        nv, h = self.nv, self.h
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        self.rows.append((sm, self.smax, [n for n, b in zip(self.NAMES, self.bits) if r & b]))

    def _loop(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            time.sleep(0.005)   # NVML queries every 0.5 ms slowed the brute-force kernel (r1zp)

    def _smi(self, dev):
        self.path = f"/tmp/hrp_clocks_{os.getpid()}.csv"
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(dev), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            self.src = "nvidia-smi"
        except Exception:
            self.p = None

    def stop(self):
        if self._t is not None:
            self._stop.set()
            self._t.join()
            try:
                self._sample()
            except Exception:
                pass
        elif self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            self.p.wait()
            for ln in open(self.path):
                f = [x.strip() for x in ln.split(",")]
                if len(f) >= 7 and f[0].isdigit():
                    self.rows.append((int(f[0]), int(f[1]),
                                      [n for k, n in enumerate(self.NAMES)
                                       if f[3 + k].lower() == "active"]))
        if not self.rows:
            return None
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for r in self.rows for n in r[2]})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": int(self.rows[0][1]),
                "reasons": reasons, "samples": len(self.rows), "source": self.src}


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
    from paper_2405_08754_b200 import parallel
    nccl_id = parallel.nccl_unique_id(dev) if world > 1 else None
    if world == 1 and args.comm1:
        nccl_id = hrp.hrp_nccl_unique_id()    # one-rank communicator: the allreduce path on 1 GPU
    pool = synth.make_pool(cfg.pool)
    sc = cfg.space
    stream = torch.cuda.Stream(dev)
    from paper_2405_08754_b200.session import space_of
    tab = hrp.hrp_layout_table(space_of(sc))           # host tables from libhrp
    osp = TableInfo(sc, tab)
    th = synth.init_weights(osp.dims(cfg.net))
    if args.scaling == "strong":
        # config 4: the global E = B = 65,536 sharded across the ranks
        assert cfg.n_envs % world == 0 and cfg.batch % world == 0
        E, B = cfg.n_envs // world, cfg.batch // world
    else:
        E, B = cfg.n_envs, cfg.batch                     # per rank (weak scaling)
    with torch.cuda.stream(stream):
        sess = Session(cfg, pool, n_envs=E, batch=B, init_weights=th, device=local, rank=rank,
                       world=world,
                       nccl_id=nccl_id, argmax_mode=args.argmax, stream=stream)
        sess.reset(synth.make_windows(pool, E, sc.window, rank=rank,
                                       first_env=parallel.env_shard(E, rank)))
    total = args.warmup + args.steps
    # per-step host streams, resident in HBM before the timed region
    streams_h = [synth.step_streams(t, E, B, sc.window, pool, rank=rank,
                                    first_env=parallel.env_shard(E, rank))
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
        evals0 = hrp.hrp_eval_counts(sess.ctx)
        cov0 = hrp.hrp_covered_counts(sess.ctx)
        graphs = []
        if args.graph:
            # one CUDA graph per timed step (each step's inputs live at their own addresses and
            # the context's host counters -- step t, replay fill -- advance as the launches are
            # recorded), replayed once each, in capture order.  With world > 1 the per-layer
            # NCCL allreduces are captured into the same graph.
            for k in range(args.steps):
                t = args.warmup + k
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    one_step(t, streams_d[t])
                graphs.append(g)
            stream.synchronize()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
        clocks = Clocks(local)
        for k in range(args.steps):
            t = args.warmup + k
            flush.zero_()                       # L2 flushed between timed steps
            ev0[k].record(stream)
            if args.graph:
                graphs[k].replay()
            else:
                one_step(t, streams_d[t])
            ev1[k].record(stream)
        stream.synchronize()
        clk = clocks.stop()
        n_launch = sess.launches() - n_launch0
        evals1 = hrp.hrp_eval_counts(sess.ctx)
        evals_k = (evals1[0] - evals0[0], evals1[1] - evals0[1])
        evals = evals_k[0] + evals_k[1]
        cov1 = hrp.hrp_covered_counts(sess.ctx)
        covered = (cov1[0] - cov0[0]) + (cov1[1] - cov0[1])
        ms = sum(a.elapsed_time(b) for a, b in zip(ev0, ev1))
        # per-kernel breakdown: a separate pass over the same step inputs with per-launch CUDA
        # events on the context's stream (kept out of the timed region above: the extra
        # event records perturb a ~1 ms step)
        # (with --graph the profiled steps are captured too, event records included, so the
        # per-launch intervals hold GPU time only, not host launch gaps of eager submission)
        hrp.hrp_profile(sess.ctx, True)
        pgraphs = []
        if args.graph:
            for k in range(args.steps):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    one_step(args.warmup + k, streams_d[args.warmup + k])
                pgraphs.append(g)
            stream.synchronize()
        for k in range(args.steps):
            t = args.warmup + k
            flush.zero_()
            if args.graph:
                pgraphs[k].replay()
            else:
                one_step(t, streams_d[t])
        stream.synchronize()
        prof = hrp.hrp_profile_read(sess.ctx)
        hrp.hrp_profile(sess.ctx, False)
        del pgraphs
    # max over ranks
    ms = parallel.max_over_ranks(ms, dev)
    value = world * E * args.steps / (ms / 1e3)     # all ranks' env-steps / slowest rank's time

    # ---- e2e: host pinned streams copied in, results copied out, inside the timed region
    with torch.cuda.stream(stream):
        # one pinned staging buffer per step holding the four input streams (256-B aligned
        # slots) -> ONE host-to-device copy; the step's outputs (actions, rewards, loss) are
        # views of one device buffer -> ONE device-to-host copy
        def layout(items):
            offs, o = {}, 0
            for k, n in items:
                offs[k] = o
                o = (o + n + 255) // 256 * 256
            return offs, o

        def as_bytes(v):
            a = np.ascontiguousarray(v.view(np.int32) if v.dtype == np.uint32 else
                                     (v.view(np.int64) if v.dtype == np.uint64 else v))
            return a.view(np.uint8).reshape(-1), a.dtype
        s0 = streams_h[args.warmup]
        in_items = [(k, as_bytes(v)[0].size) for k, v in s0.items()]
        in_off, in_size = layout(in_items)
        pinned = []
        for t in range(args.steps):
            buf = torch.empty(in_size, dtype=torch.uint8).pin_memory()
            for k, v in streams_h[args.warmup + t].items():
                b, _ = as_bytes(v)
                buf[in_off[k]:in_off[k] + b.size].copy_(torch.from_numpy(b))
            pinned.append(buf)
        # double-buffered device inputs and outputs: step k+1's inputs are copied in (copy
        # stream) while step k computes, and step k's results are copied out while step k+1
        # computes; every step's copies are inside the one timed interval
        in_dev = [torch.empty(in_size, dtype=torch.uint8, device=dev) for _ in range(2)]
        bufs = [{}, {}]
        for k, v in s0.items():
            b, dt = as_bytes(v)
            tdt = {np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64,
                   np.dtype(np.uint8): torch.uint8}[np.dtype(dt)]
            for i in range(2):
                bufs[i][k] = in_dev[i][in_off[k]:in_off[k] + b.size].view(tdt)
        out_off, out_size = layout([("actions", 8 * E), ("rewards", 4 * E), ("loss", 4)])
        out_dev = [torch.empty(out_size, dtype=torch.uint8, device=dev) for _ in range(2)]

        def bind_outputs(i):
            o = out_dev[i]
            sess.actions = o[out_off["actions"]:out_off["actions"] + 8 * E].view(torch.int64)
            sess.rewards = o[out_off["rewards"]:out_off["rewards"] + 4 * E].view(torch.float32)
            sess.loss = o[out_off["loss"]:out_off["loss"] + 4].view(torch.float32)
        out_h = [torch.empty(out_size, dtype=torch.uint8).pin_memory() for _ in range(args.steps)]
        h2d = sum(n for _, n in in_items)
        d2h = 8 * E + 4 * E + 4
        cs = torch.cuda.Stream(dev)                 # copy stream
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        ev = lambda: torch.cuda.Event(enable_timing=False)
        ev_in = [ev() for _ in range(args.steps)]
        ev_done = [ev() for _ in range(args.steps)]
        ev_out = [ev() for _ in range(args.steps)]
        fl0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        fl1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)

        def e2e_compute(k):
            bind_outputs(k % 2)
            one_step(args.warmup + k, bufs[k % 2])

        graphs_e2e = []
        if args.graph:
            for k in range(args.steps):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    e2e_compute(k)
                graphs_e2e.append(g)
            stream.synchronize()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)

        def h2d_copy(k):                        # on the copy stream
            if k >= 2:
                cs.wait_event(ev_done[k - 2])   # step k-2 has finished reading in_dev[k % 2]
            in_dev[k % 2].copy_(pinned[k], non_blocking=True)
            ev_in[k].record(cs)

        t_start.record(stream)
        cs.wait_event(t_start)
        with torch.cuda.stream(cs):
            h2d_copy(0)
        for k in range(args.steps):
            if k + 1 < args.steps:
                with torch.cuda.stream(cs):
                    h2d_copy(k + 1)
            fl0[k].record(stream)
            flush.zero_()                       # L2 flushed between steps (its time excluded)
            fl1[k].record(stream)
            stream.wait_event(ev_in[k])
            if k >= 2:
                stream.wait_event(ev_out[k - 2])  # out_dev[k % 2] has been copied out
            if args.graph:
                graphs_e2e[k].replay()
            else:
                e2e_compute(k)
            ev_done[k].record(stream)
            with torch.cuda.stream(cs):
                cs.wait_event(ev_done[k])
                out_h[k].copy_(out_dev[k % 2], non_blocking=True)
                ev_out[k].record(cs)
        stream.wait_event(ev_out[args.steps - 1])
        t_end.record(stream)
        stream.synchronize()
        cs.synchronize()
        # the outputs landed in host memory: spot-check the last two against the device copies
        for k in range(max(0, args.steps - 2), args.steps):
            assert torch.equal(out_h[k].to(dev), out_dev[k % 2])
        ms_flush = sum(a.elapsed_time(b) for a, b in zip(fl0, fl1))
        ms_e2e = t_start.elapsed_time(t_end) - ms_flush
    e2e_value = world * E * args.steps / (parallel.max_over_ranks(ms_e2e, dev) / 1e3)

    if rank == 0:
        res = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
               "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
               "dtype": "f32+i64", "data": "synthetic",
               "config": {"workload": workload_name(cfg, E, B, args.scaling),
                          "global_envs": world * E, "envs_per_gpu": E, "batch_per_gpu": B,
                          "actions_per_state": int(sess_actions(osp)),
                          "argmax": "explicit" if sess_explicit(args, sc) else "pruned-exact",
                          "gemm": "tcgen05 3xTF32 (fp32-accurate), TMA + TMEM",
                          "l2": "flushed (256 MiB memset) between timed steps",
                          "launch": "CUDA graph per step (captured before the timed region)"
                                    if args.graph else "eager stream launches",
                          "parallelism": f"dp{world} (env sharding + NCCL grad allreduce)"
                                         + (" [one-rank NCCL communicator]" if world == 1 and
                                            args.comm1 else "")},
               "q_evals_per_s": covered * world / (ms / 1e3),
               "q_evals_per_step": covered / args.steps,
               "q_evals_def": ("valid (state, joint action) pairs covered by the exact argmax of "
                               "a5 + a9 (hrp_covered_counts): every valid action of every state "
                               "whose greedy action was computed -- what an explicit "
                               "enumeration scores; the exact search reaches the same maximum"),
               "candidates_scored_per_s": evals * world / (ms / 1e3),
               "candidates_def": ("actions actually scored (hrp_eval_counts): explicit mode, "
                                  "the leaves not skipped by the fp32 suffix-max bound; pruned "
                                  "mode, the Top-list assignments searched"),
               "gpu_launches": int(n_launch),
               "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                       "d2h_bytes_per_step": int(d2h),
                       "method": ("one timed interval over the K steps: each step's inputs "
                                  "copied in from pinned host memory on a copy stream while the "
                                  "previous step computes, its actions/rewards/loss copied out "
                                  "while the next computes (double-buffered); the L2 flushes "
                                  "between steps are timed and subtracted")},
               "clocks": clk,
               "kernels_ms_per_step": {k: v[0] / args.steps for k, v in prof.items() if v[1]}}
        rl = rooflines(prof, args.steps, evals_k, cfg, osp, E, B, burst=at_max_clock(clk),
                       explicit=sess_explicit(args, sc))
        res["roofline"] = dominant(rl, args.config)
        tot = sum(v["ms_per_step"] for v in rl.values())
        res["roofline"]["share_of_step"] = rl[res["roofline"]["kernel"]]["ms_per_step"] / tot
        res["rooflines"] = rl
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
    return args.argmax == 1       # auto = the exact pruned search (hrp.h argmax_mode)


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def at_max_clock(clk):
    """True when NVML saw the SM clock at its maximum with no throttle reason during the timed
    region: the burst peaks apply (B200_PROFILING.md), else the sustained ones."""
    if not clk:
        return False
    return clk["sm_mhz"] >= 0.97 * clk["sm_max_mhz"] and not clk["reasons"]


def tensor_peak(burst=True):
    """fp32-accurate tensor-core peak of the 3xTF32 GEMMs (TFLOP/s, logical fp32 products) and
    where it comes from: the measured cuBLAS TF32 peak (profiles/measured_peaks_r2.json,
    tools/measure_peaks.py) / 3 MMAs per product, else MEASURED_PEAKS bf16 x 1/2 (the guide's
    nominal TF32 : BF16 ratio) / 3."""
    own = _own_peaks()
    key = "tf32_tflops" if burst else "tf32_tflops_sustained"
    if own.get(key):
        return own[key] / 3.0, (f"measured cuBLAS TF32 {'burst' if burst else 'sustained'} "
                                f"(profiles/measured_peaks_r2.json) x 1/3 (3xTF32 MMAs per product)")
    pk = _peaks()
    bf = float(pk.get("bf16_tflops" if burst else "bf16_tflops_sustained", 1653.9))
    return bf / 2.0 / 3.0, (f"MEASURED_PEAKS bf16_tflops{'' if burst else '_sustained'} x 1/2 "
                            "(tf32 ratio) x 1/3 (3xTF32 MMAs per product)")


def alu_peak_tops(kind="fp32"):
    """FP32 (kind "fp32": the selection kernels' fp32 adds / compares) or INT32 (kind "int":
    the brute force) lane-op peak in T lane-ops/s: the measured add microbenchmark when
    committed, else 148 SMs x 128 lanes x sm_max_mhz."""
    own = _own_peaks()
    key = "alu_int_tops" if kind == "int" else "alu_tops"
    if own.get(key):
        return own[key], (f"measured {'int32' if kind == 'int' else 'fp32'} add microbenchmark "
                          "(hrp_diag_alu, profiles/measured_peaks_r2.json)")
    pk = _peaks()
    return (148 * 128 * float(pk.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12,
            "148 SM x 128 lanes x sm_max_mhz (MEASURED_PEAKS)")


def _own_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "measured_peaks_r2.json")))
    except Exception:
        return {}


def rooflines(prof, steps, evals, cfg, osp, E=None, B=None, burst=True, explicit=True):
    """Per kernel class: achieved vs peak.  `evals` = (select, td)
    explicit Q-evaluations over the timed steps; prof = {class: (ms, launches)}.  With the
    pruned argmax (explicit False) the selection kernels' unit is the head output they read
    once (E resp. B rows of H fp32 values): HBM-bound by construction."""
    pk = _peaks()
    alu_peak, alu_src = alu_peak_tops()
    fp32_tc, tc_src = tensor_peak(burst)
    hbm = float(pk.get("hbm_gbs", 6453.7))
    dims = [osp.W * 17] + [cfg.net.hidden_width] * cfg.net.hidden_layers + [osp.H]
    F = sum(2 * dims[i] * dims[i + 1] for i in range(len(dims) - 1))
    E = cfg.n_envs if E is None else E
    B = cfg.batch if B is None else B
    out = {}
    head_struct = prof.get("head_bwd", (0.0, 0))[1] > 0
    for name, (ms, cnt) in prof.items():
        if cnt == 0 or ms <= 0:
            continue
        sec = ms / 1e3
        per = {"ms_per_step": ms / steps, "launches_per_step": cnt / steps}
        if name in ("select", "td") and not explicit:
            rows = E if name == "select" else B
            byts = rows * osp.H * 4
            ach = byts * steps / sec / 1e9
            per.update(bound="hbm", achieved=ach, peak=hbm, unit="GB/s", frac=ach / hbm,
                       work=f"{byts / 1e6:.4g} MB/step (the head rows read once by the exact "
                            "pruned argmax)")
        elif name in ("select", "td"):
            n = evals[0] if name == "select" else evals[1]
            ach = 2.0 * n / sec / 1e12
            per.update(bound="alu", achieved=ach, peak=alu_peak, unit="Tops/s",
                       frac=ach / alu_peak, work=f"{n / steps:.4g} Q-evals/step (valid actions covered) x 2 lane-ops "
                            "(one add forming the score, one compare), the naive algorithm's "
                            "cost",
                       peak_src=alu_src)
        elif name in ("gemm_fwd", "gemm_bwd"):
            rows = E + 3 * B if name == "gemm_fwd" else B
            if name == "gemm_fwd":
                if head_struct:
                    # select forward on E rows (every layer); update: online hidden layers on
                    # [s; s'] (2B rows) + online head on s' (B) + target hidden layers on s' (B)
                    Fh = sum(2 * dims[i] * dims[i + 1] for i in range(len(dims) - 2))
                    Fo = 2 * dims[-2] * dims[-1]
                    flops = E * F + 3 * B * Fh + B * Fo
                else:
                    flops = rows * F
            else:
                # weight gradients of every GEMM layer + data gradients of all but the first;
                # with the structured head (class head_bwd) the head layer has no GEMMs
                nl = len(dims) - 1
                top = nl - 1 if head_struct else nl
                flops = sum(2 * B * dims[i] * dims[i + 1] * (2 if i > 0 else 1)
                            for i in range(top))
            ach = flops * steps / sec / 1e12
            per.update(bound="tensor", achieved=ach, peak=fp32_tc, unit="TFLOP/s",
                       frac=ach / fp32_tc, work=f"{flops / 1e9:.4g} GFLOP/step (logical fp32)",
                       peak_src=tc_src)
        elif name == "encode":
            rows = E + 2 * B
            byts = rows * (osp.W * 17 * 4 + osp.W + 8)
            ach = byts * steps / sec / 1e9
            per.update(bound="hbm", achieved=ach, peak=hbm, unit="GB/s", frac=ach / hbm,
                       work=f"{byts / 1e6:.4g} MB/step")
        elif name == "head_bwd":
            # structured head backward: per sample the last hidden row h (hi + lo planes) read
            # twice (gather and scatter), dL/dh written split and transposed (4 planes); the
            # W_head rows and the fp64 accumulators stay in L2
            w = dims[-2]
            byts = B * w * 4 * (4 + 4)
            ach = byts * steps / sec / 1e9
            per.update(bound="hbm", achieved=ach, peak=hbm, unit="GB/s", frac=ach / hbm,
                       work=f"{byts / 1e6:.4g} MB/step")
        elif name == "sgd":
            n = sum(dims[i] * dims[i + 1] + dims[i + 1] for i in range(len(dims) - 1))
            byts = n * (12 + 8 + 8)   # SGD r/w + hi/lo re-split of W and W^T
            ach = byts * steps / sec / 1e9
            per.update(bound="hbm", achieved=ach, peak=hbm, unit="GB/s", frac=ach / hbm,
                       work=f"{byts / 1e6:.4g} MB/step")
        out[name] = per
    return out


def measured_traffic(cls, cfgk=2):
    """DRAM bytes per launch of kernel class `cls` from the committed ncu launch list of this
    bench command (profiles/traffic.json for config 2 and the brute force of config 3,
    profiles/traffic_cfg<k>.json otherwise; written by tools/traffic_from_launches.py), or
    None when no launch list of that configuration is committed."""
    fn = "traffic.json" if cfgk in (2, 3) else f"traffic_cfg{cfgk}.json"
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", fn)))
        return t["classes"][cls]["dram_bytes_per_launch"], t["source"]
    except Exception:
        return None, None


def dominant(rl, cfgk=2):
    name = max(rl, key=lambda k: rl[k]["ms_per_step"])
    r = rl[name]
    traffic, src = measured_traffic(name, cfgk)
    return {"kernel": name, "bound": r.get("bound"), "achieved": r.get("achieved"),
            "peak": r.get("peak"), "unit": r.get("unit"), "frac": r.get("frac"),
            "traffic": traffic, "traffic_src": src, "peak_src": r.get("peak_src"),
            "share_of_step": None}


# ------------------------------------------------------------------------------------------
# Supplementary lines (not the driver's headline): BASELINE config 3 (exhaustive brute-force
# optimum, a14) and config 5 (inference-only Q scoring, a2-a5 in SEL_INFER mode).

def _timed_calls(fn, steps, warmup, stream, flush):
    import torch
    for _ in range(warmup):
        fn()
    stream.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    for e0, e1 in ev:
        flush.zero_()
        e0.record(stream)
        fn()
        e1.record(stream)
    stream.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev)


def run_brute(args, cfg):
    """Config 3: hrp_bruteforce_optimum over Q1-Q12 (Table V) + 4096 random windows per call."""
    import torch
    from paper_2405_08754_b200 import hrp
    from paper_2405_08754_b200.session import space_of
    rank, world, local = dist_env()
    if rank != 0:
        return
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(dev)
    pool = synth.make_pool(cfg.pool)
    sc = cfg.space
    wins = np.concatenate([synth.table_v_windows(pool),
                           synth.make_windows(pool, cfg.n_windows, sc.window, step=1)])
    n, W = wins.shape
    space, prof = space_of(sc), hrp.make_profiles(pool)
    tab = hrp.hrp_layout_table(space)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    with torch.cuda.stream(stream):
        w = torch.from_numpy(wins).to(dev)
        best = torch.empty(n, dtype=torch.int64, device=dev)
        solo = torch.empty(n, dtype=torch.int64, device=dev)
        rgs = torch.empty((n, W), dtype=torch.uint8, device=dev)
        bact = torch.empty((n, W), dtype=torch.int64, device=dev)

        # the resident plan: tables uploaded once, each call only enqueues the search kernel
        plan = hrp.hrp_brute_create(space, prof, local, stream.cuda_stream)

        def call():
            hrp.hrp_brute_run(plan, n, w, best, solo, rgs, bact, stream.cuda_stream)
        clocks = Clocks(local)
        ms = _timed_calls(call, args.steps, args.warmup, stream, flush)
        clk = clocks.stop()
        # e2e: windows from pinned host memory in, results out, inside the timed region
        wh = torch.from_numpy(wins).pin_memory()
        oh = [torch.empty(n, dtype=torch.int64).pin_memory(),
              torch.empty((n, W), dtype=torch.uint8).pin_memory()]

        def call_e2e():
            w.copy_(wh, non_blocking=True)
            call()
            oh[0].copy_(best, non_blocking=True)
            oh[1].copy_(rgs, non_blocking=True)
        ms_e2e = _timed_calls(call_e2e, args.steps, 1, stream, flush)
        stream.synchronize()
        hrp.hrp_brute_destroy(plan)
    # algorithmic work: (job set, layout, slot permutation) evaluations of phase 1
    from math import comb, factorial
    nc = np.bincount(np.asarray(tab["nslots"]), minlength=5)
    evals = sum(comb(W, c) * int(nc[c]) * factorial(c) for c in range(1, 5))
    # per evaluation: CoRun = max over 2C terms (C compute terms, C memory terms), one lane-op
    # each (the (CoRun, idx) minimum update folds into the last one)
    slot_terms = sum(comb(W, c) * int(nc[c]) * factorial(c) * 2 * c for c in range(1, 5))
    sec = ms / 1e3
    value = n * args.steps / sec
    alu_peak, alu_src = alu_peak_tops("int")
    ach = slot_terms * n * args.steps / sec / 1e12
    res = {"metric": "brute-force optimum windows/s (BASELINE config 3)", "value": value,
           "unit": "windows/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "i64", "data": "synthetic",
           "config": {"workload": f"cfg3: W={W}, Cmax={sc.cmax}, MIG GI/CI x MPS "
                                  f"{{{min(sc.shares)}..{max(sc.shares)}}}%, Q1-Q12 (Table V) + "
                                  f"{cfg.n_windows} random windows per call",
                      "windows_per_call": n, "evals_per_window": evals,
                      "l2": "flushed (256 MiB memset) between timed calls"},
           "gpu_launches": 1,
           "e2e": {"value": n * args.steps / (ms_e2e / 1e3), "unit": "windows/s",
                   "h2d_bytes_per_step": int(wins.nbytes),
                   "d2h_bytes_per_step": int(n * 8 + n * W)},
           "clocks": clk,
           "roofline": {"kernel": "brute_kernel", "bound": "alu", "achieved": ach,
                        "peak": alu_peak, "unit": "Tops/s", "frac": ach / alu_peak,
                        "traffic": measured_traffic("brute")[0],
                        "work": f"{slot_terms} CoRun terms per window (2C per (set, layout, "
                                f"sigma) evaluation, one lane-op each; {evals} evaluations)",
                        "peak_src": alu_src}}
    if not args.no_cpu_baseline:
        from oracle import brute as BR
        from oracle import space as SP
        osp = SP.build_space(sc.window, sc.cmax, sc.shares, sc.mig)
        t0 = time.perf_counter()
        k = 0
        while time.perf_counter() - t0 < args.cpu_seconds:
            BR.dp_opt(osp, [int(x) for x in wins[k % n]], pool)
            k += 1
        dt = time.perf_counter() - t0
        res["cpu_baseline"] = {"value": k / dt, "unit": "windows/s", "cores": 1,
                               "kind": "oracle",
                               "sample": f"{k} windows through oracle.brute.dp_opt, 1 thread, "
                                         f"{dt:.1f} s"}
    print(json.dumps(res), flush=True)


def run_infer(args, cfg):
    """Config 5: inference-only Q scoring (hrp_q_forward) of cfg.n_states job-mix states per
    call; states sharded across ranks (replicas only, no collective)."""
    import torch
    import torch.distributed as dist
    from paper_2405_08754_b200 import hrp, parallel
    from paper_2405_08754_b200.session import Session
    rank, world, local = dist_env()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(dev)
    pool = synth.make_pool(cfg.pool)
    n = cfg.n_states // world
    chunk = 65536
    base = synth.config(2)
    ecfg = base.with_(n_envs=chunk, batch=chunk)
    from paper_2405_08754_b200.session import space_of
    sc = cfg.space
    osp = TableInfo(sc, hrp.hrp_layout_table(space_of(sc)))    # sizes from libhrp's tables
    th = synth.init_weights(osp.dims(cfg.net))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    with torch.cuda.stream(stream):
        # explicit enumeration: every valid action of every state is scored (the Q-evals metric)
        sess = Session(ecfg, pool, init_weights=th, device=local, stream=stream, replay=chunk,
                       argmax_mode=1)
        wins = synth.make_windows(pool, n, sc.window, step=5, rank=rank)
        sched = synth.sched_states(n, sc.window, rank=rank)
        wd = torch.from_numpy(wins).to(dev)
        sd = torch.from_numpy(sched.view(np.int64)).to(dev)
        am = torch.empty(n, dtype=torch.int64, device=dev)
        qm = torch.empty(n, dtype=torch.float32, device=dev)

        def call():
            hrp.hrp_q_forward(sess.ctx, n, wd, sd, am, qm, None)
        e0 = hrp.hrp_eval_counts(sess.ctx)
        c0 = hrp.hrp_covered_counts(sess.ctx)
        l0 = sess.launches()
        clocks = Clocks(local)
        ms = _timed_calls(call, args.steps, args.warmup, stream, flush)
        clk = clocks.stop()
        e1 = hrp.hrp_eval_counts(sess.ctx)
        c1 = hrp.hrp_covered_counts(sess.ctx)
        launches = (sess.launches() - l0) / (args.steps + args.warmup)
        scored = (e1[0] - e0[0]) / (args.steps + args.warmup)
        evals = (c1[0] - c0[0]) / (args.steps + args.warmup)     # every valid action covered
        wh = torch.from_numpy(wins).pin_memory()
        sh = torch.from_numpy(sched.view(np.int64)).pin_memory()
        ah = torch.empty(n, dtype=torch.int64).pin_memory()
        qh = torch.empty(n, dtype=torch.float32).pin_memory()

        def call_e2e():
            wd.copy_(wh, non_blocking=True)
            sd.copy_(sh, non_blocking=True)
            call()
            ah.copy_(am, non_blocking=True)
            qh.copy_(qm, non_blocking=True)
        ms_e2e = _timed_calls(call_e2e, args.steps, 1, stream, flush)
        sess.close()
    ms = parallel.max_over_ranks(ms, dev) if world > 1 else ms
    ms_e2e = parallel.max_over_ranks(ms_e2e, dev) if world > 1 else ms_e2e
    if rank == 0:
        sec = ms / 1e3
        res = {"metric": "Q-evals/s (inference-only Q scoring, BASELINE config 5)",
               "value": evals * world * args.steps / sec, "unit": "Q-evals/s",
               "states_per_s": n * world * args.steps / sec,
               "candidates_scored_per_s": scored * world * args.steps / sec,
               "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "f32+i64", "data": "synthetic",
               "config": {"workload": f"cfg5: {cfg.n_states} job-mix states x full action space "
                                      f"(W={sc.window}, Cmax={sc.cmax}, Q-MLP "
                                      f"{cfg.net.hidden_layers}x{cfg.net.hidden_width}), "
                                      f"{chunk}-row chunks", "states_per_call": n * world,
                          "argmax": "explicit (every valid action scored)",
                          "parallelism": f"replicas x{world} (states sharded, no collective)",
                          "l2": "flushed (256 MiB memset) between timed calls"},
               "gpu_launches": int(round(launches * args.steps)),
               "e2e": {"value": evals * world * args.steps / (ms_e2e / 1e3), "unit": "Q-evals/s",
                       "h2d_bytes_per_step": int(wins.nbytes + sched.nbytes),
                       "d2h_bytes_per_step": int(n * 12)},
               "clocks": clk}
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--argmax", type=int, default=0, help="0 auto, 1 explicit, 2 pruned")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch the timed steps eagerly instead of from per-step CUDA graphs")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--comm1", action="store_true",
                    help="world 1 with a one-rank NCCL communicator: times the per-layer "
                         "allreduce path (inside the per-step graphs) on one GPU")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="weak: E per GPU fixed (default, configs 1-2); strong: the config's "
                         "global E and B sharded over the GPUs (default for config 4)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.scaling is None:
        args.scaling = "strong" if args.config == 4 else "weak"
    cfg = synth.config(args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
    elif cfg.n_windows:
        run_brute(args, cfg)
    elif cfg.n_states:
        run_infer(args, cfg)
    else:
        run_gpu(args, cfg)


if __name__ == "__main__":
    main()
