"""Convenience wrapper over the C ABI for tests / bench / smoke: owns a libhrp context and the
torch CUDA output tensors of each call.  Marshalling only -- every computation runs in libhrp.
"""
from __future__ import annotations

import numpy as np
import torch

from . import hrp


def space_of(scfg, layouts=None):
    return hrp.make_space(scfg.window, scfg.cmax, scfg.shares, scfg.mig, scfg.interference_q3,
                          layouts)


class Session:
    def __init__(self, cfg, pool, n_envs=None, batch=None, init_weights=None, device=0,
                 rank=0, world=1, nccl_id=None, argmax_mode=0, replay=None,
                 reward_lambda=None, stream=None, optimizer="sgd", adam=(0.9, 0.999, 1e-8),
                 loss="squared", huber_kappa=1.0, precision="3xtf32", agent="joint"):
        if not torch.cuda.is_available():
            raise RuntimeError("libhrp needs a CUDA device (no CPU fallback)")
        self.cfg = cfg
        self.dev = torch.device("cuda", device)
        self.stream = stream or torch.cuda.current_stream(self.dev)
        self.E = n_envs or cfg.n_envs
        self.B = batch or cfg.batch
        self.W = cfg.space.window
        self.space = space_of(cfg.space)
        self.prof = hrp.make_profiles(pool)
        lam = cfg.space.reward_lambda if reward_lambda is None else reward_lambda
        self.tcfg = hrp.make_cfg(self.E, self.B, replay or max(1 << 16, 16 * self.E),
                                 cfg.net.hidden_layers, cfg.net.hidden_width, cfg.gamma, cfg.lr,
                                 lam, argmax_mode, optimizer, adam, loss, huber_kappa,
                                 precision, agent)
        self.ctx = hrp.hrp_env_create(self.space, self.prof, self.tcfg, device,
                                      self.stream.cuda_stream, rank, world, nccl_id,
                                      init_weights)
        self.n_params = hrp.hrp_n_params(self.ctx)
        self.H = hrp.hrp_head_width(self.ctx)
        d = self.dev
        E, B = self.E, self.B
        self.actions = torch.empty(E, dtype=torch.int64, device=d)
        self.rewards = torch.empty(E, dtype=torch.float32, device=d)
        self.done = torch.empty(E, dtype=torch.uint8, device=d)
        self.corun = torch.empty(E, dtype=torch.int64, device=d)
        self.qsel = torch.empty(E, dtype=torch.float32, device=d)
        self.greedy = torch.empty(E, dtype=torch.int64, device=d)
        self.loss = torch.empty(1, dtype=torch.float32, device=d)
        self.sidx = torch.empty(B, dtype=torch.int64, device=d)
        self.astar = torch.empty(B, dtype=torch.int64, device=d)

    def close(self):
        if self.ctx:
            hrp.hrp_env_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def to_dev(self, a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(self.dev, non_blocking=False)

    def reset(self, windows):
        self.windows0 = self.to_dev(np.asarray(windows, np.uint8))
        hrp.hrp_env_reset(self.ctx, self.windows0)

    def step(self, thr, u_explore, u_action, next_windows, extras=True):
        hrp.hrp_env_step(self.ctx, thr, u_explore, u_action, next_windows, self.actions,
                         self.rewards, self.done, self.corun if extras else None,
                         self.qsel if extras else None, self.greedy if extras else None)

    def update(self, u_replay, sync_target, extras=True):
        hrp.hrp_dqn_update(self.ctx, u_replay, sync_target, self.loss,
                           self.sidx if extras else None, self.astar if extras else None)

    def grad(self, u_replay, d_grad, extras=True):
        """hrp_dqn_grad: this rank's gradient into d_grad (no allreduce, weights unchanged)."""
        hrp.hrp_dqn_grad(self.ctx, u_replay, self.loss, d_grad,
                         self.sidx if extras else None, self.astar if extras else None)

    def apply_grad(self, d_grad, sync_target):
        hrp.hrp_apply_grad(self.ctx, d_grad, sync_target)

    def q_forward(self, windows, sched, head=False):
        n = windows.shape[0]
        am = torch.empty(n, dtype=torch.int64, device=self.dev)
        qm = torch.empty(n, dtype=torch.float32, device=self.dev)
        hd = torch.empty((n, self.H), dtype=torch.float32, device=self.dev) if head else None
        hrp.hrp_q_forward(self.ctx, n, windows, sched, am, qm, hd)
        return am, qm, hd

    def relu_masks(self, rows=None):
        """The backward's ReLU' decisions of the last update's s rows, per hidden layer (bool
        numpy [rows][w]); test hook for reading R25."""
        rows = self.B if rows is None else rows
        out = []
        for l in range(self.cfg.net.hidden_layers):
            t = torch.empty((rows, self.cfg.net.hidden_width), dtype=torch.float32,
                            device=self.dev)
            hrp.hrp_get_hidden(self.ctx, l, rows, t)
            torch.cuda.synchronize(self.dev)
            out.append((t > 0).cpu().numpy())
        return out

    def weights(self):
        return hrp.hrp_get_weights(self.ctx)

    def sync(self):
        hrp.hrp_sync(self.ctx)

    def launches(self):
        return hrp.hrp_launch_count(self.ctx)


def streams_to_dev(st, dev):
    return {
        "u_explore": torch.from_numpy(st["u_explore"].astype(np.uint32).view(np.int32)).to(dev),
        "u_action": torch.from_numpy(st["u_action"].astype(np.uint64).view(np.int64)).to(dev),
        "u_replay": torch.from_numpy(st["u_replay"].astype(np.uint32).view(np.int32)).to(dev),
        "next_windows": torch.from_numpy(np.ascontiguousarray(st["next_windows"])).to(dev),
    }


def bruteforce(scfg, pool, windows, device=0, stream=None, layouts=None):
    """hrp_bruteforce_optimum on a uint8 [n][W] numpy array; returns numpy outputs.
    layouts: optional explicit layout table [[(sm800, b8, dom), ...], ...] (restricted
    baselines)."""
    dev = torch.device("cuda", device)
    st = stream or torch.cuda.current_stream(dev)
    w = torch.from_numpy(np.ascontiguousarray(windows, np.uint8)).to(dev)
    n, W = w.shape
    best = torch.empty(n, dtype=torch.int64, device=dev)
    solo = torch.empty(n, dtype=torch.int64, device=dev)
    rgs = torch.empty((n, W), dtype=torch.uint8, device=dev)
    bact = torch.empty((n, W), dtype=torch.int64, device=dev)
    hrp.hrp_bruteforce_optimum(space_of(scfg, layouts), hrp.make_profiles(pool), n, w, best, solo, rgs,
                               bact, st.cuda_stream)
    torch.cuda.synchronize(dev)
    return best.cpu().numpy(), solo.cpu().numpy(), rgs.cpu().numpy(), bact.cpu().numpy()
