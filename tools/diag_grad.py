"""Diagnostic (GPU): per-layer gradient error of one DQN update -- libhrp (hrp_dqn_grad) vs the
fp64 oracle, next to a plain fp32 CPU recomputation of the same gradient (torch autograd in
float32 on the oracle's inputs) -- to separate kernel error from fp32's own limit.
usage: python tools/diag_grad.py CFG E [steps]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth  # noqa: E402
from oracle import env as EV, qnet as QN  # noqa: E402
from dqn_harness import make_pair  # noqa: E402


def fp32_grad(theta, dims, X, dz):
    ws = QN.unflatten(np.asarray(theta, np.float64), dims)
    h = torch.tensor(X, dtype=torch.float32)
    params = []
    for i, (Wm, b) in enumerate(ws):
        Wt = torch.tensor(Wm, dtype=torch.float32, requires_grad=True)
        bt = torch.tensor(b, dtype=torch.float32, requires_grad=True)
        params += [Wt, bt]
        h = h @ Wt.T + bt
        if i < len(ws) - 1:
            h = torch.relu(h)
    (h * torch.tensor(dz, dtype=torch.float32)).sum().backward()
    return np.concatenate([p.grad.numpy().ravel().astype(np.float64) for p in params])


def layer_errs(g, ref, dims):
    out, o = [], 0
    for i in range(len(dims) - 1):
        n = dims[i] * dims[i + 1] + dims[i + 1]
        a, r = g[o:o + n], ref[o:o + n]
        out.append(float(np.linalg.norm(a - r) / max(np.linalg.norm(r), 1e-30)))
        o += n
    return out


def main():
    cfgk, E = int(sys.argv[1]), int(sys.argv[2])
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    from paper_2405_08754_b200.session import streams_to_dev
    cfg, pool, osp, sess, orc = make_pair(cfgk, E, E)
    dims = QN.net_dims(osp, cfg.net)
    W = osp.W
    win0 = synth.make_windows(pool, E, W)
    sess.reset(win0)
    orc.reset(win0)
    n = sess.n_params
    g = torch.empty(n, dtype=torch.float32, device=sess.dev)
    rows = []
    for t in range(steps):
        st = synth.step_streams(t, E, E, W, pool)
        d = streams_to_dev(st, sess.dev)
        thr = synth.eps_threshold(t, cfg.n_decay)
        sess.step(thr, d["u_explore"], d["u_action"], d["next_windows"])
        sess.sync()
        orc.env_step(thr, st["u_explore"], st["u_action"], st["next_windows"],
                     gpu_actions=sess.greedy.cpu().numpy())
        sess.grad(d["u_replay"], g)
        sess.sync()
        # oracle gradient on the same weights (the GPU's, in fp64)
        w = sess.weights()
        orc.theta = w[:n].astype(np.float64)
        orc.theta_t = w[n:].astype(np.float64)
        out = orc.dqn_update(st["u_replay"], False, gpu_astar=sess.astar.cpu().numpy(), apply=False,
                             gpu_masks=sess.relu_masks())
        row_adopt = orc.relu_near
        # fp32 CPU recomputation of sum(dz * z) on the oracle's inputs
        idx = out["idx"]
        X = np.stack([EV.encode(orc.rep_win[i], int(orc.rep_sched[i]), pool, W) for i in idx])
        B = len(idx)
        dz = np.stack([QN.dq_dz(osp, *EV.A.decode(osp, int(orc.rep_act[i]), orc.off)) *
                       (out["q_sa"][b] - out["y"][b]) / B for b, i in enumerate(idx)])
        g32 = fp32_grad(orc.theta, dims, X, dz)
        gg = g.cpu().numpy().astype(np.float64)
        row = {"t": t, "relu_adopted_total": row_adopt, "loss_gpu": sess.loss.item(), "loss_orc": out["loss"],
               "gpu_vs_fp64": layer_errs(gg, out["grad"], dims),
               "fp32cpu_vs_fp64": layer_errs(g32, out["grad"], dims)}
        print(json.dumps(row), flush=True)
        rows.append(row)
        sess.apply_grad(g, False)
        orc.apply(out["grad"], False)
    orc.close()
    sess.close()


if __name__ == "__main__":
    main()
