"""compute-sanitizer target: config 1 (W=4, Cmax=2, 2x64) at E=B=16 for 3 env steps + DQN
updates, one inference call and one brute-force call, every libhrp kernel class launched.
usage: compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_cfg1.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2405_08754_b200.session import Session, bruteforce, streams_to_dev  # noqa: E402


def main():
    cfg = synth.config(1)
    pool = synth.make_pool(27)
    E = 16
    for mode in (1, 2):
        sess = Session(cfg, pool, n_envs=E, batch=E, replay=256, argmax_mode=mode)
        sess.reset(synth.make_windows(pool, E, 4))
        for t in range(3):
            d = streams_to_dev(synth.step_streams(t, E, E, 4, pool), sess.dev)
            sess.step(synth.eps_threshold(t + 20, cfg.n_decay), d["u_explore"], d["u_action"],
                      d["next_windows"])
            sess.update(d["u_replay"], t == 1)
        w = torch.from_numpy(synth.make_windows(pool, 8, 4)).to(sess.dev)
        s = torch.from_numpy(synth.sched_states(8, 4).view(np.int64)).to(sess.dev)
        sess.q_forward(w, s, head=True)
        sess.sync()
        sess.close()
    bruteforce(synth.SpaceCfg(6, 3, (25, 50, 75)), pool, synth.make_windows(pool, 4, 6))
    torch.cuda.synchronize()
    print("sanitize target done")


if __name__ == "__main__":
    main()
