"""World-size-2 tests of the data-parallel path on CPU (gloo backend).

The GPU path shards environments across ranks and allreduces the Q-network gradient inside
hrp_dqn_update (NCCL), scaling the head gradient by 1 / (B * world).
Here two gloo ranks run the oracle on their env shards with the same per-rank streams the
bench uses, allreduce the sum-form gradients, apply SGD, and must (a) stay bit-identical to
each other and (b) equal a single-process simulation of both shards.  The host helpers of
paper_2405_08754_b200/parallel.py (id broadcast, max over ranks) are exercised on gloo too."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import env as EV
from oracle import qnet as QN
from oracle import space as SP

E_LOCAL, STEPS, WORLD = 6, 4, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _make(rank, cfg, pool, osp, th):
    from paper_2405_08754_b200.parallel import env_shard
    orc = EV.OracleDQN(osp, pool, cfg.net, th, E_LOCAL, E_LOCAL, 256, gamma=cfg.gamma,
                       lr=cfg.lr)
    orc.reset(synth.make_windows(pool, E_LOCAL, osp.W, rank=rank,
                                 first_env=env_shard(E_LOCAL, rank)))
    return orc


def _step(orc, rank, t, cfg, pool, osp):
    from paper_2405_08754_b200.parallel import env_shard
    st = synth.step_streams(t, E_LOCAL, E_LOCAL, osp.W, pool, rank=rank,
                            first_env=env_shard(E_LOCAL, rank))
    orc.env_step(synth.eps_threshold(t, cfg.n_decay), st["u_explore"], st["u_action"],
                 st["next_windows"])
    return orc.dqn_update(st["u_replay"], False, b_total=E_LOCAL * WORLD, apply=False)


def _setup():
    cfg = synth.config(1)
    pool = synth.make_pool(27)
    osp = SP.build_space(cfg.space.window, cfg.space.cmax, cfg.space.shares)
    th = synth.init_weights(QN.net_dims(osp, cfg.net))
    return cfg, pool, osp, th


def _worker(rank, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_2405_08754_b200.parallel import broadcast_bytes, max_over_ranks
    tok = broadcast_bytes(bytes(range(128)) if rank == 0 else None, 128)
    assert tok == bytes(range(128))
    assert max_over_ranks(float(rank) + 0.5) == WORLD - 0.5
    cfg, pool, osp, th = _setup()
    orc = _make(rank, cfg, pool, osp, th)
    for t in range(STEPS):
        out = _step(orc, rank, t, cfg, pool, osp)
        g = torch.from_numpy(out["grad"].copy())
        dist.all_reduce(g)                       # the hot path's one exchange (NCCL on GPU)
        orc.apply(g.numpy(), (t + 1) % cfg.target_sync == 0)
    np.save(os.path.join(out_dir, f"theta{rank}.npy"), orc.theta)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_dqn_matches_single_process(tmp_path):
    mp.start_processes(_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True,
                       start_method="spawn")
    th0 = np.load(tmp_path / "theta0.npy")
    th1 = np.load(tmp_path / "theta1.npy")
    assert np.array_equal(th0, th1), "replicas diverged"
    # single-process simulation of the two shards
    cfg, pool, osp, th = _setup()
    orcs = [_make(r, cfg, pool, osp, th) for r in range(WORLD)]
    for t in range(STEPS):
        gs = [_step(o, r, t, cfg, pool, osp)["grad"] for r, o in enumerate(orcs)]
        g = gs[0] + gs[1]
        for o in orcs:
            o.apply(g, (t + 1) % cfg.target_sync == 0)
    assert np.allclose(th0, orcs[0].theta, rtol=0, atol=1e-12)
    assert not np.allclose(th0, th), "weights did not move"


def test_env_shards_are_disjoint_streams():
    from paper_2405_08754_b200.parallel import env_shard
    pool = synth.make_pool(27)
    w0 = synth.make_windows(pool, 64, 16, rank=0, first_env=env_shard(64, 0))
    w1 = synth.make_windows(pool, 64, 16, rank=1, first_env=env_shard(64, 1))
    assert not np.array_equal(w0, w1)
    s0 = synth.step_streams(3, 64, 64, 16, pool, rank=0)
    s1 = synth.step_streams(3, 64, 64, 16, pool, rank=1)
    assert not np.array_equal(s0["u_replay"], s1["u_replay"])
