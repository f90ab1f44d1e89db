"""GPU parity of the schedule-quality path: per-job co-run times
(hrp_job_times) bit-exact against the oracle's co-run model, time sharing's AppSlowdown and
Fairness exactly 1, the greedy episodes of a trained policy equal to the
oracle's greedy choices on the same weights, and the optimum's metrics equal to the oracle's."""
from fractions import Fraction

import numpy as np
import pytest
import torch

import synth
from oracle import actions as A
from oracle import env as EV
from oracle import metrics as MT
from oracle import space as SP

pytestmark = pytest.mark.gpu
S10 = tuple(range(10, 100, 10))


def _plan(scfg, pool, layouts=None):
    from paper_2405_08754_b200 import hrp
    from paper_2405_08754_b200.schedule import make_plan
    from paper_2405_08754_b200.session import space_of
    return make_plan(space_of(scfg, layouts), hrp.make_profiles(pool))


def test_job_times_bit_exact():
    from paper_2405_08754_b200 import hrp
    pool = synth.make_pool(27)
    scfg = synth.SpaceCfg(12, 4, S10)
    sp = SP.build_space(12, 4, S10)
    plan = _plan(scfg, pool)
    rng = np.random.default_rng(4)
    n = 3000
    wins = synth.make_windows(pool, n, 12, step=21)
    acts = rng.integers(0, A.n_actions(sp), n)
    acts[:3] = [-1, A.n_actions(sp), 0]                 # out of range -> -1, first action
    dev = torch.device("cuda", 0)
    dw = torch.from_numpy(wins).to(dev)
    da = torch.from_numpy(acts.astype(np.int64)).to(dev)
    cr = torch.empty(n, dtype=torch.int64, device=dev)
    so = torch.empty(n, dtype=torch.int64, device=dev)
    mt = torch.empty((n, 4), dtype=torch.int64, device=dev)
    hrp.hrp_job_times(plan, n, dw, da, cr, so, mt, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    cr, so, mt = cr.cpu().numpy(), so.cpu().numpy(), mt.cpu().numpy()
    assert cr[0] == -1 and cr[1] == -1 and (mt[:2] == -1).all()
    off = A.offsets(sp)
    for r in range(2, n, 7):
        c, s, mem = MT.member_times(sp, wins[r], int(acts[r]), pool, off=off)
        assert cr[r] == c and so[r] == s
        assert list(mt[r, :len(mem)]) == [t for _, _, t in mem]
        assert (mt[r, len(mem):] == -1).all()
    hrp.hrp_brute_destroy(plan)


def test_time_sharing_slowdown_and_fairness_through_libhrp():
    from paper_2405_08754_b200.schedule import job_metrics, time_sharing_schedules
    from paper_2405_08754_b200.session import space_of
    pool = synth.make_pool(27)
    scfg = synth.SpaceCfg(12, 4, S10)
    plan = _plan(scfg, pool)
    Q = synth.table_v_windows(pool)
    res = job_metrics(plan, pool, Q, time_sharing_schedules(space_of(scfg), Q))
    for m in res:
        assert m["throughput"] == 1.0 and m["fairness"] == 1.0
        assert all(s == 1.0 for s in m["slowdown"])


def test_optimum_metrics_equal_oracle():
    from paper_2405_08754_b200.schedule import job_metrics, optimum_schedules
    pool = synth.make_pool(27)
    scfg = synth.SpaceCfg(12, 4, S10)
    sp = SP.build_space(12, 4, S10)
    plan = _plan(scfg, pool)
    Q = synth.table_v_windows(pool)
    sch, best = optimum_schedules(plan, Q)
    res = job_metrics(plan, pool, Q, sch)
    for w, acts, m in zip(Q, sch, res):
        ref = MT.queue_metrics(sp, w, acts, pool)
        assert m["corun"] == ref["corun"] and m["solo"] == ref["solo"]
        np.testing.assert_allclose(m["slowdown"], [float(x) for x in ref["slowdown"]],
                                   rtol=1e-15)
        assert m["fairness"] == pytest.approx(float(ref["fairness"]), rel=1e-15)


def test_greedy_rollout_equals_oracle_greedy():
    # a briefly trained policy (config 3's space, 2 x 64 MLP), run greedily on Q1-Q12 through
    # hrp_env_step; the oracle takes the greedy action of the same (fp32) weights at every state
    from paper_2405_08754_b200.schedule import greedy_rollout
    from paper_2405_08754_b200.session import Session, streams_to_dev
    pool = synth.make_pool(27)
    sc = synth.SpaceCfg(12, 4, S10)
    cfg = synth.config(1).with_(space=sc)
    sp = SP.build_space(12, 4, S10)
    from oracle import qnet as QN
    th = synth.init_weights(QN.net_dims(sp, cfg.net))
    tr = Session(cfg, pool, n_envs=64, batch=64, init_weights=th, replay=1024)
    tr.reset(synth.make_windows(pool, 64, 12))
    for t in range(10):
        d = streams_to_dev(synth.step_streams(t, 64, 64, 12, pool), tr.dev)
        tr.step(synth.eps_threshold(t, 5), d["u_explore"], d["u_action"], d["next_windows"])
        tr.update(d["u_replay"], False)
    w = tr.weights()[:tr.n_params]
    tr.close()
    Q = synth.table_v_windows(pool)
    ev = Session(cfg, pool, n_envs=12, batch=12, init_weights=w, replay=1024)
    sch = greedy_rollout(ev, Q)
    ev.close()
    orc = EV.OracleDQN(sp, pool, cfg.net, w.astype(np.float64), 12, 12, 1024, argmax="pruned")
    orc.reset(Q)
    ref = [[] for _ in Q]
    live = np.ones(12, bool)
    for k in range(12):
        gpu_k = [s[k] if k < len(s) else None for s in sch]
        a, r, d, cr, q = orc.env_step(0, np.zeros(12, np.uint32), np.zeros(12, np.uint64), Q,
                                      gpu_actions=gpu_k)
        for e in np.nonzero(live)[0]:
            ref[e].append(int(a[e]))
            if d[e]:
                live[e] = False
        if not live.any():
            break
    assert sch == ref
    assert orc.near_ties <= 1
    orc.close()


@pytest.mark.parametrize("pi", [0, 7, 17, 38])
def test_mig_mps_default_tables_brute_force(pi):
    # MIG+MPS Default (R27): the exhaustive optimum over one partition's default-MPS
    # table, bit-exact against the oracle's DP over the oracle's own table of that partition
    from paper_2405_08754_b200.schedule import default_mps_table, mig_partitions
    from paper_2405_08754_b200.session import bruteforce
    from oracle import brute as BR
    pool = synth.make_pool(27)
    part = mig_partitions(12, 4)[pi]
    table = default_mps_table(part, 4)
    scfg = synth.SpaceCfg(12, 4, S10)
    sp = SP.build_space(12, 4, S10, True, layouts=SP.default_mps_layouts(SP.mig_partitions(4)[pi], 4))
    Q = synth.table_v_windows(pool)[:4]
    best, solo, rgs, bact = bruteforce(scfg, pool, Q, layouts=table)
    for i, w in enumerate(Q):
        ref = BR.dp_opt(sp, [int(x) for x in w], pool)
        assert best[i] == ref["cost"] and solo[i] == ref["solo"]
        assert list(rgs[i]) == ref["rgs"] and list(bact[i]) == ref["block_action"]
