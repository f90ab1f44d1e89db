"""GPU parity of the sequential agent (reading R28): flat duelling head
[v, a_l] over the partition setups (P:259's "A = 29" outputs), job sets taken in queue order --
hand-computed greedy choices through libhrp and lockstep runs against the oracle."""
import numpy as np
import pytest
import torch

import synth
from oracle import space as SP
from dqn_harness import run_lockstep

pytestmark = pytest.mark.gpu


def test_sequential_hand_case_through_libhrp():
    # tests/test_oracle_dqn.py::test_sequential_agent_hand_case_and_queue_order: v = 0,
    # a = [1, 3] -> the greedy episode of window (J0, J1, J2) is [3, 2]
    from paper_2405_08754_b200 import hrp
    from paper_2405_08754_b200.session import Session
    cfg = synth.config(1).with_(space=synth.SpaceCfg(3, 2, (50,), mig=False),
                                net=synth.NetCfg(1, 4))
    pool = synth.make_pool(27)
    sp = SP.build_space(3, 2, (50,), False, seq=True)
    fin, w, H = 3 * 17, 4, sp.H
    th = np.concatenate([np.zeros(w * fin), np.ones(w), np.zeros(H * w), [0.0, 1.0, 3.0]])
    sess = Session(cfg, pool, n_envs=1, batch=1, init_weights=th.astype(np.float32), replay=64,
                   agent="sequential")
    assert sess.H == 3
    d = sess.dev
    sess.reset(np.array([[4, 11, 20]], np.uint8))
    z32 = torch.zeros(1, dtype=torch.int32, device=d)
    z64 = torch.zeros(1, dtype=torch.int64, device=d)
    nxt = torch.zeros((1, 3), dtype=torch.uint8, device=d)
    acts = []
    for _ in range(2):
        sess.step(0, z32, z64, nxt)
        sess.sync()
        acts.append(int(sess.actions.item()))
    assert acts == [3, 2] and int(sess.done.item()) == 1
    sess.close()


@pytest.mark.parametrize("cfgk,E,steps,resync", [(1, 64, 30, False), (2, 64, 10, True)])
def test_sequential_lockstep(cfgk, E, steps, resync):
    st = run_lockstep(cfgk, E, E, steps, resync=resync, variant={"agent": "sequential"},
                      name=f"seq_cfg{cfgk}_E{E}")
    print(st)


def test_sequential_cfg3_space_lockstep():
    # config 3's space (W = 12, Cmax = 4: 386 setups) with the sequential agent
    st = run_lockstep(2, 64, 64, 10, W=12, cmax=4, resync=True,
                      variant={"agent": "sequential"}, name="seq_W12_C4")
    print(st)
