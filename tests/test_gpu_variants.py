"""GPU parity of the SURVEY §8(f) row 4 variants: Adam, Huber loss and the fast (one TF32 MMA
per product) precision mode, against the fp64 oracle / the fp32-accurate path."""
import numpy as np
import pytest
import torch

import synth
from oracle import qnet as QN
from oracle import space as SP
from dqn_harness import run_lockstep

pytestmark = pytest.mark.gpu


def _hand_session(**variant):
    from test_oracle_dqn import DDQN_Z_ONLINE, DDQN_Z_TARGET, _hand_dqn_weights
    from paper_2405_08754_b200 import hrp
    from paper_2405_08754_b200.session import Session
    cfg = synth.config(1).with_(space=synth.SpaceCfg(3, 1, (50,), mig=False),
                                net=synth.NetCfg(1, 4), gamma=0.9, lr=0.01)
    pool = synth.make_pool(27)
    osp = SP.build_space(3, 1, (50,), False)
    dims, th_on, th_tg = _hand_dqn_weights(osp, cfg.net, DDQN_Z_ONLINE, DDQN_Z_TARGET)
    sess = Session(cfg, pool, n_envs=1, batch=1, init_weights=th_on.astype(np.float32),
                   replay=64, **variant)
    hrp.hrp_set_weights(sess.ctx, np.concatenate([th_on, th_tg]).astype(np.float32))
    d = sess.dev
    sess.reset(np.array([[4, 11, 20]], np.uint8))
    sess.step(1 << 32, torch.zeros(1, dtype=torch.int32, device=d),
              torch.zeros(1, dtype=torch.int64, device=d),
              torch.zeros((1, 3), dtype=torch.uint8, device=d))
    sess.update(torch.zeros(1, dtype=torch.int32, device=d), False)
    sess.sync()
    return sess, osp, th_on


def test_huber_hand_case_through_libhrp():
    # tests/test_oracle_dqn.py::test_huber_loss_hand_computed through the C ABI
    from test_oracle_dqn import DDQN_DQDZ, DDQN_Z_ONLINE
    sess, osp, _ = _hand_session(loss="huber", huber_kappa=0.25)
    assert abs(sess.loss.item() - 0.10625) <= 1e-6
    n, H = sess.n_params, osp.H
    w = sess.weights()
    np.testing.assert_allclose(w[n - H:n], np.array(DDQN_Z_ONLINE) + 0.01 * 0.25 *
                               np.array(DDQN_DQDZ), atol=1e-6)
    sess.close()


def test_adam_first_step_through_libhrp():
    # the first Adam step moves every parameter with a nonzero gradient by lr * sign(-g)
    from test_oracle_dqn import DDQN_DELTA, DDQN_DQDZ, DDQN_Z_ONLINE
    sess, osp, th_on = _hand_session(optimizer="adam", adam=(0.9, 0.999, 1e-12))
    n, H = sess.n_params, osp.H
    w = sess.weights()[:n]
    gb = DDQN_DELTA * np.array(DDQN_DQDZ)
    np.testing.assert_allclose(w[n - H:], np.array(DDQN_Z_ONLINE) - 0.01 * np.sign(gb),
                               atol=1e-6)
    sess.close()


@pytest.mark.parametrize("variant", [{"loss": "huber", "huber_kappa": 10.0},
                                     {"optimizer": "adam"},
                                     {"optimizer": "adam", "loss": "huber",
                                      "huber_kappa": 10.0}])
def test_variant_lockstep_config1(variant):
    # config 1, 30 seeded steps, same protocol as the SGD runs (bit-exact integers, 1e-4 floats)
    st = run_lockstep(1, 64, 64, 30, variant=variant, oracle_argmax="explicit",
                      name="variant_" + "_".join(f"{k}{v}" for k, v in variant.items()))
    print(st)


def test_variant_lockstep_config2_adam_huber():
    st = run_lockstep(2, 256, 256, 20, resync=True,
                      variant={"optimizer": "adam", "loss": "huber", "huber_kappa": 10.0},
                      name="variant_cfg2_adam_huber")
    print(st)


def test_fast_precision_policy_level():
    # fast mode (one TF32 MMA per product): policy-level agreement with the fp32-accurate path
    # on the same weights -- greedy actions on 4096 config 2 states and Q^max within 1e-2
    from paper_2405_08754_b200.session import Session
    cfg = synth.config(2)
    pool = synth.make_pool(27)
    osp = SP.build_space(16, 3, cfg.space.shares)
    th = synth.init_weights(QN.net_dims(osp, cfg.net))
    s3 = Session(cfg, pool, n_envs=256, batch=256, init_weights=th)
    sf = Session(cfg, pool, n_envs=256, batch=256, init_weights=th, precision="fast")
    wins = synth.make_windows(pool, 4096, 16, step=11)
    sched = synth.sched_states(4096, 16, step=11)
    dw = torch.from_numpy(wins).to(s3.dev)
    ds = torch.from_numpy(sched.view(np.int64)).to(s3.dev)
    a3, q3, _ = s3.q_forward(dw, ds)
    af, qf, _ = sf.q_forward(dw, ds)
    torch.cuda.synchronize()
    agree = (a3 == af).float().mean().item()
    qerr = ((qf - q3).abs() / q3.abs().clamp_min(1.0)).max().item()
    print({"action_agreement": agree, "qmax_rel_err": qerr})
    assert agree >= 0.99
    assert qerr <= 1e-2
    s3.close()
    sf.close()
