"""GPU parity across the W / Cmax grid of the scaling study (Fig. 9-10,
P:281-289): the exhaustive optimum bit-exact against the oracle's subset DP at every grid point
of tools/wcmax_study.py, and the DQN step at windows beyond config 2 (W = 32 and 64)."""
import numpy as np
import pytest

import synth
from oracle import brute as BR
from oracle import space as SP
from dqn_harness import run_lockstep

pytestmark = pytest.mark.gpu
S10 = tuple(range(10, 100, 10))


@pytest.mark.parametrize("W,cmax", [(4, 4), (6, 4), (8, 4), (10, 4), (12, 1), (12, 2), (12, 3)])
def test_brute_force_grid(W, cmax):
    from paper_2405_08754_b200.session import bruteforce
    pool = synth.make_pool(27)
    scfg = synth.SpaceCfg(W, cmax, S10)
    sp = SP.build_space(W, cmax, S10)
    wins = np.concatenate([synth.table_v_windows(pool)[:3, :W],
                           synth.make_windows(pool, 3, W, step=100 + W + cmax)])
    best, solo, rgs, bact = bruteforce(scfg, pool, wins)
    for i, w in enumerate(wins):
        ref = BR.dp_opt(sp, [int(x) for x in w], pool)
        assert best[i] == ref["cost"] and solo[i] == ref["solo"]
        assert list(rgs[i]) == ref["rgs"] and list(bact[i]) == ref["block_action"]


@pytest.mark.parametrize("W,cmax", [(32, 3), (64, 2)])
def test_dqn_step_large_windows(W, cmax):
    st = run_lockstep(2, 32, 32, 5, W=W, cmax=cmax, name=f"wcmax_W{W}_C{cmax}")
    print(st)
