"""GPU parity: hrp_bruteforce_optimum (a14) vs the oracle's subset DP -- bit-exact.

The oracle's DP is itself pinned to the RGS enumeration and the literal search
(tests/test_oracle_pruned_brute.py)."""
import numpy as np
import pytest

import synth
from oracle import brute as BR
from oracle import space as SP
from synth.configs import SpaceCfg

pytestmark = pytest.mark.gpu
S10 = tuple(range(10, 100, 10))


def _cmp(scfg, pool, wins, layouts=None):
    from paper_2405_08754_b200.session import bruteforce
    best, solo, rgs, bact = bruteforce(scfg, pool, wins, layouts=layouts)
    L = SP.select_layouts(layouts, scfg.cmax, scfg.shares) if layouts else None
    sp = SP.build_space(scfg.window, scfg.cmax, scfg.shares, scfg.mig, layouts=L)
    for i, w in enumerate(wins):
        ref = BR.dp_opt(sp, [int(x) for x in w], pool, scfg.interference_q3)
        assert best[i] == ref["cost"], i
        assert solo[i] == ref["solo"], i
        assert list(rgs[i]) == ref["rgs"], i
        assert list(bact[i]) == ref["block_action"], i


@pytest.mark.parametrize("W,cmax,S,mig", [(3, 2, (25, 50, 75), True), (5, 3, (25, 50, 75), True),
                                          (6, 4, (50,), True), (7, 3, S10, False),
                                          (8, 2, S10, True), (1, 1, (50,), True)])
def test_small_spaces(W, cmax, S, mig):
    pool = synth.make_pool(27)
    scfg = SpaceCfg(W, cmax, S, mig)
    wins = synth.make_windows(pool, 24, W, step=W * 10 + cmax)
    _cmp(scfg, pool, wins)


def test_heavy_ties():
    from types import SimpleNamespace
    T = np.array([1000, 1000, 2000, 4000], np.int64)
    pool = SimpleNamespace(solo_ticks=T, compute_pm=np.full(4, 100, np.int16),
                           memory_pm=np.full(4, 100, np.int16),
                           features=np.zeros((4, 12), np.float32))
    rng = np.random.default_rng(9)
    wins = rng.integers(0, 4, (16, 8)).astype(np.uint8)
    _cmp(SpaceCfg(8, 4, (25, 50, 75)), pool, wins)


def test_config3_table_v_and_random():
    # config 3: W = 12, Cmax = 4, Q1-Q12 of Table V + random class-stratified windows
    pool = synth.make_pool(27)
    scfg = synth.config(3).space
    wins = np.concatenate([synth.table_v_windows(pool),
                           synth.make_windows(pool, 8, 12, step=77)])
    _cmp(scfg, pool, wins)


def test_config3_full_launch_sampled():
    # the bench's launch: Q1-Q12 + 4096 windows in one call; oracle checks a sample
    from paper_2405_08754_b200.session import bruteforce
    pool = synth.make_pool(27)
    scfg = synth.config(3).space
    wins = np.concatenate([synth.table_v_windows(pool),
                           synth.make_windows(pool, 4096, 12, step=1)])
    best, solo, rgs, bact = bruteforce(scfg, pool, wins)
    assert (best <= solo).all() and (best > 0).all()
    sp = SP.build_space(12, 4, S10)
    for i in (0, 11, 12, 1000, 2047, 4107):
        ref = BR.dp_opt(sp, [int(x) for x in wins[i]], pool)
        assert (best[i], solo[i], list(rgs[i]), list(bact[i])) == \
            (ref["cost"], ref["solo"], ref["rgs"], ref["block_action"])


@pytest.mark.parametrize("name", ["mig_only", "mps_only"])
def test_restricted_baselines_table_v(name):
    # P:245-248 compared methods (synth.BASELINE_SPACES) on Q1-Q12: MIG Only through an
    # explicit layout table (Fig. 2's two options), MPS Only through the MIG-off space
    pool = synth.make_pool(27)
    scfg, lay = synth.BASELINE_SPACES[name]
    _cmp(scfg, pool, synth.table_v_windows(pool), layouts=lay)


def test_resident_plan_equals_one_shot_and_is_graph_capturable():
    # hrp_brute_create / run / destroy: tables uploaded once, the run only enqueues the kernel
    # (captured in a CUDA graph here); results equal the one-shot call and the oracle on Q1-Q12
    import torch
    from paper_2405_08754_b200 import hrp
    from paper_2405_08754_b200.session import bruteforce, space_of
    pool = synth.make_pool(27)
    scfg = SpaceCfg(12, 4, S10)
    wins = np.concatenate([synth.table_v_windows(pool), synth.make_windows(pool, 20, 12, step=7)])
    n = len(wins)
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    plan = hrp.hrp_brute_create(space_of(scfg), hrp.make_profiles(pool), 0, st.cuda_stream)
    with torch.cuda.stream(st):
        w = torch.from_numpy(wins).to(dev)
        outs = [torch.full((n,), -7, dtype=torch.int64, device=dev),
                torch.full((n,), -7, dtype=torch.int64, device=dev),
                torch.zeros((n, 12), dtype=torch.uint8, device=dev),
                torch.zeros((n, 12), dtype=torch.int64, device=dev)]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            hrp.hrp_brute_run(plan, n, w, *outs, st.cuda_stream)
        g.replay()
    st.synchronize()
    hrp.hrp_brute_destroy(plan)
    ref = bruteforce(scfg, pool, wins)
    for a, b in zip(outs, ref):
        np.testing.assert_array_equal(a.cpu().numpy(), b)
    _cmp(scfg, pool, wins[:12])
