"""The five workload presets of BASELINE.json "configs" (sizes per SURVEY.md §8(a)).

These are parameters, not arithmetic: window W, Cmax, MPS share set S (PAPER.md:66,
Table VII), MIG on/off, the Q-MLP shape, env count E, batch B, pool size.
Hyper-parameters the paper leaves open follow reading R12.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace


@dataclass(frozen=True)
class SpaceCfg:
    window: int                 # W
    cmax: int                   # Cmax
    shares: tuple               # MPS shares allowed inside a CI, in percent
    mig: bool = True            # False = MIG-off (MPS-only) layouts only
    interference_q3: int = 1    # extra-co-runner memory penalty, in 1/8 units
    reward_lambda: float = 0.0  # weight of the intermediate reward r_i (Table VI)


@dataclass(frozen=True)
class NetCfg:
    hidden_layers: int
    hidden_width: int


@dataclass(frozen=True)
class Config:
    name: str
    space: SpaceCfg
    net: NetCfg = None
    n_envs: int = 0
    batch: int = 0
    pool: int = 27
    gamma: float = 0.99
    lr: float = 1e-3
    target_sync: int = 25
    n_decay: int = 50
    steps: int = 100
    n_states: int = 0           # inference-only config
    n_windows: int = 0          # brute-force config: random windows beside Q1-Q12
    extra: dict = field(default_factory=dict)

    @property
    def replay_capacity(self) -> int:
        return max(1 << 16, 16 * self.n_envs)

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


S10 = tuple(range(10, 100, 10))
CONFIGS = {
    1: Config("cfg1", SpaceCfg(4, 2, (25, 50, 75)), NetCfg(2, 64), n_envs=64, batch=64,
              steps=100, n_decay=50),
    2: Config("cfg2", SpaceCfg(16, 3, S10), NetCfg(3, 256), n_envs=4096, batch=4096,
              steps=100, n_decay=50),
    3: Config("cfg3", SpaceCfg(12, 4, S10), n_windows=4096),
    4: Config("cfg4", SpaceCfg(64, 4, S10), NetCfg(4, 512), n_envs=65536, batch=65536,
              pool=256, steps=20, n_decay=50),
    5: Config("cfg5", SpaceCfg(16, 3, S10), NetCfg(3, 256), n_states=1 << 20),
}


# The paper's compared methods as search spaces for the exhaustive optimum at
# config 3's window (W = 12, Cmax = 4).  "MIG Only (C = 2)" explores the two options
# of Fig. 2: [{0.375}+{0.5},1m] (one 7-slice GI, CIs of 4 and 3 GPCs sharing its 8
# memory eighths) and [{0.375},0.5m]+[{0.5},0.5m] (GIs of 4 and 3 GPCs, 4 memory eighths and
# a memory domain each), plus the whole GPU for a job left alone (= time sharing).
# Slots are (sm800, b8, domain) in R6's units; this is an input table, not arithmetic.
MIG_ONLY_LAYOUTS = [[(800, 8, 0)], [(400, 8, 0), (300, 8, 0)], [(400, 4, 0), (300, 4, 1)]]
BASELINE_SPACES = {
    "mig_only": (SpaceCfg(12, 2, S10), MIG_ONLY_LAYOUTS),
    "mps_only": (SpaceCfg(12, 4, S10, mig=False), None),
    "mig_mps": (SpaceCfg(12, 4, S10), None),
}


def config(k: int) -> Config:
    return CONFIGS[k]
