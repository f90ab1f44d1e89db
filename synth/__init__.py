"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no layouts, action indexing, co-run
model, Q-network or search).  It only produces the *inputs* the paper's method consumes:

* the job-profile pool ("Job Profiles Repository") -- a synthetic stand-in
  for the Nsight-Compute profiles of the Table IV programs (Table III
  counters PAPER.md:199-205), recipe in SURVEY.md §8(d) / DESIGN.md "Input recipe";
* job windows Q = {J_1..J_W} (Table V job mixes PAPER.md:219-236);
* the per-step random streams of the DQN step (u_explore, u_action, u_replay, next windows;
  epsilon schedule of PAPER.md:242) and the initial Q-network weights;
* the five workload presets named by BASELINE.json "configs".

All random numbers come from numpy's counter-based Philox generator, seeded with
240508754 + stream offset {0 profiles, 1 windows, 2 epsilon/explore, 3 actions, 4 replay,
5 init}.
"""
from .pool import (TABLE_IV, TABLE_V, UNSEEN, Pool, make_pool, class_counts)
from .streams import (SEED, philox, make_windows, table_v_windows, step_streams,
                      eps_threshold, init_weights, sched_states)
from .configs import CONFIGS, SpaceCfg, NetCfg, config, MIG_ONLY_LAYOUTS, BASELINE_SPACES

__all__ = ["TABLE_IV", "TABLE_V", "UNSEEN", "Pool", "make_pool", "class_counts", "SEED",
           "philox", "make_windows", "table_v_windows", "step_streams", "eps_threshold",
           "init_weights", "sched_states", "CONFIGS", "SpaceCfg", "NetCfg", "config",
           "MIG_ONLY_LAYOUTS", "BASELINE_SPACES"]
