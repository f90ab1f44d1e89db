"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, float64 / Python-int implementation of the hot path of arXiv 2405.08754
("Hierarchical Resource Partitioning on Modern GPUs: A Reinforcement Learning Approach"),
written from /root/reference/PAPER.md (cited as P:<line>) and the readings listed in
DESIGN.md ("Readings of the paper").  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import it.  It shares no code with the CUDA path
(paper_2405_08754_b200/) and never imports it; both consume inputs from synth/ only.

Modules
  space    a1  MIG GI/CI x MPS layout enumeration, slot types, Table VII notation
  actions  a5  joint-action index (layout, group, permutation), rank/unrank, counts
  corun    a6  co-run performance model, CoRunTime/SoloRunTime, rewards r_f / r_i
  qnet     a3/a4/a10/a11  duelling Q-MLP forward/backward, centering, fixed point
  env      a2/a5/a7/a8/a9/a13  encoding, argmax, epsilon-greedy step, replay, DQN update
  pruned   a5  exact top-C pruned argmax (config 4)
  brute    a14 exhaustive optimum: RGS enumeration and subset DP (two algorithms)

Parity status per function is stated in each module header; "parity unpinned" marks a
function with no pin independent of itself (also listed in DESIGN.md).
"""
