"""Schedule-quality report for the paper's compared methods (P:245-248,
Fig. 8): relative throughput Solo / CoRun of the exhaustive optimum on Q1-Q12
(Table V, W = 12) for Time Sharing, MIG Only (C = 2), MPS Only (C <= 4) and MIG+MPS
(C <= 4), computed on the GPU by hrp_bruteforce_optimum (parity with the oracle:
tests/test_gpu_brute.py).  The co-run model is R8's synthetic one, so the numbers are the
synthetic analogue of Fig. 8, not a reproduction of it.

usage: python tools/schedule_quality.py [--out profiles/r1_schedule_quality.md]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    from paper_2405_08754_b200.session import bruteforce
    pool = synth.make_pool(27)
    Q = synth.table_v_windows(pool)
    rows, times = {}, {}
    for name, (scfg, lay) in synth.BASELINE_SPACES.items():
        bruteforce(scfg, pool, Q, layouts=lay)               # warm-up (tables, module load)
        t = time.perf_counter()
        best, solo, rgs, _ = bruteforce(scfg, pool, Q, layouts=lay)
        times[name] = time.perf_counter() - t
        rows[name] = (solo / best, rgs)
    names = ["mig_only", "mps_only", "mig_mps"]
    hdr = "| mix | Time Sharing | MIG Only (C=2) | MPS Only (C<=4) | MIG+MPS (C<=4) | MIG+MPS job sets |"
    out = [hdr, "|" + "---|" * 6]
    for i in range(len(Q)):
        sets = rows["mig_mps"][1][i]
        out.append(f"| Q{i + 1} | 1.000 | " + " | ".join(f"{rows[n][0][i]:.3f}" for n in names)
                   + " | " + "".join(str(int(x)) for x in sets) + " |")
    out.append("| AM | 1.000 | " + " | ".join(f"{rows[n][0].mean():.3f}" for n in names) + " | |")
    out.append("| max | 1.000 | " + " | ".join(f"{rows[n][0].max():.3f}" for n in names) + " | |")
    txt = "\n".join(out)
    print(txt)
    meta = {"device": torch.cuda.get_device_name(0),
            "seconds_per_call_12_windows": {k: round(v, 4) for k, v in times.items()},
            "am": {n: float(rows[n][0].mean()) for n in names}}
    print(json.dumps(meta))
    if args.out:
        with open(args.out, "w") as f:
            f.write("# Schedule quality of the compared methods on Q1-Q12 (synthetic co-run model R8)\n\n"
                    "Relative throughput = SoloRunTime / optimal CoRunTime (P:139-140), exhaustive "
                    "optimum per method's search space (P:245-248), W = 12; produced by "
                    "`tools/schedule_quality.py` on the GPU (hrp_bruteforce_optimum).  "
                    "Job sets column: RGS of the MIG+MPS optimum (window position -> set).\n\n"
                    + txt + "\n\n```\n" + json.dumps(meta, indent=1) + "\n```\n")


if __name__ == "__main__":
    main()
