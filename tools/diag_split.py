"""Diagnostic (GPU): time and accuracy of the tensor-core GEMM per shared-memory split mode
(hrp_diag_config key 1) at the Q-MLP shapes.  usage: python tools/diag_split.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_08754_b200 import hrp  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(1)
    shapes = [(4096, 256, 272), (8192, 256, 256), (4096, 904, 256), (65536, 512, 1088),
              (65536, 512, 512), (65536, 5379, 512)]
    for (M, N, K) in shapes:
        A = np.maximum(rng.standard_normal((M, K)), 0).astype(np.float32)
        Wm = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
        dA, dW = torch.from_numpy(A).to(dev), torch.from_numpy(Wm).to(dev)
        db = torch.zeros(N, dtype=torch.float32, device=dev)
        D = torch.empty(M, N, dtype=torch.float32, device=dev)
        rows = slice(0, 256)
        ref = A[rows].astype(np.float64) @ Wm.astype(np.float64).T
        bound = np.abs(A[rows].astype(np.float64)) @ np.abs(Wm.astype(np.float64)).T + 1e-30
        for mode, atm in ((1, 0), (2, 0), (2, 1)):
            hrp.hrp_diag_config(1, mode)
            hrp.hrp_diag_config(2, atm)
            ms = hrp.hrp_diag_gemm(0, st, M, N, K, dA, dW, db, D, 20, 64 if N <= 1024 else 0)
            torch.cuda.synchronize()
            e = (D[:256].cpu().numpy().astype(np.float64) - ref) / bound
            tf = 2.0 * M * N * K / (ms * 1e-3) / 1e12
            print(f"M={M:6d} N={N:5d} K={K:5d} split {mode} atm {atm}: {ms * 1e3:8.1f} us  {tf:6.1f} TF/s  "
                  f"err mean {e.mean():+.2e} max {np.abs(e).max():.2e}", flush=True)
    hrp.hrp_diag_config(1, 2)
    hrp.hrp_diag_config(2, 1)


if __name__ == "__main__":
    main()
