"""Diagnostic (GPU): accuracy of the 3xTF32 tcgen05 GEMM per TMEM accumulator layout
(hrp_diag_config key 0) against fp64, next to fp32 CPU (torch) -- errors in units of the
abs-sum bound sum_k |a_k b_k|, signed mean (truncation bias) and rms / max.
usage: python tools/diag_precision.py > profiles/r2_gemm_precision.txt"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_08754_b200 import hrp  # noqa: E402


def stats(D, ref, bound):
    e = (D - ref) / bound
    return f"mean {e.mean():+.2e} rms {np.sqrt((e ** 2).mean()):.2e} max {np.abs(e).max():.2e}"


def main():
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(0)
    M, N = 512, 256
    print("3xTF32 GEMM D = A W^T + b vs fp64; error / sum_k |a_k w_k|")
    for kind in ("signed", "relu-positive"):
        for K in (256, 512, 1088, 2048):
            A = rng.standard_normal((M, K))
            Wm = rng.standard_normal((N, K)) / np.sqrt(K)
            if kind == "relu-positive":
                A = np.maximum(A, 0.0)
                Wm = np.abs(Wm)
            b = np.zeros(N)
            A32, W32 = A.astype(np.float32), Wm.astype(np.float32)
            ref = A32.astype(np.float64) @ W32.astype(np.float64).T
            bound = np.abs(A32.astype(np.float64)) @ np.abs(W32.astype(np.float64)).T
            bound = np.maximum(bound, 1e-30)
            cpu = (torch.from_numpy(A32) @ torch.from_numpy(W32).T).numpy().astype(np.float64)
            print(f"{kind:14s} K={K:5d} fp32 CPU     {stats(cpu, ref, bound)}")
            dA = torch.from_numpy(A32).to(dev)
            dW = torch.from_numpy(W32).to(dev)
            db = torch.zeros(N, dtype=torch.float32, device=dev)
            for mode in (0, 1, 2):
                hrp.hrp_diag_config(0, mode)
                for bn in (64, 128, 256):
                    D = torch.empty(M, N, dtype=torch.float32, device=dev)
                    hrp.hrp_diag_gemm(0, st, M, N, K, dA, dW, db, D, 0, bn)
                    torch.cuda.synchronize()
                    g = D.cpu().numpy().astype(np.float64)
                    print(f"{kind:14s} K={K:5d} mode {mode} BN={bn:3d} {stats(g, ref, bound)}")
    hrp.hrp_diag_config(0, 2)


if __name__ == "__main__":
    main()
