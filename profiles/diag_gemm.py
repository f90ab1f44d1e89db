"""Diagnostics: time the tcgen05 3xTF32 GEMM alone at the Q-MLP shapes and dump the per-event
trace of CTA (0,0) (hrp_diag_gemm).  Usage (GPU): python profiles/diag_gemm.py"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08754_b200 import hrp  # noqa: E402


def run(M, N, K, reps=20, bn=0):
    L = hrp.lib()
    L.hrp_diag_gemm.argtypes = ([C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 5
                                + [C.c_int, C.c_int, C.c_void_p])
    L.hrp_diag_gemm.restype = C.c_int
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    A = torch.randn(M, K, device=dev, generator=g)
    W = torch.randn(N, K, device=dev, generator=g) * 0.05
    b = torch.randn(N, device=dev, generator=g)
    D = torch.empty(M, N, device=dev)
    tr = torch.zeros(256, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream().cuda_stream

    ms_k = C.c_float(0.0)

    def call(trace=None, n=0):
        r = L.hrp_diag_gemm(0, C.c_void_p(st), M, N, K, C.c_void_p(A.data_ptr()),
                            C.c_void_p(W.data_ptr()), C.c_void_p(b.data_ptr()),
                            C.c_void_p(D.data_ptr()),
                            C.c_void_p(trace.data_ptr()) if trace is not None else None,
                            n, bn, C.byref(ms_k))
        assert r == 0, L.hrp_last_error()
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    ref = torch.addmm(b.double(), A.double(), W.double().t())
    err = ((D.double() - ref).abs().max() / ref.abs().max()).item()
    call(None, reps)
    torch.cuda.synchronize()
    ms = ms_k.value                   # GEMM kernel only, back-to-back launches
    call(tr)
    torch.cuda.synchronize()
    t = tr.cpu().tolist()
    t0 = t[0]
    nk = (K + 31) // 32
    ev = {"setup": t[1] - t0, "tma": [t[2 + k] - t0 for k in range(min(nk, 64))],
          "mma": [t[130 + k] - t0 for k in range(min(nk, 64))], "acc": t[194] - t0,
          "end": t[195] - t0}
    flops = 2.0 * M * N * K
    return {"M": M, "N": N, "K": K, "bn": bn, "ms_kernel": ms, "tflops_logical": flops / ms / 1e9,
            "max_rel_err": err, "trace_ns": ev}


if __name__ == "__main__":
    shapes = [(4096, 256, 272), (4096, 256, 256), (4096, 904, 256), (8192, 256, 256),
              (8192, 904, 256), (65536, 512, 1088), (65536, 512, 512), (65536, 5379, 512)]
    bns = [int(x) for x in sys.argv[1:]] or [0]
    for shp in shapes:
        for bn in bns:
            o = run(*shp, bn=bn)
            o["trace_ns"] = {k: o["trace_ns"][k] for k in ("setup", "acc", "end")}
            print(json.dumps(o), flush=True)
