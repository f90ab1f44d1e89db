"""Measure the roofline peaks MEASURED_PEAKS.json does not hold (GPU): cuBLAS TF32 dense
(torch.matmul fp32 with TF32 enabled, 8192^3, best of 10 = burst, back to back for 4 s =
sustained) and the fp32 / int32 add issue rate (hrp_diag_alu).  Writes
profiles/measured_peaks_r2.json (read by bench.py's rooflines).
usage: python tools/measure_peaks.py"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_08754_b200 import hrp  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device=dev)
    b = torch.randn(n, n, device=dev)
    flop = 2.0 * n ** 3
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    t0 = time.time()
    k = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 4.0:
        a @ b
        k += 1
        if k % 16 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sus = e0.elapsed_time(e1) / k
    alu_f = max(hrp.hrp_diag_alu(0, 0, 4096) for _ in range(3))
    alu_i = max(hrp.hrp_diag_alu(0, 1, 4096) for _ in range(3))
    out = {"tf32_tflops": flop / best / 1e9, "tf32_tflops_sustained": flop / sus / 1e9,
           "alu_tops": alu_f / 1e12, "alu_int_tops": alu_i / 1e12,
           "gpu": torch.cuda.get_device_name(dev),
           "how": "torch.matmul fp32 8192^3 with allow_tf32 (cuBLAS TF32): best of 10 (burst), "
                  "back to back for 4 s (sustained); hrp_diag_alu: 148x8 CTAs x 256 threads x 8 "
                  "independent add chains (fp32 add.f32 -> alu_tops, int add.u32 -> alu_int_tops)",
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    print(json.dumps(out, indent=1))
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "measured_peaks_r2.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
