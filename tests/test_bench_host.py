"""Host-side logic of bench.py and the profiling tools (no GPU): roofline accounting of the
structured update and the ncu launch-list -> DRAM-traffic summary."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import bench  # noqa: E402
import synth  # noqa: E402


class _Osp:
    W, T, L, H = 16, 52, 71, 1 + 71 + 16 * 52


def _prof(head):
    p = {"gemm_fwd": (1.0, 11), "gemm_bwd": (1.0, 5), "select": (1.0, 1), "td": (1.0, 2),
         "encode": (1.0, 3), "sgd": (1.0, 1)}
    if head:
        p["head_bwd"] = (1.0, 7)
    return p


def test_roofline_flops_structured_vs_dense():
    cfg = synth.config(2)
    E, B = cfg.n_envs, cfg.batch
    dims = [_Osp.W * 17] + [cfg.net.hidden_width] * cfg.net.hidden_layers + [_Osp.H]
    F = sum(2 * dims[i] * dims[i + 1] for i in range(len(dims) - 1))
    Fh = sum(2 * dims[i] * dims[i + 1] for i in range(len(dims) - 2))
    Fo = 2 * dims[-2] * dims[-1]
    dense = bench.rooflines(_prof(False), 1, (1, 1), cfg, _Osp)
    struct = bench.rooflines(_prof(True), 1, (1, 1), cfg, _Osp)
    # 1 ms per step: achieved TFLOP/s = flops / 1e9
    assert dense["gemm_fwd"]["achieved"] == pytest.approx((E + 3 * B) * F / 1e9)
    assert struct["gemm_fwd"]["achieved"] == pytest.approx((E * F + 3 * B * Fh + B * Fo) / 1e9)
    # backward: weight gradients of every GEMM layer, data gradients of all but the first;
    # the structured head has neither
    bw = lambda top: sum(2 * B * dims[i] * dims[i + 1] * (2 if i > 0 else 1) for i in range(top))
    nl = len(dims) - 1
    assert dense["gemm_bwd"]["achieved"] == pytest.approx(bw(nl) / 1e9)
    assert struct["gemm_bwd"]["achieved"] == pytest.approx(bw(nl - 1) / 1e9)
    assert struct["head_bwd"]["bound"] == "hbm"
    assert "head_bwd" not in dense


CSV = '''"ID","Process ID","Process Name","Host Name","Kernel Name","Context","Stream","Block Size","Grid Size","Device","CC","Section Name","Metric Name","Metric Unit","Metric Value"
"0","1","python","h","void hrp::<unnamed>::tc_gemm_kernel<64, 4, 1>(CUtensorMap_st)","1","7","(256, 1, 1)","(4, 32, 1)","0","10.0","Command line profiler metrics","dram__bytes_read.sum","Mbyte","8.00"
"0","1","python","h","void hrp::<unnamed>::tc_gemm_kernel<64, 4, 1>(CUtensorMap_st)","1","7","(256, 1, 1)","(4, 32, 1)","0","10.0","Command line profiler metrics","dram__bytes_write.sum","Mbyte","1.00"
"0","1","python","h","void hrp::<unnamed>::tc_gemm_kernel<64, 4, 1>(CUtensorMap_st)","1","7","(256, 1, 1)","(4, 32, 1)","0","10.0","Command line profiler metrics","gpu__time_duration.sum","us","10.00"
"1","1","python","h","void hrp::<unnamed>::tc_gemm_kernel<64, 4, 2>(CUtensorMap_st)","1","7","(256, 1, 1)","(4, 32, 1)","0","10.0","Command line profiler metrics","dram__bytes_read.sum","Kbyte","500"
"1","1","python","h","void hrp::<unnamed>::tc_gemm_kernel<64, 4, 2>(CUtensorMap_st)","1","7","(256, 1, 1)","(4, 32, 1)","0","10.0","Command line profiler metrics","gpu__time_duration.sum","ms","0.02"
"2","1","python","h","hrp::head_scatter_kernel(hrp::HeadArgs, int)","1","7","(256, 1, 1)","(586, 1, 1)","0","10.0","Command line profiler metrics","dram__bytes_read.sum","byte","4096"
"2","1","python","h","hrp::head_scatter_kernel(hrp::HeadArgs, int)","1","7","(256, 1, 1)","(586, 1, 1)","0","10.0","Command line profiler metrics","gpu__time_duration.sum","us","5"
"3","1","python","h","void at::vectorized_elementwise_kernel<4>(int)","1","7","(128, 1, 1)","(4, 1, 1)","0","10.0","Command line profiler metrics","gpu__time_duration.sum","us","99"
'''


def test_traffic_from_launch_list(tmp_path):
    import traffic_from_launches as TL
    src = tmp_path / "l.csv"
    src.write_text(CSV)
    out = tmp_path / "t.json"
    TL.main(str(src), str(out))
    t = json.load(open(out))["classes"]
    assert t["gemm_fwd"] == {"launches": 1, "us_per_launch": pytest.approx(10.0),
                             "dram_bytes_per_launch": pytest.approx(9e6)}
    assert t["gemm_bwd"]["us_per_launch"] == pytest.approx(20.0)
    assert t["gemm_bwd"]["dram_bytes_per_launch"] == pytest.approx(5e5)
    assert t["head_bwd"]["dram_bytes_per_launch"] == pytest.approx(4096)
    assert set(t) == {"gemm_fwd", "gemm_bwd", "head_bwd"}   # torch's fill kernel is not ours


def test_kernel_classes_match_header():
    # the binding's class names follow include/hrp.h's HRP_K_* order
    import re
    from paper_2405_08754_b200 import hrp
    hdr = open(os.path.join(ROOT, "include", "hrp.h")).read()
    ids = {m.group(1): int(m.group(2)) for m in re.finditer(r"HRP_K_(\w+)\s*=\s*(\d+)", hdr)}
    assert ids["COUNT"] == len(hrp.KERNEL_CLASSES)
    assert ids["HEAD_BWD"] == hrp.KERNEL_CLASSES.index("head_bwd")
    assert ids["GEMM_BWD"] == hrp.KERNEL_CLASSES.index("gemm_bwd")


def test_measured_traffic_is_per_configuration():
    # the roofline's `traffic` comes from a launch list of the same configuration only
    t2, src2 = bench.measured_traffic("gemm_fwd", 2)
    t4, src4 = bench.measured_traffic("gemm_fwd", 4)
    assert t2 and "cfg2" in src2 and t4 and "cfg4" in src4 and t4 > 10 * t2
    assert bench.measured_traffic("gemm_fwd", 1) == (None, None)   # no cfg1 list committed
    tb, srcb = bench.measured_traffic("brute", 3)
    assert tb and "brute" in srcb


def test_clock_sampler_without_gpu():
    # no NVML device and no nvidia-smi here: the sampler must not raise, and reports None
    c = bench.Clocks(0)
    out = c.stop()
    assert out is None or {"sm_mhz", "sm_max_mhz", "reasons", "samples"} <= set(out)
