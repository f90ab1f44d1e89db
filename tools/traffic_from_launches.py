"""Per-kernel-class DRAM traffic from an ncu launch list taken with
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
(cold caches: ncu flushes them before every launch).  Writes a JSON that bench.py reads to fill
roofline["traffic"] (DRAM bytes per launch of the dominant kernel class).
Usage: python tools/traffic_from_launches.py launches.csv OUT.json [steps]"""
import collections
import csv
import json
import re
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}


def klass(name):
    """Kernel name -> bench.py kernel class (the libhrp profiling classes)."""
    m = re.search(r"tc_gemm_kernel<\s*(\d+),\s*(\d+),\s*(\d+)", name)
    if m:
        return "gemm_fwd" if int(m.group(3)) in (0, 1) else "gemm_bwd"
    for key, cls in (("encode_kernel", "encode"), ("sel_kernel", "select"),
                     ("sel_tail_kernel", "select"), ("td_kernel", "td"), ("tdq_kernel", "td"),
                     ("sample_kernel", "sample"), ("sgd", "sgd"), ("split_kernel", "sgd"),
                     ("split_t_kernel", "sgd"), ("reduce_splits", "gemm_bwd"),
                     ("rowsum", "gemm_bwd"), ("transpose_kernel", "gemm_bwd"),
                     ("loss_kernel", "misc"), ("brute_kernel", "brute"), ("head_", "head_bwd")):
        if key in name:
            return cls
    return None


def main(path, out, steps=None):
    hdr, rows = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            rows.append(dict(zip(hdr, r)))
    per = collections.defaultdict(dict)
    names = {}
    for d in rows:
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
        per[d["ID"]][d["Metric Name"]] = v
        names[d["ID"]] = d["Kernel Name"]
    agg = collections.defaultdict(lambda: {"launches": 0, "us": 0.0, "dram_bytes": 0.0})
    for i, m in per.items():
        c = klass(names[i])
        if c is None:
            continue
        a = agg[c]
        a["launches"] += 1
        a["us"] += m.get("gpu__time_duration.sum", 0.0)
        a["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    res = {"source": path, "note": "ncu launch list, cold caches (flushed per launch); "
                                   "dram__bytes_read.sum + dram__bytes_write.sum", "classes": {}}
    for c, a in sorted(agg.items()):
        res["classes"][c] = {"launches": a["launches"], "us_per_launch": a["us"] / a["launches"],
                             "dram_bytes_per_launch": a["dram_bytes"] / a["launches"]}
    json.dump(res, open(out, "w"), indent=1)
    for c, a in res["classes"].items():
        print(f"{c:10s} n={a['launches']:4d} {a['us_per_launch']:9.2f} us  "
              f"{a['dram_bytes_per_launch'] / 1e6:9.3f} MB/launch")


if __name__ == "__main__":
    main(*sys.argv[1:3])
