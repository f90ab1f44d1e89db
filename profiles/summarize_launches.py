"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, total us, share of the step.  Usage: python summarize_launches.py launches.csv"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "")[:70]
        v = float(d["Metric Value"].replace(",", ""))
        if d["Metric Unit"] == "us":
            v *= 1e3
        elif d["Metric Unit"] == "ms":
            v *= 1e6
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':70s} {'n':>4s} {'total_us':>10s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:70s} {v[0]:4d} {v[1] / 1e3:10.1f} {100 * v[1] / tot:5.1f}%")
    print(f"{'TOTAL':70s} {sum(v[0] for v in agg.values()):4d} {tot / 1e3:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
