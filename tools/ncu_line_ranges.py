"""Instruction / stall totals of an ncu report (source page) grouped by file:line ranges.
Usage: python tools/ncu_line_ranges.py REP file:lo-hi[=name] ..."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ranges = []
for a in sys.argv[2:]:
    spec, _, name = a.partition("=")
    f, _, lr = spec.partition(":")
    lo, _, hi = lr.partition("-")
    ranges.append((name or spec, f, int(lo), int(hi)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname = None
hdr = None
tot = {r[0]: [0, 0] for r in ranges}
all_i = all_s = 0
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        try:
            ie = int(r[hdr.index("Instructions Executed")])
            ss = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except ValueError:
            continue
        all_i += ie
        all_s += ss
        ln = int(r[0])
        for name, f, lo, hi in ranges:
            if f == fname and lo <= ln <= hi:
                tot[name][0] += ie
                tot[name][1] += ss
print(f"total warp-instructions {all_i}, stall samples {all_s}")
for name, (ie, ss) in tot.items():
    print(f"{name:24s} {100 * ie / max(all_i, 1):5.1f}% inst {100 * ss / max(all_s, 1):5.1f}% stall")
