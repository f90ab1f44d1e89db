"""Per-CUDA-source-line instruction counts and stall samples from an ncu report (source page).
Usage: python tools/ncu_hot_lines.py REP [top_n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
res = []
fname = None
hdr = None
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
        if ie or ss:
            res.append((ie, ss, fname, int(r[0]), r[1].strip()[:90]))
tot_i = sum(x[0] for x in res) or 1
tot_s = sum(x[1] for x in res) or 1
print(f"total warp-instructions {tot_i}, stall samples {tot_s}")
for ie, ss, f, ln, src in sorted(res, key=lambda x: -x[1])[:top]:
    print(f"{100*ie/tot_i:5.1f}% inst {100*ss/tot_s:5.1f}% stall  {f}:{ln}  {src}")
