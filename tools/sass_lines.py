"""Static SASS size of one kernel by CUDA source line (nvdisasm -g): which source lines the
compiler expanded into the most instructions.  Usage:
  python tools/sass_lines.py OBJ.o KERNEL_SUBSTRING [top_n] [file:lo-hi=name ...]"""
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

obj, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 25
ranges = [a for a in sys.argv[3:] if ":" in a]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True,
                     text=True).stdout
cnt = Counter()
cur = None
inside = False
total = 0
for ln in dis.split("\n"):
    if ln.startswith("//--------------------- .text."):
        inside = kern in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
        total += 1
        cnt[cur] += 1
print(f"{kern}: {total} instructions")
if ranges:
    for a in ranges:
        spec, _, name = a.partition("=")
        f, _, lr = spec.partition(":")
        lo, _, hi = lr.partition("-")
        n = sum(v for (ff, l), v in cnt.items() if ff == f and int(lo) <= l <= int(hi))
        print(f"{name or spec:24s} {n:6d}")
else:
    for (f, l), v in cnt.most_common(top):
        print(f"{v:6d}  {f}:{l}")
