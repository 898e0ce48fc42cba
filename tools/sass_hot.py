"""Print the hottest SASS lines (warp-stall samples) of an ncu report.
    python tools/sass_hot.py REPORT.ncu-rep [N] [--around ADDR_SUFFIX]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
ia, isrc = h.index("Address"), h.index("Source")
iw = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
tot = sum(float(r[iw] or 0) for r in data)
print("total samples", tot)
c, s = Counter(), Counter()
for r in data:
    parts = r[isrc].split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") else parts[0]
    op = op.split(".")[0]
    c[op] += float(r[ie] or 0)
    s[op] += float(r[iw] or 0)
for op, v in sorted(s.items(), key=lambda x: -x[1])[:12]:
    print(f"{op:10s} samples {100 * v / tot:5.1f}%  executed {c[op]:.3e}")
print("--- top lines")
for r in sorted(data, key=lambda r: -float(r[iw] or 0))[:n]:
    print(r[ia][-5:], r[isrc][:70].ljust(70), r[iw], r[ie])
