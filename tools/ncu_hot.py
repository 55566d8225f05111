"""Hottest SASS lines of an ncu capture by warp-stall samples (tools only).

  python tools/ncu_hot.py REP [N]    -> top-N SASS instructions + their stall share,
                                        and the stall totals per CUDA source line
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    try:
        data.append((int(r[isamp]), r[ia], r[isrc].strip()))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
data_sorted = sorted(data, key=lambda d: -d[0])
print(f"total stall samples {tot}")
for s, a, src in data_sorted[:top]:
    print(f"{s / tot * 100:5.1f}%  {a[-5:]}  {src[:110]}")
# cumulative share by opcode
from collections import Counter
c = Counter()
for s, a, src in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    c[op.split(".")[0]] += s
print("by opcode:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in c.most_common(15)))
