"""Aggregate an ncu source page (cuda,sass) by CUDA source line: instructions + stall samples.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [top]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
path = None
hdr = None
agg = defaultdict(lambda: [0, 0, ""])
cur_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {n: i for i, n in enumerate(r)}
        continue
    if hdr is None:
        continue
    if r[0]:
        cur_line = (path, r[0], r[1])
        continue
    # sass row under the current source line (Line No empty)
    try:
        s = int(r[4] or 0)
        i = int(r[7] or 0)
    except (ValueError, IndexError):
        continue
    a = agg[cur_line[:2]]
    a[0] += s
    a[1] += i
    a[2] = cur_line[2]
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total samples {ts}, warp instructions {ti}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{v[1] / ti * 100:5.1f}%i {v[0] / ts * 100:5.1f}%s {k[0]}:{k[1]:>4} {v[2].strip()[:80]}")
