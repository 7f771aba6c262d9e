"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into markdown.

    python tools/launch_summary.py launches.csv "command" > profiles/rNN_launches_bench.md
"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0}[r[ui]]
    a = agg[r[ki][:70]]
    a[0] += 1
    a[1] += float(r[vi].replace(",", "")) * scale
total = sum(v[1] for v in agg.values())
cmd = sys.argv[2] if len(sys.argv) > 2 else ""
print(f"# ncu launch list: `{cmd}`\n")
print("`ncu --metrics gpu__time_duration.sum --clock-control none -c 400` (cold-cache, serialised: compare shares)\n")
print("| kernel | launches | total ms | avg us | share |\n|---|---|---|---|---|")
for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{k}` | {n} | {ms:.3f} | {ms / n * 1e3:.1f} | {100 * ms / total:.1f}% |")
