"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/launch_summary.py launches.csv
"""
import csv
import re
import sys
from collections import defaultdict

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        rows.append((r["Kernel Name"], float(r["Metric Value"])))
agg = defaultdict(lambda: [0, 0.0])
for name, ns in rows:
    short = re.sub(r"\(.*", "", name)[:70]
    agg[short][0] += 1
    agg[short][1] += ns
tot = sum(v[1] for v in agg.values())
print(f"launches {len(rows)}  total {tot / 1e6:.2f} ms (serialised, cold-cache ncu times)")
print(f"{'kernel':70s} {'calls':>6s} {'ms':>9s} {'share':>6s}")
for k, (c, ns) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{k:70s} {c:6d} {ns / 1e6:9.2f} {100 * ns / tot:5.1f}%")
