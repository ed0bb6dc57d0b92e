"""Warp-stall samples per CUDA source line of one kernel in an ncu report.

    python tools/ncu_lines.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--kernel-name", "regex:" + kern, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
agg, src, tot = defaultdict(float), {}, 0.0
for r in rows[hi + 1:]:
    try:
        ln, s = int(r[0]), float(r[4] or 0)
    except (ValueError, IndexError):
        continue
    agg[ln] += s
    src[ln] = r[1]
    tot += s
print("samples", tot)
for ln, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{ln:5d} {100 * v / tot:5.1f}% {src[ln].strip()[:110]}")
