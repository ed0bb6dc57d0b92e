"""Per-kernel device-time table of one partition (torch.profiler / CUPTI, no replay).

    python tools/kprof.py C5 [--warm]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_1805_01208_b200 import KMeansSettings  # noqa: E402
from paper_1805_01208_b200.kmeans import _Timer, partition_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
dev = torch.device("cuda")
c, pts_d, w_d, _ = bench.device_workload(cfg, dev)
s = KMeansSettings(k=c["k"], epsilon=c["epsilon"], seed=0)
partition_device(pts_d, w_d, s, device=dev)  # warm
torch.cuda.synchronize()
N0 = __import__("paper_1805_01208_b200._native", fromlist=["calls"])
N0.calls.clear()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    out, stats = partition_device(pts_d, w_d, s, device=dev)
    torch.cuda.synchronize()
rows = {}
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    r = rows.setdefault(e.name[:70], [0, 0.0])
    r[0] += 1
    r[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
tot = sum(v[1] for v in rows.values())
longest = sorted(((e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total,
                   e.name[:60]) for e in prof.events() if e.device_type.name == "CUDA"),
                 reverse=True)[:12]
print("longest launches (ms):", [(round(t / 1e3, 2), n) for t, n in longest])
print("API calls:", dict(sorted(N0.calls.items())))
print(f"{'kernel':72s} {'calls':>6s} {'ms':>10s} {'%':>6s}")
for k, v in sorted(rows.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{k:72s} {v[0]:6d} {v[1] / 1e3:10.2f} {100 * v[1] / tot:6.1f}")
# per-call durations (in launch order) of the fold chain and assign kernels
pat = os.environ.get("KPROF_CALLS", "fold_|run_mark|run_emit|RadixSort|Select|filter_kernel|scan_kernel")
import re  # noqa: E402
seq = [(e.time_range.start if hasattr(e, "time_range") else 0, e.name[:40],
        (e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total) / 1e3)
       for e in prof.events() if e.device_type.name == "CUDA" and re.search(pat, e.name)]
seq.sort()
print("per-call ms (launch order):")
line = []
for _, nm, ms_ in seq:
    line.append(f"{nm.split('(')[0].split('<')[0].replace('void ', '').replace('gp::', '')[-18:]}={ms_:.3f}")
    if len(line) == 6:
        print("  " + " ".join(line))
        line = []
if line:
    print("  " + " ".join(line))
print("device total ms", tot / 1e3, "rounds", sum(r.balance_rounds for r in stats.iterations),
      "iterations", len(stats.iterations))
print("phase active rounds scanned/round evals/scanned")
for r in stats.iterations[::4] + stats.iterations[-3:]:
    sc = r.total_decisions - r.skip_decisions
    print(r.phase, r.active_points, r.balance_rounds, sc // max(r.balance_rounds, 1),
          round(r.distance_evals / max(sc, 1), 2))

t = _Timer()
out, stats = partition_device(pts_d, w_d, s, device=dev, timer=t)
torch.cuda.synchronize()
os.environ["GP_SCAN_STATS"] = "1"     # separate run: the statistics cost atomics
t2 = _Timer()
partition_device(pts_d, w_d, s, device=dev, timer=t2)
torch.cuda.synchronize()
t.scan = t2.scan
ms = [a.elapsed_time(b) for a, b in t.events]
full = [(m, r) for m, r in zip(ms, t.rounds) if r[0] == c["n"]]
samp = [(m, r) for m, r in zip(ms, t.rounds) if r[0] != c["n"]]
print("assign ms: sample %.1f (%d rounds), full %.1f (%d rounds, %.3f ms/round, scanned/round %.0f)"
      % (sum(m for m, _ in samp), len(samp), sum(m for m, _ in full), len(full),
         sum(m for m, _ in full) / max(len(full), 1),
         sum(r[1] for _, r in full) / max(len(full), 1)))

import numpy as np  # noqa: E402
from paper_1805_01208_b200 import _native as N  # noqa: E402
st = np.zeros(4, dtype=np.int64)
N.lib.gp_fold_stats(st.ctypes.data)
print("last fold: runs", st[0], "valid runs", st[2], "pairs", st[3])
by = {}
for ms_, r in zip(ms, t.rounds):
    e = by.setdefault(r[0], [0, 0.0, 0, 0])
    e[0] += 1; e[1] += ms_; e[2] += r[1]; e[3] += r[2]
print("active  rounds  ms  ms/round  scanned/round  qevals/scanned")
for m_, e in sorted(by.items()):
    print(m_, e[0], round(e[1], 1), round(e[1] / e[0], 3), e[2] // e[0], round(e[3] / max(e[2], 1), 1))

if t.scan:
    print("scan stats per active size: units  pts/unit  nsrc/unit  ncand/unit  overflow%  "
          "exact/pt  walk/pass  passes/unit")
    by = {}
    for st_, r in zip(t.scan, t.rounds):
        e = by.setdefault(r[0], np.zeros(8, dtype=np.float64))
        e += st_.astype(np.float64)
    for m_, e in sorted(by.items()):
        u = max(e[0], 1)
        print(m_, int(e[0]), round(e[1] / u, 1), round(e[2] / u, 1), round(e[3] / u, 1),
              round(100 * e[4] / u, 2), round(e[5] / max(e[1], 1), 3),
              round(e[6] / max(e[7], 1), 1), round(e[7] / u, 2))
