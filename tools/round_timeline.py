"""Kernel / memcpy timeline of a few balance rounds of one partition (torch.profiler):
every device activity between the filter launches of rounds R..R+N, with start offsets,
durations and the idle gap before each.

    python tools/round_timeline.py C5 300 2
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_1805_01208_b200 import KMeansSettings  # noqa: E402
from paper_1805_01208_b200.kmeans import partition_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
first = int(sys.argv[2]) if len(sys.argv) > 2 else 300
count = int(sys.argv[3]) if len(sys.argv) > 3 else 2
dev = torch.device("cuda")
c, pts_d, w_d, _ = bench.device_workload(cfg, dev)
s = KMeansSettings(k=c["k"], epsilon=c["epsilon"], seed=0)
partition_device(pts_d, w_d, s, device=dev)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    partition_device(pts_d, w_d, s, device=dev)
    torch.cuda.synchronize()
ev = sorted(((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
             if e.device_type.name == "CUDA"), key=lambda x: x[0])
filters = [i for i, e in enumerate(ev) if "filter_kernel" in e[2]]
lo, hi = filters[first], filters[min(first + count, len(filters) - 1)]
t0 = ev[lo][0]
prev_end = ev[lo - 1][1] if lo else t0
for a, b, name in ev[lo:hi + 1]:
    short = name.split("(")[0].replace("void ", "").replace("gp::", "")[-44:]
    print(f"{a - t0:9.1f} us  dur {b - a:8.1f}  gap {a - prev_end:7.1f}  {short}")
    prev_end = max(prev_end, b)
