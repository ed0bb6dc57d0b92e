"""Device activities of one partition longer than a threshold, and the idle gaps before
them, for a window of the timeline (torch.profiler).

    python tools/phase_timeline.py C5 [min_us] [t0_ms] [t1_ms]
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
min_us = float(sys.argv[2]) if len(sys.argv) > 2 else 200.0
w0 = float(sys.argv[3]) * 1e3 if len(sys.argv) > 3 else 0.0
w1 = float(sys.argv[4]) * 1e3 if len(sys.argv) > 4 else 1e12
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
t0 = ev[0][0]
prev_end = t0
for a, b, name in ev:
    gap = a - prev_end
    if w0 <= a - t0 <= w1 and (b - a >= min_us or gap >= min_us / 4):
        short = (name.split("(")[0].replace("void ", "").replace("gp::", "") or name)[-50:]
        print(f"{(a - t0) / 1e3:9.3f} ms  dur {(b - a) / 1e3:8.3f}  gap {gap / 1e3:7.3f}  {short}")
    prev_end = max(prev_end, b)
