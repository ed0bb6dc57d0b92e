"""GPU idle gaps of one partition, attributed to the kernels around them.

    python tools/gaps.py C5
"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_1805_01208_b200 import KMeansSettings  # noqa: E402
from paper_1805_01208_b200.kmeans import partition_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
dev = torch.device("cuda")
c, pts_d, w_d, _ = bench.device_workload(cfg, dev)
s = KMeansSettings(k=c["k"], epsilon=c["epsilon"], seed=0)
partition_device(pts_d, w_d, s, device=dev)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    partition_device(pts_d, w_d, s, device=dev)
    torch.cuda.synchronize()
ev = []
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    t0 = e.time_range.start
    t1 = e.time_range.end
    ev.append((t0, t1, e.name[:50]))
ev.sort()
gaps = defaultdict(lambda: [0, 0.0])
total_gap = 0.0
end = ev[0][1]
prev = ev[0][2]
for t0, t1, name in ev[1:]:
    g = t0 - end
    if g > 2.0:   # microseconds
        key = f"{prev} -> {name}"
        gaps[key][0] += 1
        gaps[key][1] += g
        total_gap += g
    if t1 > end:
        end = t1
        prev = name
span = ev[-1][1] - ev[0][0]
print(f"span {span / 1e3:.1f} ms, idle gaps > 2 us: {total_gap / 1e3:.1f} ms")
for key, (n, g) in sorted(gaps.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{g / 1e3:8.2f} ms {n:6d}  {key}")
