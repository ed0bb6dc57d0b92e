"""Device time of one partition of a bench workload (CUDA events, resident input):
a quick A/B tool for tuning switches (GP_WALK_RATIO=..., GP_LIB_PATH=...).

    python tools/time_partition.py C5 [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1805_01208_b200 import KMeansSettings  # noqa: E402
from paper_1805_01208_b200.kmeans import partition_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda")
c, pts_d, w_d, _ = bench.device_workload(cfg, dev)
s = KMeansSettings(k=c["k"], epsilon=c["epsilon"], seed=0)
partition_device(pts_d, w_d, s, device=dev)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out, stats = partition_device(pts_d, w_d, s, device=dev)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(cfg, "ms", [round(t, 1) for t in ts], "best", round(min(ts), 1),
      "sha", hash(out[:: max(1, out.numel() // 4096)].cpu().numpy().tobytes()) & 0xffffffff)
