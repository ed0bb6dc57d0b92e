"""One partition of a bench workload on cuda:0 (for ncu captures).

    python tools/one_partition.py C5
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1805_01208_b200 import KMeansSettings  # noqa: E402
from paper_1805_01208_b200.kmeans import partition_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
dev = torch.device("cuda")
c, pts_d, w_d, _ = bench.device_workload(cfg, dev)
s = KMeansSettings(k=c["k"], epsilon=c["epsilon"], seed=0)
out, stats = partition_device(pts_d, w_d, s, device=dev)
torch.cuda.synchronize()
print(cfg, "iterations", len(stats.iterations), "rounds", sum(r.balance_rounds for r in stats.iterations))
