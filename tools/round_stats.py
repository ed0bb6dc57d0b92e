"""Per-round (active, scanned, q-evals) of one partition, for matching ncu captures
(filter/scan launch i belongs to round i // 2 when the regex selects both kernels).

    python tools/round_stats.py C5 550 551
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1805_01208_b200 import KMeansSettings  # noqa: E402
from paper_1805_01208_b200.kmeans import _Timer, partition_device  # noqa: E402

cfg = sys.argv[1]
dev = torch.device("cuda")
c, pts_d, w_d, _ = bench.device_workload(cfg, dev)
s = KMeansSettings(k=c["k"], epsilon=c["epsilon"], seed=0)
t = _Timer()
partition_device(pts_d, w_d, s, device=dev, timer=t)
torch.cuda.synchronize()
wb = 0 if w_d is None else 8
d = c["d"]
for r in (int(x) for x in sys.argv[2:]):
    nact, nscan, nev = t.rounds[r]
    alg = nact * (4 + 16 + wb) + nscan * (8 * d + 20)
    print(f"round {r}: active {nact} scanned {nscan} qevals {nev} algorithmic_bytes {alg}")
