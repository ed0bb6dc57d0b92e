"""Per-round counters of one partition (for matching ncu captures of a given round).

    GP_NVTX=1 python tools/round_trace.py C5 [first last]

Prints round index (the GP_NVTX range number), active entries, rescanned entries and
distance evaluations, i.e. the §8d algorithmic bytes and flops of each round.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1805_01208_b200 import KMeansSettings  # noqa: E402
from paper_1805_01208_b200.kmeans import _Timer, partition_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3]) if len(sys.argv) > 3 else 10 ** 9
dev = torch.device("cuda")
c, pts_d, w_d, _ = bench.device_workload(cfg, dev)
s = KMeansSettings(k=c["k"], epsilon=c["epsilon"], seed=0)
t = _Timer()
partition_device(pts_d, w_d, s, device=dev, timer=t)
torch.cuda.synchronize()
d = c["d"]
wb = 0 if w_d is None else 8
for i, ((nact, nscan, nev), (e0, e1)) in enumerate(zip(t.rounds, t.events)):
    if lo <= i <= hi:
        print(f"round {i} active {nact} scanned {nscan} evals {nev} "
              f"filter_alg_bytes {nact * (20 + wb)} scan_alg_bytes {nscan * (8 * d + 20)} "
              f"flops {nev * (3 * d + 1)} ms {e0.elapsed_time(e1):.3f}")
