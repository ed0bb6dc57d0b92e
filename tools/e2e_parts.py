"""Where the end-to-end time of one C5 partition goes (host buffers in, labels out)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1805_01208_b200 import KMeansSettings, balanced_kmeans_points  # noqa: E402
from paper_1805_01208_b200.kmeans import _finish, partition_device  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
dev = torch.device("cuda")
c, pts_d, w_d, host = bench.device_workload(cfg, dev)
pts, w = host()
s = KMeansSettings(k=c["k"], epsilon=c["epsilon"], seed=0)


def t(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t0


for it in range(3):
    x, th2d = t(lambda: torch.from_numpy(pts).to(dev, non_blocking=True))
    (a, st), tdev = t(lambda: partition_device(x, None, s, device=dev))
    _, tfin = t(lambda: _finish(a, st, s.k, True))
    _, tall = t(lambda: balanced_kmeans_points(pts, None, s, return_stats=True))
    print(f"h2d {th2d:.3f}  partition_device(host-AoS copy on device) {tdev:.3f}  finish {tfin:.3f}  "
          f"public API total {tall:.3f}")
    _, tsoa = t(lambda: partition_device(pts_d, None, s, device=dev))
    print(f"   partition_device(SoA device view) {tsoa:.3f}  peak GB "
          f"{torch.cuda.max_memory_allocated() / 1e9:.1f} reserved {torch.cuda.max_memory_reserved() / 1e9:.1f}")
