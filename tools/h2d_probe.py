"""Host<->device copy rates for the e2e path: pinned vs pageable vs chunked staging.

    python tools/h2d_probe.py [GiB]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1805_01208_b200 import staging  # noqa: E402

gib = float(sys.argv[1]) if len(sys.argv) > 1 else 16.0
n = int(gib * (1 << 30) // 8)
dev = torch.device("cuda")
page = np.random.default_rng(0).random(n)
t0 = time.perf_counter()
pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
t_alloc = time.perf_counter() - t0
pin.numpy()[:] = page
d = torch.empty(n, dtype=torch.float64, device=dev)


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best


res = {"GiB": gib, "pinned_alloc_s": t_alloc}
res["h2d_pinned_GBs"] = n * 8 / timed(lambda: d.copy_(pin, non_blocking=True)) / 1e9
res["h2d_pageable_GBs"] = n * 8 / timed(lambda: d.copy_(torch.from_numpy(page))) / 1e9
res["h2d_staged_GBs"] = n * 8 / timed(lambda: staging.h2d_into(d, page)) / 1e9
out = np.empty(n)
res["d2h_pinned_GBs"] = n * 8 / timed(lambda: pin.copy_(d, non_blocking=True)) / 1e9
res["d2h_pageable_GBs"] = n * 8 / timed(lambda: torch.from_numpy(out).copy_(d)) / 1e9
res["d2h_staged_GBs"] = n * 8 / timed(lambda: staging.d2h_into(out, d)) / 1e9
assert np.array_equal(out, page)
print(res)
