"""Device timings of the path's callers (gp_predict, the SFC baseline).

    python tools/callers_bench.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1805_01208_b200 import _native as N  # noqa: E402
from paper_1805_01208_b200.baselines import sfc_labels_device  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


g = torch.Generator(device="cuda").manual_seed(0)
sh = torch.cuda.current_stream().cuda_stream
for d, n, k in ((2, 1 << 24, 1024), (3, 1 << 24, 1024), (2, 1 << 22, 16384)):
    X = torch.rand((n, d), dtype=torch.float64, device="cuda", generator=g)
    C = torch.rand((k, d), dtype=torch.float64, device="cuda", generator=g)
    f = torch.rand(k, dtype=torch.float64, device="cuda", generator=g) * 0.5 + 0.75
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    t = timed(lambda: N.call("gp_predict", X.data_ptr(), n, d, C.data_ptr(), f.data_ptr(), k, 1,
                             out.data_ptr(), sh))
    fl = n * k * (3 * d + 2)
    print(f"predict d={d} n={n} k={k}: {t*1e3:.2f} ms  {n*k/t/1e9:.1f} G pairs/s  "
          f"{fl/t/1e12:.2f} TFLOP/s (fp64, 3d+2 per pair)")
for d, n, k, wk in ((2, 1 << 24, 1024, "unit"), (3, 1 << 24, 1024, "int"),
                    (2, 1 << 24, 1024, "f64"), (2, 1 << 28, 16384, "unit")):
    X = torch.rand((n, d), dtype=torch.float64, device="cuda", generator=g)
    w = None
    if wk == "int":
        w = torch.randint(1, 61, (n,), device="cuda", generator=g).to(torch.float64)
    elif wk == "f64":
        w = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) + 0.5
    t = timed(lambda: sfc_labels_device(X, w, k), reps=3)
    print(f"sfc_labels d={d} n={n} k={k} w={wk}: {t*1e3:.2f} ms  {n/t/1e9:.2f} G pts/s")
    del X, w
