"""Device time of selected kernels of one C5 partition under several env settings.

    python tools/variants.py CFG REGEX "ENV=V ENV2=W" "ENV=V2" ...

Each variant runs in its own process (the library reads its tuning env once);
prints per-variant kernel totals (ms) for the kernels matching REGEX and the
partition's device time.
"""
import json
import os
import subprocess
import sys

CHILD = r'''
import os, re, sys, json
sys.path.insert(0, os.getcwd())
import torch
from torch.profiler import ProfilerActivity, profile
import bench
from paper_1805_01208_b200 import KMeansSettings
from paper_1805_01208_b200.kmeans import partition_device
cfg, pat = sys.argv[1], sys.argv[2]
dev = torch.device("cuda")
c, pts_d, w_d, _ = bench.device_workload(cfg, dev)
s = KMeansSettings(k=c["k"], epsilon=c["epsilon"], seed=0)
a0, st0 = partition_device(pts_d, w_d, s, device=dev)
ref = a0.cpu()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); a1, st1 = partition_device(pts_d, w_d, s, device=dev); e1.record()
torch.cuda.synchronize()
step_ms = e0.elapsed_time(e1)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    partition_device(pts_d, w_d, s, device=dev)
    torch.cuda.synchronize()
rows = {}
for e in prof.events():
    if e.device_type.name != "CUDA" or not re.search(pat, e.name):
        continue
    k = e.name.split("(")[0][-40:]
    r = rows.setdefault(k, [0, 0.0, 0.0])
    t = (e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total) / 1e3
    r[0] += 1
    r[1] += t
    r[2] = max(r[2], t)
print("RESULT", json.dumps({"step_ms": step_ms, "kernels": rows,
      "same_labels": bool(torch.equal(ref, a1.cpu())),
      "centers_equal": bool((st0.final_state.centers == st1.final_state.centers).all())}))
'''


def main():
    cfg, pat = sys.argv[1], sys.argv[2]
    for var in sys.argv[3:] or [""]:
        env = dict(os.environ)
        for kv in var.split():
            k, v = kv.split("=", 1)
            env[k] = v
        out = subprocess.run([sys.executable, "-c", CHILD, cfg, pat], env=env, capture_output=True,
                             text=True, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        line = [ln for ln in out.stdout.splitlines() if ln.startswith("RESULT")]
        if not line:
            print(var or "(default)", "FAILED", out.stderr[-2000:])
            continue
        r = json.loads(line[0][7:])
        tot = sum(v[1] for v in r["kernels"].values())
        print(f"{var or '(default)':30s} step {r['step_ms']:.1f} ms  matched {tot:.1f} ms  "
              f"same_labels {r['same_labels']}")
        for k, v in sorted(r["kernels"].items(), key=lambda x: -x[1][1])[:8]:
            print(f"     {k:42s} {v[0]:5d} {v[1]:9.2f}  max/call {v[2]:.3f}")


if __name__ == "__main__":
    main()
