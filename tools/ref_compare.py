"""Like-for-like: the unmodified reference vs the B200 path on complete partitions.

    python tools/ref_compare.py [C1 C2 C3] > profiles/round2/ref_compare.json

For every config: the reference's `geopart.kmeans.balanced_kmeans_points`
(baseline/_ref, installed by build()) at p = 1 and p = 256, each in its own
single-threaded process pinned to one core (OMP/MKL/OPENBLAS_NUM_THREADS=1,
sched_setaffinity), all configs' runs concurrently on distinct cores; and the
B200 path end to end through the same public call with host numpy inputs
(H2D and D2H inside the timed region), best of 3 after one warm-up.  Both
sides partition the identical seeded arrays; the labels are compared.
"""
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _ref_run(cfg, p, core, q):
    for v in ("OMP_NUM_THREADS", "MKL_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        os.environ[v] = "1"
    try:
        os.sched_setaffinity(0, {core})
    except Exception:
        pass
    import numpy as np

    import bench
    from paper_1805_01208_b200.workloads import CONFIGS, GENERATORS

    K = bench.reference_module()
    c = CONFIGS[cfg]
    pts, w = GENERATORS[cfg](seed=0)
    s = K.KMeansSettings(k=c["k"], epsilon=c["epsilon"], seed=0)
    t0 = time.perf_counter()
    part, st = K.balanced_kmeans_points(pts, w, s, p=p, return_stats=True)
    dt = time.perf_counter() - t0
    dec = sum(r.total_decisions for r in st.iterations)
    sha = hashlib.sha256(part.assignment.astype(np.int64).tobytes()).hexdigest()[:16]
    q.put((cfg, p, dt, dec, sha))


def gpu_run(cfg):
    import hashlib

    import numpy as np
    import torch

    from paper_1805_01208_b200 import KMeansSettings, balanced_kmeans_points
    from paper_1805_01208_b200.workloads import CONFIGS, GENERATORS

    c = CONFIGS[cfg]
    pts, w = GENERATORS[cfg](seed=0)
    s = KMeansSettings(k=c["k"], epsilon=c["epsilon"], seed=0)
    ts = []
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        part, st = balanced_kmeans_points(pts, w, s, return_stats=True)
        dt = time.perf_counter() - t0
        if i:
            ts.append(dt)
    dec = sum(r.total_decisions for r in st.iterations)
    sha = hashlib.sha256(part.assignment.astype(np.int64).tobytes()).hexdigest()[:16]
    return min(ts), dec, sha


def main():
    cfgs = sys.argv[1:] or ["C1", "C2", "C3"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    try:
        cores = sorted(os.sched_getaffinity(0))
    except Exception:
        cores = list(range(os.cpu_count() or 1))
    jobs = [(cfg, p) for cfg in cfgs for p in (1, 256)]
    procs = [ctx.Process(target=_ref_run, args=(cfg, p, cores[i % len(cores)], q))
             for i, (cfg, p) in enumerate(jobs)]
    for pr in procs:
        pr.start()
    gpu = {cfg: gpu_run(cfg) for cfg in cfgs}    # while the CPU runs go on other cores
    ref = {}
    for _ in jobs:
        cfg, p, dt, dec, sha = q.get()
        ref[(cfg, p)] = (dt, dec, sha)
    for pr in procs:
        pr.join()
    out = {"host_cores": len(cores), "configs": {}}
    for cfg in cfgs:
        g_dt, g_dec, g_sha = gpu[cfg]
        r1, r256 = ref[(cfg, 1)], ref[(cfg, 256)]
        best = min(r1[0], r256[0])
        out["configs"][cfg] = {
            "reference_s_p1": r1[0], "reference_s_p256": r256[0], "reference_best_s": best,
            "reference_gpt_s_best": r1[1] / best / 1e9,
            "b200_e2e_s": g_dt, "b200_e2e_gpt_s": g_dec / g_dt / 1e9,
            "speedup_vs_best_reference": best / g_dt,
            "point_assignments": g_dec, "reference_point_assignments": r1[1],
            "labels_identical": g_sha == r1[2] == r256[2],
        }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
