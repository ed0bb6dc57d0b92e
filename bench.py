"""Benchmark of the balanced k-means hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl b200|reference]

One step = one complete partition (SFC bootstrap + every movement iteration
and balance round of Alg. 2) of the named synthetic configuration.

  value : point-assignments/s (G/s) with inputs resident in HBM, timed with
          CUDA events around each step (L2 flushed between steps);
          point-assignments = the reference's total_decisions (one active
          point processed in one balance round, kmeans.py:309).
  e2e   : the same metric through the public API balanced_kmeans_points with
          host numpy inputs (H2D of coords/weights and D2H of the int64
          assignment inside the timed region).
  roofline : the assign kernel (gp_assign_round), algorithmic bytes per
          SURVEY §8d (B = n_act*(20+w_B) + n_scan*(8d+20)) over its
          CUDA-event time, against MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline : the reference's own path (the unmodified geopart package that
          build() installs into baseline/_ref; the oracle port if it is absent) on
          a bounded sample of the same workload, single-threaded, on this host.

--impl reference times that CPU implementation alone, one single-threaded run per
host core in parallel (the reference is single-threaded numpy).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

DESCR = {
    "C1": "2D uniform n=100000, unit weights, k=16, eps=0.03",
    "C2": "2D 32-component Gaussian mixture n=2^20, integer weights 1-60, k=64, eps=0.03",
    "C3": "3D jittered 128^3 grid n=2^21, unit weights, k=256, eps=0.03",
    "C4": "3D radially refined cloud n=2^24, float32 weights in [1,4], k=1024, eps=0.05",
    "C5": "2D half uniform / half 1024-component mixture n=2^30, unit weights, k=16384, eps=0.03",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    # C5 (BASELINE configs[4], 2^30 points, k=16384) is the north star's headline
    # configuration and fits one B200; C1-C4 are selectable and are parity-tested
    ap.add_argument("--config", default=os.environ.get("GP_BENCH_CONFIG", "C5"))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pageable", action="store_true")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(cfg):
    """DRAM bytes of one captured assign round (ncu --set full, committed under
    profiles/) next to that round's algorithmic bytes, or None."""
    path = os.path.join(ROOT, "profiles", "round2", f"ncu_traffic_{cfg}.json")
    if not os.path.exists(path):
        path = os.path.join(ROOT, "profiles", "round1", f"ncu_traffic_{cfg}.json")
    try:
        with open(path) as f:
            t = json.load(f)
        return t
    except Exception:
        return None


def split_roofline(f_bytes, f_ms, s_bytes, s_ms, flops, world, peak, tr):
    """Filter (skip test + block weights: n_act*(20+w_B)) and scan (rescans:
    n_scan*(8d+20) bytes, n_eval*(3d+1) flops) separately, live CUDA-event times."""
    out = {}
    for name, b, ms in (("filter", f_bytes, f_ms), ("scan", s_bytes, s_ms)):
        ach = b / world / (ms / 1e3) / 1e9 if ms > 0 else None
        out[name] = {"alg_bytes": b / world, "ms": ms, "achieved_gbs": ach,
                     "frac": ach / peak if ach else None,
                     "dram": ((tr or {}).get("kernels") or {}).get(name)}
    return out


def fp64_roofline(flops, world, s_ms, tr):
    """FP64 term of north_star's roofline: surviving distance evaluations x (3d+1)
    over the scan time, against the FP64 peak measured on the box (tools/fp64_peak)."""
    pk = None
    try:
        with open(os.path.join(ROOT, "profiles", "round2", "fp64_peak.json")) as f:
            pk = json.load(f)
    except Exception:
        pass
    ach = flops / world / (s_ms / 1e3) / 1e12 if s_ms > 0 else None
    peak = pk["tflops"] if pk else None
    return {"alg_flops": flops / world, "achieved_tflops": ach, "peak_tflops": peak,
            "peak_source": pk.get("how") if pk else None,
            "frac": (ach / peak) if (ach and peak) else None,
            "ncu": (tr or {}).get("fp64")}


def workload(cfg):
    from paper_1805_01208_b200.workloads import CONFIGS, GENERATORS

    c = CONFIGS[cfg]
    pts, w = GENERATORS[cfg](seed=0)
    return c, pts, w


def device_workload(cfg, dev):
    """(config, points (n,d) device view, weights or None, host-array getter)."""
    import torch

    from paper_1805_01208_b200.workloads import CONFIGS, c5_device

    c = CONFIGS[cfg]
    if cfg == "C5":
        X = c5_device(n=c["n"], seed=0, device=dev)       # (2, n) as generated
        # resident input in the reference's layout: a C-contiguous (n, 2) float64 array
        # (the same layout the e2e call copies from the host)
        pts_d = X.t().contiguous()
        del X
        torch.cuda.empty_cache()

        def host():
            h = torch.empty((c["n"], 2), dtype=torch.float64, pin_memory=True)
            h.copy_(pts_d)
            return h.numpy(), None
        return c, pts_d, None, host
    _, pts, w = workload(cfg)
    pts_d = torch.from_numpy(pts).to(dev)
    w_d = None if w is None else torch.from_numpy(w).to(dev)
    return c, pts_d, w_d, (lambda: (pts, w))


def cpu_inputs(cfg):
    """Bounded CPU-baseline input: the config itself (C1-C3), or for C4/C5 (hours to
    infeasible on the reference) the same recipe scaled down with the same points
    per block -- a labelled extrapolation, see the 'sample' string."""
    from paper_1805_01208_b200.workloads import CONFIGS, c4, c5_host

    if cfg == "C5":
        # the reference cannot run C5 (16 GiB input, days): same recipe at 1/1024 scale
        # with the same points per block (n/k = 65536)
        n = 1 << 20
        c = dict(CONFIGS["C5"], n=n, k=16)
        pts, w = c5_host(seed=0, n=n)
        return c, pts, w, ("EXTRAPOLATION: C5 recipe at 1/1024 scale (n=2^20, k=16: the same "
                           "65536 points/block)")
    if cfg == "C4":
        n = 1 << 20
        c = dict(CONFIGS["C4"], n=n, k=64)
        pts, w = c4(seed=0, n=n)
        return c, pts, w, ("EXTRAPOLATION: C4 recipe at 1/16 scale (n=2^20, k=64: the same "
                           "16384 points/block)")
    c, pts, w = workload(cfg)
    return c, pts, w, f"{cfg} input (full size)"


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_module():
    """The unmodified reference package installed by build() into baseline/_ref
    (pip --target, no network); None when it is not there."""
    if not os.path.isdir(os.path.join(REF_DIR, "geopart")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import geopart.kmeans as K

    return K


def ref_p(cfg, k):
    """The reference's faster rank count (SURVEY §8d "report the better of p=1 and
    p=256"): p=1 for small k, p=256 (per-rank box pruning) for large k."""
    return 1 if k <= 64 else 256


# ------------------------------------------------------------ CPU arm
def cpu_sample(cfg, budget_s=25.0):
    """One single-threaded run of the reference path on the config's (sample) input:
    the real reference package when installed (kind "reference"), else the oracle
    port (kind "port").  Full configs C1-C3 run completely; the scaled C4/C5 samples
    run their warm-up phase plus as many full iterations as fit the budget."""
    c, pts, w, what = cpu_inputs(cfg)
    K = reference_module()
    p = ref_p(cfg, c["k"])
    full = cfg == "C1"      # C2/C3 complete partitions take minutes: tools/ref_compare.py

    def once(max_iter):
        t0 = time.perf_counter()
        if K is not None:
            s = K.KMeansSettings(k=c["k"], epsilon=c["epsilon"], seed=0,
                                 **({} if full else {"max_iter": max_iter}))
            _, st = K.balanced_kmeans_points(pts, w, s, p=p, return_stats=True)
            dec = sum(r.total_decisions for r in st.iterations)
        else:
            from oracle import geographer_oracle as O

            kw = {} if full else {"max_iter": max_iter}
            r = O.run(pts, w, O.Knobs(k=c["k"], epsilon=c["epsilon"], seed=0, **kw),
                      scan_chunks=p)
            dec = sum(rec["total_decisions"] for rec in r.records)
        return dec, time.perf_counter() - t0

    iters = 1
    dec, dt = once(iters)
    if not full and dt < budget_s / 3:
        iters = max(1, min(50, int(budget_s / max(dt, 1e-3))))
        dec, dt = once(iters)
    kind = "reference" if K is not None else "port"
    impl = ("geopart.kmeans.balanced_kmeans_points (unmodified reference, baseline/_ref)"
            if K is not None else "oracle numpy port (reference package not installed)")
    run = "complete partition" if full else f"warm-up phase + {iters} full iteration(s)"
    return dict(value=dec / dt / 1e9, unit="Gpt/s", cores=1, kind=kind,
                sample=f"{what}; {run}; {impl}, p={p}, single-threaded; "
                       f"{dec} point-assignments in {dt:.2f} s",
                seconds=dt)


def _cpu_worker(cfg, budget_s, barrier, queue):
    barrier.wait()
    r = cpu_sample(cfg, budget_s=budget_s)
    queue.put((r["value"] * 1e9 * r["seconds"], r["seconds"], r["sample"], r["kind"]))


def reference_workers():
    """Host threads the reference arm may use: every core this process may run on,
    bounded by memory (one C5 sample peaks at ~0.5 GB RSS; 1 GB is budgeted; a full
    C3 run ~3 GB)."""
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    try:
        import psutil

        mem = int(psutil.virtual_memory().available // (1 << 30)) // 4
    except Exception:
        mem = 8
    return max(1, min(cores, mem, 256))


def cpu_sample_parallel(cfg, workers, budget_s):
    """The reference's numpy path is single-threaded (one simulated rank after the
    other), so the most the host can do is run one independent sample per core:
    W processes start together, value = all their point-assignments / the slowest."""
    import multiprocessing as mp

    for v in ("OMP_NUM_THREADS", "MKL_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        os.environ[v] = "1"
    ctx = mp.get_context("spawn")
    barrier, queue = ctx.Barrier(workers), ctx.Queue()
    procs = [ctx.Process(target=_cpu_worker, args=(cfg, budget_s, barrier, queue))
             for _ in range(workers)]
    for p in procs:
        p.start()
    res = [queue.get() for _ in procs]
    for p in procs:
        p.join()
    dec = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return dict(value=dec / wall / 1e9, seconds=wall, cores=workers, kind=res[0][3],
                sample=f"{workers} concurrent single-threaded runs, each: {res[0][2]}")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1805_01208_b200.workloads import CONFIGS

    c = CONFIGS[args.config]     # the arm's workload; each step times a bounded sample of it
    workers = reference_workers()
    vals = []
    last = None
    for i in range(args.warmup + args.steps):
        s = cpu_sample_parallel(args.config, workers, budget_s=10.0)
        if i >= args.warmup:
            vals.append(s["value"])
            last = s
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": "point-assignments/s", "value": v, "unit": "Gpt/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": last["seconds"] * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SURVEY §8d recipe)",
        "config": {"workload": f"{args.config}: {DESCR[args.config]}", "n": int(c["n"]),
                   "d": int(c["d"]), "k": c["k"], "epsilon": c["epsilon"]},
        "cpu_baseline": {"value": v, "unit": "Gpt/s", "cores": last["cores"],
                         "kind": last["kind"], "sample": last["sample"]},
        "e2e": {"value": v, "unit": "Gpt/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------ result gate
def _torch_argmin(P, centers, infl, chunk=4096):
    """Exact weighted-Voronoi argmin with the reference's per-pair fp64 arithmetic
    (kmeans.py:157-159: diff, separately rounded squares summed in the einsum order,
    correctly rounded sqrt and division; one eager torch op per kernel, so nothing
    is contracted into FMA), first minimum on ties.  Independent of the product's
    kernels."""
    import torch

    from paper_1805_01208_b200.numerics import einsum_order3

    C = torch.from_numpy(np.ascontiguousarray(centers)).to(P.device)
    f = torch.from_numpy(np.ascontiguousarray(infl)).to(P.device)
    d = P.shape[1]
    order = [0, 1] if d == 2 else {0: [0, 1, 2], 1: [0, 2, 1], 2: [1, 2, 0]}[einsum_order3()]
    out = []
    for s in range(0, P.shape[0], chunk):
        p = P[s:s + chunk]
        sq = []
        for j in range(d):
            dj = p[:, None, j] - C[None, :, j]
            sq.append(dj * dj)
        q = sq[order[0]] + sq[order[1]]
        for j in order[2:]:
            q = q + sq[j]
        out.append(torch.argmin(torch.sqrt(q) / f[None, :], dim=1))
    return torch.cat(out)


def result_gate(pts_d, w_d, labels, stats, c, single):
    """Correctness of the benchmarked partition (SURVEY §8c for C5): final imbalance
    recomputed from the labels, the flags, and an exact-argmin audit of a random
    2^20-point subsample of the final state."""
    import torch

    from paper_1805_01208_b200.control import imbalance

    st = stats.final_state
    out = {"final_imbalance": float(imbalance(st.block_weights)),
           "balance_failed": bool(stats.balance_failed), "converged": bool(stats.converged),
           "iterations": len(stats.iterations), "epsilon": c["epsilon"]}
    if not single:
        return out
    n = labels.shape[0]
    w = (torch.ones(n, dtype=torch.float64, device=labels.device) if w_d is None
         else w_d.to(torch.float64))
    bw = torch.zeros(c["k"], dtype=torch.float64, device=labels.device)
    bw.index_add_(0, labels, w)
    out["labels_block_weights_match"] = bool(np.array_equal(bw.cpu().numpy(), st.block_weights))
    m = min(n, 1 << 20)
    ids = torch.from_numpy(np.sort(np.random.default_rng(11).choice(n, m, replace=False)))
    ids = ids.to(labels.device)
    P = pts_d[ids].contiguous()
    bad = int((_torch_argmin(P, st.centers, st.influence) != labels[ids]).sum().item())
    out["argmin_audit"] = {"sample_points": int(m), "mismatches": bad,
                           "checker": "torch fp64 brute force over all k (bench.py _torch_argmin)"}
    return out


# ------------------------------------------------------------------ GPU arm
def run_b200(args):
    import torch

    from paper_1805_01208_b200 import KMeansSettings, balanced_kmeans_points
    from paper_1805_01208_b200 import _native as N
    from paper_1805_01208_b200.kmeans import _Timer, partition_device, partition_distributed

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("GP_DIST_BACKEND", "nccl") != "nccl":
        local = 0  # test mode: every rank shares GPU 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("GP_DIST_BACKEND", "nccl")  # gloo: several ranks on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    c, pts_d, w_d, host_inputs = device_workload(args.config, dev)
    n, d = pts_d.shape
    settings = KMeansSettings(k=c["k"], epsilon=c["epsilon"], seed=0)
    rows = None
    if world > 1:
        # SFC-range sharding: each rank starts from its contiguous block of the input rows
        lo_r, hi_r = (rank * n) // world, ((rank + 1) * n) // world
        rows = slice(lo_r, hi_r)
        pts_d = pts_d[rows].contiguous()
        w_d = None if w_d is None else w_d[rows].contiguous()
        torch.cuda.empty_cache()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    N.reset_launch_count()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    last = {}

    def step(timer=None):
        last.clear()   # the previous labels are released before the next partition
        if world > 1:
            a, stats = partition_distributed(pts_d, w_d, settings, device=dev, timer=timer)
        else:
            a, stats = partition_device(pts_d, w_d, settings, device=dev, timer=timer)
        last["labels"] = a
        return stats

    for _ in range(args.warmup):
        step()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    times, decisions, timers = [], 0, []
    N.reset_launch_count()
    for _ in range(args.steps):
        flush.fill_(1)
        barrier()
        timer = _Timer()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        stats = step(timer)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
        timers.append((timer, stats))
        decisions += sum(r.total_decisions for r in stats.iterations)
    launches = N.launch_count()
    clk = clocks.stop()
    result = result_gate(pts_d, w_d, last["labels"], stats, c, rows is None)
    t_total = sum(times)
    if dist is not None:
        tt = torch.tensor([t_total], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total = float(tt.item())
        # the point-assignment counts in the stats are already global (all ranks agree)
    value = decisions / t_total / 1e9

    # roofline of the assign kernel
    wb = 0 if w_d is None else 8
    alg_bytes, kern_ms, flops = 0.0, 0.0, 0.0
    f_bytes, s_bytes, f_ms, s_ms = 0.0, 0.0, 0.0, 0.0
    for timer, stats in timers:
        kern_ms += timer.total_ms()
        fm, sm = timer.split_ms()
        f_ms += fm
        s_ms += sm
        for (nact, nscan, nev) in timer.rounds:
            alg_bytes += nact * (4 + 16 + wb) + nscan * (8 * d + 20)
            f_bytes += nact * (4 + 16 + wb)
            s_bytes += nscan * (8 * d + 20)
            flops += nev * (3 * d + 1)
    launches_assign = sum(len(t.events) for t, _ in timers)
    peak, peak_kind = load_peaks()
    # per-round counts in the stats are global: the per-GPU kernel roofline is the
    # global algorithmic bytes / world over this rank's kernel time
    achieved = alg_bytes / world / (kern_ms / 1e3) / 1e9 if kern_ms > 0 else None

    # end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        pts, w = host_inputs()
        if rows is not None:
            pts = pts[rows]
            w = None if w is None else w[rows]
        e2e_t = []
        for i in range(max(1, min(args.steps, 3)) + 1):
            flush.fill_(1)
            barrier()
            t0 = time.perf_counter()
            if world > 1:
                lab, st2 = partition_distributed(pts, w, settings, device=dev)
                lab_h = lab.cpu()
            else:
                part = None   # the previous result is consumed: its pinned buffer is reused
                part, st2 = balanced_kmeans_points(pts, w, settings, return_stats=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if dist is not None:
                tt = torch.tensor([dt], dtype=torch.float64, device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                dt = float(tt.item())
            if i > 0:
                e2e_t.append(dt)
            else:
                e2e_cold = dt   # includes the first pinned allocation of the result buffer
        dec1 = sum(r.total_decisions for r in st2.iterations)
        e2e = {"value": dec1 / statistics.mean(e2e_t) / 1e9, "unit": "Gpt/s",
               "h2d_bytes_per_step": int(pts.nbytes + (0 if w is None else w.nbytes)) * world,
               "d2h_bytes_per_step": int(c["n"] * 8), "partition_s": statistics.mean(e2e_t),
               "input_memory": "page-locked", "cold_first_call_s": e2e_cold}
        if world == 1 and not args.no_pageable:
            # the same call with a plain (pageable) numpy input, as the reference's callers
            # pass it: staged through pinned chunks inside the library (staging.py)
            pts_pg = np.array(pts, copy=True)
            w_pg = None if w is None else np.array(w, copy=True)
            del pts
            tp = []
            for i in range(2):
                flush.fill_(1)
                barrier()
                t0 = time.perf_counter()
                part = None
                part, st3 = balanced_kmeans_points(pts_pg, w_pg, settings, return_stats=True)
                torch.cuda.synchronize()
                tp.append(time.perf_counter() - t0)
            e2e["pageable"] = {"value": dec1 / min(tp) / 1e9, "partition_s": min(tp),
                               "input_memory": "pageable numpy (np.array copy)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample(args.config)
        cpu.pop("seconds", None)

    if rank == 0:
        tr = ncu_traffic(args.config)
        line = {
            "metric": "point-assignments/s", "value": value, "unit": "Gpt/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_total / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded SURVEY §8d recipe; paper meshes not available)",
            "config": {"workload": f"{args.config}: {DESCR[args.config]}", "n": int(n),
                       "d": int(d), "k": c["k"], "epsilon": c["epsilon"],
                       "parallelism": f"sfc-range shards x{world} (NCCL)" if world > 1
                       else "single",
                       "l2": "flushed (256 MiB write) between timed steps",
                       "partition_s": t_total / args.steps},
            "roofline": {"bound": "hbm", "kernel": "gp_assign_round",
                         "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
                         "traffic": (tr["dram_bytes_per_round"][0] if tr else None),
                         "traffic_alg_bytes": (tr["alg_bytes_per_round"][0] if tr else None),
                         "traffic_source": (f"one full-phase round (round {tr['rounds'][0]}) of "
                                            f"{args.config}: {tr['source']}" if tr else None),
                         "launches": launches_assign,
                         "avg_launch_us": kern_ms * 1e3 / max(launches_assign, 1),
                         "alg_bytes_per_launch": alg_bytes / max(launches_assign, 1),
                         "fp64_flops_per_launch": flops / max(launches_assign, 1),
                         "kernel_share_of_step": kern_ms / 1e3 / t_total,
                         # the two launches of every round, each on its own §8d bytes
                         "split": split_roofline(f_bytes, f_ms, s_bytes, s_ms, flops, world,
                                                 peak, tr),
                         "frac_dram": (tr or {}).get("frac_dram"),
                         "fp64": fp64_roofline(flops, world, s_ms, tr)},
            "result": result,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches // max(args.steps, 1) if launches else None,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
