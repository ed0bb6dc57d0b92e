"""Throughput of the formats and metrics either side of the path.

    python tools/graphio_bench.py [--side 4096] [--cpu-side 256] [--out FILE]

Workload: a side x side 2D grid mesh (n = side^2 vertices, ~2n edges) as a METIS file
plus its coordinate file, tiles of 128 x 128 vertices as the partition.  The METIS text
is produced on the device (this tool's own use of gp_format_ints); timings:

  * load_metis_graph / load_coords / read_partition / write_partition end to end from a
    file on disk (page cache) to numpy arrays, and the device part alone (CUDA events);
  * evaluate(graph, partition) and each metric kernel;
  * a per-kernel device-time table (torch.profiler / CUPTI) of one load + one evaluate;
  * the CPU baseline: the unmodified reference (baseline/_ref) or, without it, the CPU
    oracle, on a cpu-side x cpu-side grid (bounded sample), one core.
"""
import argparse
import io
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1805_01208_b200 import _native as N  # noqa: E402
from paper_1805_01208_b200 import fileio, metrics  # noqa: E402
from paper_1805_01208_b200.types import Partition  # noqa: E402


def grid_csr_device(side):
    """CSR (offsets, neighbors) of the side x side grid on the device, rows sorted."""
    n = side * side
    v = torch.arange(n, device="cuda", dtype=torch.int64)
    x, y = v % side, v // side
    cand = torch.stack([v - side, v - 1, v + 1, v + side], 1)
    ok = torch.stack([y > 0, x > 0, x < side - 1, y < side - 1], 1)
    deg = ok.sum(1)
    off = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    off[1:] = torch.cumsum(deg, 0)
    return n, off, cand[ok], ok


def metis_text_device(n, off, nbrs):
    """METIS text of an unweighted CSR graph, formatted by gp_format_ints (one id per
    'line'), then every separator that is not a row end turned into a blank."""
    sh = torch.cuda.current_stream().cuda_stream
    ids = (nbrs + 1).contiguous()
    m = int(ids.shape[0])
    wsb = N.size_query("gp_format_ints_workspace_bytes", m)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    total = torch.empty(1, dtype=torch.int64, device="cuda")
    N.call("gp_format_ints_plan", ids.data_ptr(), m, total.data_ptr(), ws.data_ptr(), wsb, sh)
    out = torch.empty(int(total.item()), dtype=torch.uint8, device="cuda")
    N.call("gp_format_ints_write", ids.data_ptr(), m, out.data_ptr(), ws.data_ptr(), sh)
    lens = torch.ones(m, dtype=torch.int64, device="cuda") + 1
    for p in range(1, 11):
        lens += (ids >= 10 ** p).to(torch.int64)
    ends = torch.cumsum(lens, 0) - 1           # byte of every separator
    row_end = torch.zeros(m, dtype=torch.bool, device="cuda")
    row_end[off[1:] - 1] = True
    out[ends[~row_end]] = 32
    head = f"% {n} vertex grid\n{n} {m // 2}\n".encode()
    return head + out.cpu().numpy().tobytes()


def cuda_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def wall(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def kernel_table(fn, top=16):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    rows = {}
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        r = rows.setdefault(e.name[:64], [0, 0.0])
        r[0] += 1
        r[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    tot = sum(v[1] for v in rows.values())
    tab = [{"kernel": k, "calls": v[0], "ms": round(v[1] / 1e3, 3),
            "share": round(v[1] / tot, 3)} for k, v in
           sorted(rows.items(), key=lambda x: -x[1][1])[:top]]
    return {"device_ms": round(tot / 1e3, 2), "kernels": tab}


def cpu_baseline(side):
    """The reference (or the oracle port) on a side x side grid, one core."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    n, off, nbrs, _ = grid_csr_device(side)
    text = metis_text_device(n, off, nbrs).decode()
    xs = np.arange(n) % side
    ys = np.arange(n) // side
    ctext = "".join(f"{x} {y}\n" for x, y in zip(xs, ys))
    lab = (ys // 64) * ((side + 63) // 64) + xs // 64
    k = int(lab.max()) + 1
    res = {"n": n, "k": k, "cores": 1}
    if os.path.isdir(os.path.join(ref, "geopart")):
        sys.path.insert(0, ref)
        from geopart import fileio as RF
        from geopart import metrics as RM
        from geopart.graph import Partition as RP

        res["kind"] = "reference"
        t0 = time.perf_counter()
        g = RF.load_metis_graph(io.StringIO(text), io.StringIO(ctext))
        res["load_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        rep = RM.evaluate(g, RP(assignment=lab, k=k))
        res["evaluate_s"] = time.perf_counter() - t0
        res["edge_cut"] = rep.edge_cut
    else:
        from oracle import graphio_oracle as O

        res["kind"] = "port"
        t0 = time.perf_counter()
        o, nb, vw, ew = O.parse_metis(text)
        O.coords_of(ctext)
        res["load_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        rep = O.report(o, nb, vw, ew, lab, k)
        res["evaluate_s"] = time.perf_counter() - t0
        res["edge_cut"] = rep["edge_cut"]
    res["load_bytes"] = len(text) + len(ctext)
    res["load_MBps"] = res["load_bytes"] / res["load_s"] / 1e6
    res["evaluate_Medges_per_s"] = (len(nbrs) // 2) / res["evaluate_s"] / 1e6
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=4096)
    ap.add_argument("--cpu-side", type=int, default=256)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    side = args.side
    n, off, nbrs, _ = grid_csr_device(side)
    text = metis_text_device(n, off, nbrs)
    xs, ys = np.arange(n) % side, np.arange(n) // side
    pts = np.stack([xs * 0.125 + 0.1, ys * 0.3 - 7.7], 1)
    tiles = (side + 127) // 128
    lab = (ys // 128) * tiles + xs // 128
    k = int(lab.max()) + 1
    tmp = tempfile.mkdtemp(prefix="graphio_bench_")
    gpath, cpath, ppath = (os.path.join(tmp, f) for f in ("g.graph", "g.xyz", "g.part"))
    with open(gpath, "wb") as f:
        f.write(text)
    nc = min(n, 1 << 21)            # np.savetxt is slow: the coordinate file holds 2^21 rows
    s = io.StringIO()
    np.savetxt(s, pts[:nc], fmt="%.17g")
    ctext = s.getvalue().encode()
    with open(cpath, "wb") as f:
        f.write(ctext)
    res = {"workload": f"{side}x{side} grid mesh, {tiles}x{tiles} tiles", "n": n,
           "edges": int(nbrs.shape[0]) // 2, "k": k, "graph_bytes": len(text),
           "coords_bytes": len(ctext)}
    del nbrs, off
    torch.cuda.empty_cache()

    # --- readers
    t = wall(lambda: fileio.load_metis_graph(gpath))
    res["load_metis_graph"] = {"s": t, "GBps": len(text) / t / 1e9, "what":
                               "file (page cache) -> validated GeometricGraph in numpy arrays"}
    t = wall(lambda: fileio.load_coords(cpath, expect_n=nc))
    res["load_coords"] = {"s": t, "rows": nc, "GBps": len(ctext) / t / 1e9,
                          "Mvalues_per_s": 2 * nc / t / 1e6}
    c = fileio.load_coords(cpath, expect_n=nc)
    assert c.tobytes() == pts[:nc].tobytes(), "coords differ from what was written"
    g = fileio.load_metis_graph(gpath)
    part = Partition(assignment=lab, k=k)
    # the device part of the tokenizer alone
    buf = torch.from_numpy(np.frombuffer(text, dtype=np.uint8).copy()).cuda()
    sh = torch.cuda.current_stream().cuda_stream
    L = int(buf.shape[0])
    wsb = N.size_query("gp_text_index_workspace_bytes", L)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    counts = torch.empty(3, dtype=torch.int64, device="cuda")
    N.call("gp_text_index", buf.data_ptr(), L, 0, counts.data_ptr(), ws.data_ptr(), wsb, sh)
    nl, nt, _ = (int(v) for v in counts.cpu().tolist())
    lo = torch.empty(nl + 1, dtype=torch.int64, device="cuda")
    lt = torch.empty(nl + 1, dtype=torch.int64, device="cuda")
    tv = torch.empty(nt, dtype=torch.int64, device="cuda")
    tk = torch.empty(nt, dtype=torch.uint8, device="cuda")
    t1 = cuda_time(lambda: N.call("gp_text_index", buf.data_ptr(), L, 0, counts.data_ptr(),
                                  ws.data_ptr(), wsb, sh))
    t2 = cuda_time(lambda: N.call("gp_text_tokens", buf.data_ptr(), L, 0, ws.data_ptr(), nl, nt,
                                  lo.data_ptr(), lt.data_ptr(), tv.data_ptr(), tk.data_ptr(), sh))
    alg = 2 * L + 9 * nt + 16 * nl     # text read twice; value + kind per token; two line arrays
    res["tokenizer"] = {"index_ms": t1 * 1e3, "tokens_ms": t2 * 1e3, "tokens": nt, "lines": nl,
                        "text_GBps": L / (t1 + t2) / 1e9, "alg_bytes": alg,
                        "alg_GBps": alg / (t1 + t2) / 1e9}
    del buf, lo, lt, tv, tk, ws
    # --- writer
    t = wall(lambda: fileio.write_partition(part, ppath))
    res["write_partition"] = {"s": t, "Mlines_per_s": n / t / 1e6}
    t = wall(lambda: fileio.read_partition(ppath, expect_n=n))
    res["read_partition"] = {"s": t, "Mlines_per_s": n / t / 1e6}
    assert np.array_equal(fileio.read_partition(ppath, expect_n=n).assignment, lab)
    # --- metrics
    dg = metrics.DeviceGraph(g, part)
    res["evaluate"] = {"s": wall(lambda: metrics.evaluate(g, part), reps=2),
                       "what": "numpy graph + labels -> full report (5 BFS sweeps of all blocks)"}
    for name, fn in (("edge_cut", lambda: metrics.edge_cut(dg, part)),
                     ("comm_volumes", lambda: metrics.comm_volumes(dg, part)),
                     ("block_weights", lambda: metrics.block_weights(dg, part)),
                     ("block_diameter_lower_bounds",
                      lambda: metrics.block_diameter_lower_bounds(dg, part))):
        t = cuda_time(fn, reps=2)
        res[name] = {"ms": t * 1e3, "Gedges_per_s": g.m / t / 1e9}
    rep = metrics.evaluate(g, part)
    th = 128
    want_cut = 2 * (tiles - 1) * side if side % th == 0 else None
    res["check"] = {"edge_cut": rep.edge_cut, "expected_cut": want_cut,
                    "diameter_max": max(rep.block_diameters), "imbalance": rep.imbalance}
    if want_cut is not None:
        assert rep.edge_cut == want_cut and max(rep.block_diameters) == 2 * (th - 1)
    res["profile_load"] = kernel_table(lambda: fileio.load_metis_graph(gpath))
    res["profile_evaluate"] = kernel_table(lambda: metrics.evaluate(g, part))
    res["cpu_baseline"] = cpu_baseline(args.cpu_side)
    cb = res["cpu_baseline"]
    res["speedup_vs_cpu"] = {
        "load": (res["load_metis_graph"]["GBps"] * 1e3) / cb["load_MBps"],
        "evaluate": (g.m / res["evaluate"]["s"] / 1e6) / cb["evaluate_Medges_per_s"],
        "note": "GPU at the full size vs one CPU core on the bounded sample, per byte / per edge",
    }
    print(json.dumps(res, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)
    for p in (gpath, cpath, ppath):
        os.remove(p)
    os.rmdir(tmp)


if __name__ == "__main__":
    main()
