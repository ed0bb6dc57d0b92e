"""Per-kernel DRAM traffic, duration and FP64 instruction counts of an ncu report.

    python tools/ncu_summary.py REPORT.ncu-rep [--json OUT.json --round-trace TRACE --round R]

With --json, writes the roofline evidence bench.py reads (profiles/round2/
ncu_traffic_C5.json): for the captured assign round R (filter + scan), each kernel's
DRAM bytes, ncu duration and DRAM fraction of the measured peak, the round's
algorithmic bytes (tools/round_trace.py) and the FP64 instruction counts.
"""
import csv
import io
import json
import re
import subprocess
import sys

FP64 = ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
        "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "sm__sass_thread_inst_executed_op_dadd_pred_on.sum")


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = dict(zip(h, row))
        res.append(d)
    return res, dict(zip(h, units))


def num(d, k, unit=None):
    v = d.get(k, "")
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x


def scale(v, u):
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1, "ms": 1, "s": 1e3,
                "nsecond": 1e-6}.get(u, 1)


def summarize(rep):
    rs, units = rows(rep)
    out = []
    for d in rs:
        name = d["Kernel Name"]
        ms = scale(num(d, "gpu__time_duration.sum"), units.get("gpu__time_duration.sum", "ms"))
        rd = scale(num(d, "dram__bytes_read.sum") or 0, units.get("dram__bytes_read.sum", "byte"))
        wr = scale(num(d, "dram__bytes_write.sum") or 0, units.get("dram__bytes_write.sum", "byte"))
        fp = {k.split("_op_")[1].split("_")[0]: num(d, k) for k in FP64 if k in d}
        out.append(dict(kernel=name, ms=ms, dram_read=rd, dram_write=wr, fp64=fp))
    return out


def main():
    rep = sys.argv[1]
    ks = summarize(rep)
    peak = 6541.1
    try:
        peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
    except Exception:
        pass
    for k in ks:
        gbs = (k["dram_read"] + k["dram_write"]) / (k["ms"] * 1e-3) / 1e9 if k["ms"] else 0
        print(f"{k['kernel'][:60]:60s} {k['ms']:9.3f} ms  dram {(k['dram_read'] + k['dram_write']) / 1e9:7.3f} GB"
              f"  {gbs:7.0f} GB/s ({gbs / peak:.2f} of peak)")
    if "--json" in sys.argv:
        out = sys.argv[sys.argv.index("--json") + 1]
        trace = sys.argv[sys.argv.index("--round-trace") + 1]
        rnd = int(sys.argv[sys.argv.index("--round") + 1])
        alg = {}
        for line in open(trace):
            m = re.match(r"round (\d+) active (\d+) scanned (\d+) evals (\d+) filter_alg_bytes (\d+) "
                         r"scan_alg_bytes (\d+) flops (\d+)", line)
            if m and int(m.group(1)) == rnd:
                alg = dict(active=int(m.group(2)), scanned=int(m.group(3)), evals=int(m.group(4)),
                           filter_alg_bytes=int(m.group(5)), scan_alg_bytes=int(m.group(6)),
                           flops=int(m.group(7)))
        kern = {}
        for k in ks:
            key = "filter" if "filter_kernel" in k["kernel"] else (
                "scan" if ("scan_kernel" in k["kernel"] or "walk_kernel" in k["kernel"]) else None)
            if key is None:
                continue
            dram = k["dram_read"] + k["dram_write"]
            kern[key] = dict(kernel=k["kernel"], ncu_ms=k["ms"], dram_bytes=dram,
                             dram_gbs=dram / (k["ms"] * 1e-3) / 1e9,
                             frac_dram=dram / (k["ms"] * 1e-3) / 1e9 / peak,
                             alg_bytes=alg.get(key + "_alg_bytes"), fp64_inst=k["fp64"])
        tot_dram = sum(v["dram_bytes"] for v in kern.values())
        tot_ms = sum(v["ncu_ms"] for v in kern.values())
        sc = kern.get("scan", {}).get("fp64_inst") or {}
        fp64_flops = (2 * (sc.get("dfma") or 0) + (sc.get("dmul") or 0) + (sc.get("dadd") or 0))
        res = {
            "kernel": "gp_assign_round = filter_kernel + scan_kernel (one full-phase balance round)",
            "config": "C5", "rounds": [rnd],
            "dram_bytes_per_round": [tot_dram],
            "alg_bytes_per_round": [(alg.get("filter_alg_bytes") or 0) + (alg.get("scan_alg_bytes") or 0)],
            "ncu_ms_per_round": [tot_ms],
            "frac_dram": tot_dram / (tot_ms * 1e-3) / 1e9 / peak,
            "peak_gbs": peak, "kernels": kern, "round": alg,
            "fp64": {"scan_sass_flops": fp64_flops,
                     "scan_tflops": fp64_flops / (kern.get("scan", {}).get("ncu_ms", 1) * 1e-3) / 1e12,
                     "alg_flops": alg.get("flops"),
                     "note": "SASS dfma counted as 2 flops; includes the bound, candidate and "
                             "prefilter arithmetic, not only the surviving evaluations"},
            "source": f"{rep} (ncu --set full --clock-control none, NVTX range round{rnd} of "
                      f"tools/one_partition.py C5; algorithmic bytes from tools/round_trace.py)",
        }
        with open(out, "w") as f:
            json.dump(res, f, indent=1)
        print("wrote", out)


if __name__ == "__main__":
    main()
