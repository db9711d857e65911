#!/usr/bin/env python
"""Summaries of ncu outputs for profiles/: launch-list shares and key metrics of a --set full capture.

  python tools/ncu_summary.py launches gpurun_out/launches.csv
  python tools/ncu_summary.py full gpurun_out/prof_flux.ncu-rep
  python tools/ncu_summary.py traffic gpurun_out/full.ncu-rep "tgv 128x128x128 cgks5-linear" > profiles/ncu_traffic.json

The traffic mode writes the measured DRAM bytes (read + write) per launch of each library kernel
of a --set full capture, keyed by the bench's kernel names; bench.py reports it as roofline.traffic
for the dominant kernel when the workload matches.
"""
import json
import re
import collections
import csv
import io
import subprocess
import sys

UNITS = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3,
         "second": 1e3}

KEYS = [
    "gpu__time_duration.sum",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sass__inst_executed_local_loads",
    "sass__inst_executed_local_stores",
    "smsp__inst_executed.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        ms = float(r[vi].replace(",", "")) * UNITS.get(r[ui], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(a[1] for a in agg.values())
    out = [f"{'kernel':58s} {'launches':>8s} {'total_ms':>10s} {'ms/launch':>10s} {'share':>7s}"]
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:58s} {n:8d} {ms:10.3f} {ms / n:10.4f} {ms / tot * 100:6.1f}%")
    out.append(f"{'TOTAL':58s} {'':8s} {tot:10.3f}")
    return "\n".join(out)


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1])) if len(rows) > 2 else {}
    out = []
    for vals in rows[2:] if len(rows) > 2 else rows[1:]:
        d = dict(zip(hdr, vals))
        out.append(f"kernel: {d.get('Kernel Name', '?')}")
        for k in KEYS:
            if k in d:
                out.append(f"  {k} = {d[k]} {units.get(k, '')}".rstrip())
        stalls = sorted(((float(v), h) for h, v in d.items()
                         if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")
                         and v.replace(".", "", 1).isdigit()), reverse=True)[:6]
        for v, h in stalls:
            out.append(f"  stall {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} = {v:.3f}")
        try:
            fl = 2 * float(d["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]) + \
                float(d["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]) + \
                float(d["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"])
            t = float(d["gpu__time_duration.sum"]) * 1e-9
            out.append(f"  executed DP flops = {fl:.4g}  ->  {fl / t / 1e12:.2f} TFLOP/s over the launch")
        except Exception:
            pass
    return "\n".join(out)


BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def bench_name(kernel):
    m = re.search(r"k_flux1?<(\d+), (\d+), \d+, \d+, \d+, \d+(?:, (\d+))?>", kernel)
    if m:  # the 7th template argument (TONLY) marks the second-stage sweeps
        return "flux_" + "xyz"[int(m.group(2))] + ("_t" if m.group(3) == "1" else "")
    for k in ("recon5", "recon2", "update", "dt_finalize", "dt", "step_end", "pack", "unpack"):
        if "k_" + k + "<" in kernel or kernel.startswith("k_" + k) or "::k_" + k in kernel:
            return k
    return None


def traffic(path, workload):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    per = {}
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        name = bench_name(d.get("Kernel Name", ""))
        if name is None:
            continue
        b = sum(float(d[k].replace(",", "")) * BYTES.get(units.get(k, "byte"), 1.0)
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        per.setdefault(name, []).append(b)
    return json.dumps({"workload": workload, "source": path.split("/")[-1],
                       "metric": "dram__bytes_read.sum + dram__bytes_write.sum per launch (ncu --set full)",
                       "per_launch_bytes": {k: sum(v) / len(v) for k, v in per.items()}}, indent=1)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "traffic":
        print(traffic(path, sys.argv[3]))
    else:
        print(launches(path) if mode == "launches" else full(path))
