#!/usr/bin/env python
"""Turn ncu captures in gpurun_out/ into committed summaries under profiles/.

  python tools/ncu_summary.py <tag> <report.ncu-rep>[=traffic_key]... [--launches launches.csv]

For each --set full report: key raw metrics (duration, DRAM bytes, throughput,
occupancy, registers) and the stall-reason breakdown -> profiles/<tag>_<name>.txt,
For a launch list: per-kernel count / total / share.  (Per-launch traffic for
bench.py's roofline.traffic is recorded by tools/traffic_record.py, tied to
the source hash of the profiled build.)
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "smsp__inst_executed.sum"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1}


def ncu(*args) -> str:
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (r[i], units[i])
        out.append(d)
    return out


def si(val_unit):
    v, u = val_unit
    try:
        return float(v.replace(",", "")) * UNIT.get(u, 1)
    except ValueError:
        return None


def stalls(rep) -> str:
    src = ncu("-i", rep, "--page", "source", "--csv")
    tmp = os.path.join("/tmp", os.path.basename(rep) + ".src.csv")
    open(tmp, "w").write(src)
    return subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_stalls.py"), tmp, "12"],
                          capture_output=True, text=True).stdout


def main():
    tag = sys.argv[1]
    args = sys.argv[2:]
    launches = None
    if "--launches" in args:
        i = args.index("--launches")
        launches = args[i + 1]
        del args[i:i + 2]
    os.makedirs(PROF, exist_ok=True)
    for spec in args:
        rep = spec.partition("=")[0]
        name = os.path.basename(rep).replace(".ncu-rep", "")
        lines = [f"# ncu --set full summary: {rep} ({tag})"]
        for d in raw(rep):
            lines.append(f"kernel: {d['kernel']}")
            for k in KEYS:
                if k in d:
                    lines.append(f"  {k:62s} {d[k][0]:>14s} {d[k][1]}")
            rd, wr = si(d.get("dram__bytes_read.sum", ("", ""))), si(d.get("dram__bytes_write.sum", ("", "")))
            if rd is not None and wr is not None:
                lines.append(f"  dram read+write per launch: {rd + wr:.4e} B")
        lines.append("")
        lines.append(stalls(rep))
        open(os.path.join(PROF, f"{tag}_{name}.txt"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
    if launches:
        rows = [r for r in csv.reader(open(launches)) if r and not r[0].startswith("==")]
        hdr = rows[0]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        agg = {}
        for r in rows[1:]:
            if len(r) != len(hdr):
                continue
            agg.setdefault(r[ki], []).append(float(r[vi]))
        tot = sum(sum(v) for v in agg.values())
        out = [f"# ncu launch list (gpu__time_duration.sum, cold-cache, serialised): {launches} ({tag})",
               f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'mean_us':>10s} {'share':>7s}"]
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            out.append(f"{k[:60]:60s} {len(v):8d} {sum(v) / 1e3:12.1f} {sum(v) / len(v) / 1e3:10.1f} {sum(v) / tot:7.1%}")
        open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(out) + "\n")
        print("\n".join(out))


if __name__ == "__main__":
    main()
