#!/usr/bin/env python
"""Record ncu per-launch traffic of the bench kernel in profiles/traffic.json.

  python tools/traffic_record.py <key> <source_sha> <csv-or-ncu-rep>... [--note TEXT]

`key` is bench.py's traffic key `<kernel>:<algo>:<n>:<dtype>:<count>:<nvlink|virtual>`;
`source_sha` is `bench.source_sha()` printed ON THE GPU BOX next to the
capture (so the record is tied to the sources that were profiled, and
bench.py reports it as stale once the kernels change).  Inputs: `ncu --csv
--log-file` metric lists (tools/ncu_rank0.sh) or `--set full` reports.
Recognised metrics: dram__bytes_{read,write}.sum -> dram_bytes,
nvltx__bytes.sum -> nvltx_bytes, nvlrx__bytes.sum -> nvlrx_bytes,
gpu__time_duration.sum -> duration_s.
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1}


def metrics_from_csv(path: str) -> dict:
    """{metric: value in base units} from an `ncu --csv` metric list (one
    launch: -c 1); sums if several rows name the same metric."""
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ni, ui, vi = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    out = {}
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1)
        out[r[ni]] = out.get(r[ni], 0.0) + v
    return out


def metrics_from_rep(path: str) -> dict:
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for k, u, v in zip(hdr, units, vals):
        try:
            out[k] = float(v.replace(",", "")) * UNIT.get(u, 1)
        except ValueError:
            pass
    return out


KERNEL_OF = {"flat": "hfr_flat_tma_kernel", "dbt": "hfr_tree_kernel", "pair_dbt": "hfr_tree_kernel",
             "nvls": "hfr_nvls_kernel"}


def record_from_pm(path: str):
    """profiles/traffic.json entries from a tools/pm_nvlink.py result (CUPTI
    PM sampling over K launches at N>1): rank 0's bytes per launch, keyed like
    bench.py's N>1 roofline (`<kernel>:<algo>:<n>:<dtype>:<count>:nvlink`)."""
    d = json.loads(open(path).read().strip().splitlines()[-1])
    r0 = d["ranks"][0]
    pl = r0["per_launch"]
    key = f"{KERNEL_OF.get(r0['algo'], r0['algo'])}:{r0['algo']}:{r0['n']}:{r0['dtype']}:{r0['count']}:nvlink"
    rec = {"source": os.path.relpath(path, ROOT) + " (CUPTI PM sampling, tools/pm_nvlink.py, rank 0, "
                      f"{r0['steps']} launches)", "source_sha": r0["source_sha"],
           "nvltx_bytes": pl.get("nvltx__bytes.sum"), "nvlrx_bytes": pl.get("nvlrx__bytes.sum"),
           "nvltx_user_bytes": pl.get("nvltx__bytes_data_user.sum"),
           "nvlrx_user_bytes": pl.get("nvlrx__bytes_data_user.sum"),
           "dram_bytes": (pl.get("dram__bytes_read.sum") or 0) + (pl.get("dram__bytes_write.sum") or 0)}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    traffic[key] = rec
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)
    print(key, json.dumps(rec))


def main():
    args = sys.argv[1:]
    if args and args[0] == "--from-pm":
        for p in args[1:]:
            record_from_pm(p)
        return
    note = None
    if "--note" in args:
        i = args.index("--note")
        note = args[i + 1]
        del args[i:i + 2]
    key, sha, srcs = args[0], args[1], args[2:]
    m = {}
    for p in srcs:
        m.update(metrics_from_rep(p) if p.endswith(".ncu-rep") else metrics_from_csv(p))
    rec = {"source": " + ".join(os.path.relpath(p, ROOT) for p in srcs), "source_sha": sha}
    if "dram__bytes_read.sum" in m and "dram__bytes_write.sum" in m:
        rec["dram_bytes"] = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    for k, name in (("nvltx__bytes.sum", "nvltx_bytes"), ("nvlrx__bytes.sum", "nvlrx_bytes"),
                    ("nvltx__bytes_data_user.sum", "nvltx_user_bytes"), ("nvlrx__bytes_data_user.sum", "nvlrx_user_bytes"),
                    ("gpu__time_duration.sum", "duration_s")):
        if k in m:
            rec[name] = m[k]
    if note:
        rec["note"] = note
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    old = traffic.get(key)
    if isinstance(old, dict) and old.get("source_sha") == sha:
        # same sources: merge (DRAM and NVLink come from separate single-pass runs)
        src = old.get("source", "")
        old.update(rec)
        if src and src not in old["source"]:
            old["source"] = src + " + " + old["source"]
        rec = old
    traffic[key] = rec
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)
    print(key, json.dumps(rec))


if __name__ == "__main__":
    main()
