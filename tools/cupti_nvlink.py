#!/usr/bin/env python
"""NVLink / DRAM bytes of the FLAT allreduce at N>1 without kernel replay.

  torchrun --nproc-per-node N tools/cupti_nvlink.py [--steps K] [--out DIR]

ncu could not profile a multi-rank run (profiles/r02/ncu_multirank_attempts.txt).
This uses CUPTI's range profiler through PyTorch's Kineto
(torch.profiler with _ExperimentalConfig(profiler_metrics=...,
profiler_measure_per_kernel=False)): the counters are collected over one
user range covering K back-to-back C2 allreduces, a single pass, so no
kernel is ever replayed and the ranks' kernels pair up as usual.  Each rank
writes its Chrome trace and the metric values found in it; rank 0 prints a
JSON line with the per-launch bytes next to the algorithmic ones
(2(n-1)/n * S per direction for FLAT).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = ["nvltx__bytes.sum", "nvlrx__bytes.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]


def find_metrics(obj, out):
    """every numeric value whose key names one of METRICS, anywhere in the trace"""
    if isinstance(obj, dict):
        for k, v in obj.items():
            if any(m.split(".")[0] in str(k) for m in METRICS) and isinstance(v, (int, float)):
                out.setdefault(str(k), []).append(float(v))
            else:
                find_metrics(v, out)
    elif isinstance(obj, list):
        for v in obj:
            find_metrics(v, out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--out", default="gpurun_out/cupti_nvlink")
    ap.add_argument("--metrics", default=",".join(METRICS))
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    from torch._C._profiler import _ExperimentalConfig

    import paper_2408_14158_b200 as hfr
    from paper_2408_14158_b200 import _build
    _build.build()
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    comm = hfr.Comm.init(device=local, config=hfr.Config(algo="flat", scale=1.0 / world, timeout_ms=60000))
    count = (186 << 20) // 4
    t = comm.empty(count, torch.float32)
    t.normal_()
    for _ in range(3):
        comm.allreduce(t)
    torch.cuda.synchronize()
    dist.barrier()
    metrics = a.metrics.split(",")
    cfg = _ExperimentalConfig(profiler_metrics=metrics, profiler_measure_per_kernel=False)
    os.makedirs(a.out, exist_ok=True)
    trace = os.path.join(a.out, f"rank{rank}.json")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA],
                                experimental_config=cfg) as prof:
        for _ in range(a.steps):
            comm.allreduce(t)
        torch.cuda.synchronize()
    prof.export_chrome_trace(trace)
    found = {}
    find_metrics(json.load(open(trace)), found)
    S = count * 4
    rec = {"rank": rank, "n": world, "steps": a.steps, "metrics": {k: sum(v) for k, v in found.items()},
           "per_launch": {k: sum(v) / a.steps for k, v in found.items()},
           "algorithmic_nvlink_bytes_per_dir_per_launch": 2.0 * (world - 1) / world * S,
           "algorithmic_dram_bytes_per_launch": 2.0 * S, "status": hfr.status_string(comm.status())}
    with open(os.path.join(a.out, f"rank{rank}_metrics.json"), "w") as f:
        json.dump(rec, f, indent=1)
    all_recs = [None] * world
    dist.all_gather_object(all_recs, rec)
    if rank == 0:
        print(json.dumps({"tool": "cupti_nvlink", "ranks": all_recs}), flush=True)
    comm.finalize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
