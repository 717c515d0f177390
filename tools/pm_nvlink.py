#!/usr/bin/env python
"""NVLink / DRAM bytes of the FLAT allreduce at N>1 from CUPTI PM sampling.

  torchrun --nproc-per-node N tools/pm_nvlink.py [--steps K] [--out FILE]

tools/pm_sampler.cu (built here into tools/libpm_sampler.so) samples the
GPU's performance monitors at a fixed interval while K back-to-back C2
allreduces run — no kernel replay, so the ranks' kernels pair up as in the
bench.  Each rank samples its own GPU; the counters summed over the window
and divided by K give bytes per launch, next to the algorithmic ones
(FLAT: 2(n-1)/n * S per direction over NVLink, S read + S written in HBM).
The metric names are picked from the device's PM-sampling base metrics
(nvltx/nvlrx bytes, dram read/write bytes).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SRC = os.path.join(ROOT, "tools", "pm_sampler.cu")
LIB = os.path.join(ROOT, "tools", "libpm_sampler.so")
WANT = [r"^nvltx__bytes$", r"^nvlrx__bytes$", r"^nvltx__bytes_data_user$", r"^nvlrx__bytes_data_user$",
        r"^dram__bytes_read$", r"^dram__bytes_write$"]


def lib():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-O2", "-shared", "-Xcompiler", "-fPIC", "-o", LIB, SRC,
                        "-L/usr/local/cuda/lib64", "-lcupti", "-lcuda"], check=True, capture_output=True)
    L = ctypes.CDLL(LIB)
    L.pm_query_metrics.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t]
    L.pm_start.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.c_uint64, ctypes.c_uint64]
    L.pm_series.argtypes = [ctypes.c_char_p]
    L.pm_stop.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.POINTER(ctypes.c_uint64),
                          ctypes.POINTER(ctypes.c_uint64)]
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--interval", type=int, default=20000, help="sampling interval (GPU sysclk cycles)")
    ap.add_argument("--out", default="")
    ap.add_argument("--algo", default="flat")
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--series", default="", help="per-sample CSV prefix (rank r writes <prefix>_rank<r>.csv)")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2408_14158_b200 as hfr
    from paper_2408_14158_b200 import _build
    _build.build()
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    L = lib() if local == 0 else None
    dist.barrier()
    L = L or lib()
    buf = ctypes.create_string_buffer(1 << 20)
    nq = L.pm_query_metrics(local, buf, len(buf))
    base = buf.value.decode().split()
    picked = [m for m in base if any(re.match(w, m) for w in WANT)]
    metrics = [m + ".sum" for m in picked]
    nvls = (200 << 20) if a.algo == "nvls" else 0
    comm = hfr.Comm.init(device=local, config=hfr.Config(algo=a.algo, scale=1.0 / world, timeout_ms=60000,
                                                         nvls_bytes=nvls))
    esz = 2 if a.dtype == "bf16" else 4
    count = (186 << 20) // esz
    t = comm.empty(count, torch.bfloat16 if a.dtype == "bf16" else torch.float32)
    t.normal_()
    for _ in range(3):
        comm.allreduce(t)
    torch.cuda.synchronize()
    dist.barrier()
    comm.barrier()
    torch.cuda.synchronize()
    import bench
    res = {"rank": rank, "n": world, "algo": a.algo, "dtype": a.dtype, "count": count, "steps": a.steps,
           "query_count": nq, "metrics": metrics, "source_sha": bench.source_sha()}
    if metrics:
        if a.series:
            L.pm_series(f"{a.series}_rank{rank}.csv".encode())
        rc = L.pm_start(local, ",".join(metrics).encode(), a.interval, 1 << 16)
        res["start_rc"] = rc
        if rc == 0:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                comm.allreduce(t)
            e1.record()
            torch.cuda.synchronize()
            sums = (ctypes.c_double * len(metrics))()
            t0, t1 = ctypes.c_uint64(), ctypes.c_uint64()
            ns = L.pm_stop(sums, len(metrics), ctypes.byref(t0), ctypes.byref(t1))
            res.update({"samples": ns, "window_ns": t1.value - t0.value, "timed_ms": e0.elapsed_time(e1),
                        "sum": dict(zip(metrics, list(sums))),
                        "per_launch": {m: v / a.steps for m, v in zip(metrics, list(sums))}})
    S = count * esz
    res["algorithmic_per_launch"] = {"nvlink_bytes_per_direction": bench.variant_dir_bytes(hfr, a.algo, world, S, esz)
                                     if a.algo != "flat" else 2.0 * (world - 1) / world * S, "dram_bytes": 2.0 * S}
    res["status"] = hfr.status_string(comm.status())
    allr = [None] * world
    dist.all_gather_object(allr, res)
    if rank == 0:
        line = json.dumps({"tool": "pm_nvlink", "ranks": allr})
        print(line, flush=True)
        if a.out:
            with open(a.out, "w") as f:
                f.write(line + "\n")
    comm.finalize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
