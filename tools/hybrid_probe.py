#!/usr/bin/env python
"""Probe (not a product path): can NVLS and FLAT share the links?

  torchrun --nproc-per-node N tools/hybrid_probe.py [--dtype f32|bf16] [--bytes B]

One GPU's NVLS traffic (multimem.ld_reduce / multimem.st) tops out near
550 GB/s per direction on this box while SM-driven P2P pushes reach ~680
(DESIGN.md §7).  If that cap is a switch / multicast rate limit rather than
the links being full, a fraction f of the buffer on NVLS and 1-f on FLAT,
running at the same time, would move more bytes per second than either.
Splits S bytes per rank: f*S through an NVLS comm, (1-f)*S through a second
comm running FLAT, on two streams at once; prints busBW (2(n-1)/n * S / t)
per f, max over ranks, median of 5 runs.  (Two comms = two signal pads, so the
two kernels' handshakes never mix.)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--bytes", type=int, default=186 << 20)
    ap.add_argument("--fracs", default="0,0.5,0.6,0.7,0.8,0.9,1")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default="")
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
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    n = world
    tdt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
    esz = 2 if a.dtype == "bf16" else 4
    N = a.bytes // esz
    cn = hfr.Comm.init(device=local, config=hfr.Config(algo="nvls", nvls_bytes=a.bytes + (64 << 20), scale=1.0 / n,
                                                       timeout_ms=30000))
    cf = hfr.Comm.init(device=local, config=hfr.Config(algo="flat", scale=1.0 / n, timeout_ms=30000))
    A = cn.empty(N, tdt)
    B = cf.empty(N, tdt)
    A.normal_()
    B.normal_()
    s1 = torch.cuda.current_stream()
    s2 = torch.cuda.Stream()
    out = open(a.out, "a") if (a.out and rank == 0) else None

    def run(f):
        k = int(N * f) // 64 * 64
        if k > 0:
            cn.allreduce(A[:k], stream=s1)
        if N - k > 0:
            s2.wait_stream(s1)
            cf.allreduce(B[: N - k], stream=s2)
            s1.wait_stream(s2)

    for f in [float(x) for x in a.fracs.split(",")]:
        for _ in range(5):
            run(f)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            dist.barrier()
            cn.barrier(s1)
            cf.barrier(s1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s1)
            for _ in range(a.iters):
                run(f)
            e1.record(s1)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / 1e3 / a.iters], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ts.append(float(t.item()))
        t = statistics.median(ts)
        for c in (cn, cf):
            if c.status() != hfr.SUCCESS:
                raise SystemExit(hfr.status_string(c.status()))
        rec = {"probe": "nvls+flat", "n": n, "dtype": a.dtype, "bytes": a.bytes, "nvls_frac": f,
               "us": t * 1e6, "busbw": a.bytes / t * 2 * (n - 1) / n / 1e9}
        if rank == 0:
            print(json.dumps(rec), flush=True)
            if out:
                out.write(json.dumps(rec) + "\n")
    cn.finalize()
    cf.finalize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
