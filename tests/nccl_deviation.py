#!/usr/bin/env python
"""NCCL's numerical deviation from the rank-ascending fold, for context only
(SURVEY §8(c) "NCCL: parity unpinned ... record its max deviation").

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tests/nccl_deviation.py --out gpurun_out/nccl_dev.jsonl

For each dtype and value distribution, every rank all-reduces its seeded
buffer with torch.distributed (NCCL) and rank 0 compares the result with the
oracle's fold: fraction of elements whose bits differ, max |d| / A with
A = sum_r |x_r| (reading R18's normaliser), and whether every element lies
inside R18's bound.  The same is printed for HFR FLAT (bit-exact: 0).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=1 << 22)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import hfr_inputs as gen
    import paper_2408_14158_b200 as hfr
    from oracle import hfr_oracle as O
    from tests.gpu_util import as_f32, to_numpy, to_torch, torch_dtype

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = hfr.Comm.init(device=local, config=hfr.Config(algo="flat"))
    out = open(a.out, "a") if (a.out and rank == 0) else None
    for dtype in (gen.FP32, gen.BF16):
        for dist_name in ("normal", "loguniform"):
            xs = gen.rank_inputs(world, a.count, dtype, dist_name, seed_base=2000)
            want = O.fold_ascending(xs)
            Ab = np.zeros(a.count)
            for x in xs:
                Ab += np.abs(as_f32(x).astype(np.float64))
            for impl in ("nccl", "hfr_flat"):
                if impl == "nccl":
                    t = to_torch(xs[rank], f"cuda:{local}")
                    dist.all_reduce(t)
                else:
                    t = comm.empty(a.count, torch_dtype(dtype))
                    t.copy_(to_torch(xs[rank], t.device))
                    comm.allreduce(t)
                torch.cuda.synchronize()
                got = to_numpy(t)
                if rank != 0:
                    continue
                g = as_f32(got).astype(np.float64)
                w = as_f32(want).astype(np.float64)
                fin = np.isfinite(w)
                d = np.abs(g[fin] - w[fin])
                rel = d / np.maximum(Ab[fin], 1e-300)
                if dtype == gen.FP32:
                    lim = 1e-6 * Ab[fin]
                else:
                    ex = np.floor(np.log2(np.maximum(np.abs(w[fin]), 2.0 ** -126)))
                    ulp = 2.0 ** (ex - 7)
                    lim = np.maximum(ulp, 8.3e-7 * Ab[fin] + 0.5 * ulp)
                rec = {"impl": impl, "n": world, "dtype": dtype, "dist": dist_name, "count": a.count,
                       "bits_differ_frac": float(np.mean(got.view(np.uint16 if got.dtype.itemsize == 2 else np.uint32)
                                                         != want.view(np.uint16 if want.dtype.itemsize == 2 else np.uint32))),
                       "max_abs_over_A": float(rel.max()) if rel.size else 0.0,
                       "beyond_r18": int((d > lim).sum()),
                       "env": {k: v for k, v in os.environ.items() if k.startswith("NCCL_")}}
                s = json.dumps(rec)
                print(s, flush=True)
                if out:
                    out.write(s + "\n")
            comm.free_all()
    comm.finalize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
