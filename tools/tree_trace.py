#!/usr/bin/env python
"""Record and summarise per-CTA chunk timelines of the tree schedules.

  torchrun --nproc-per-node N tools/tree_trace.py --algo dbt --chunk 32768 --ctas 64 --out gpurun_out/tr
  python tools/tree_trace.py --analyze gpurun_out/tr

Each rank dumps rank<r>.npy = [CTA, event, 8] u64 {tag, t_wait, t_work, t_stores_issued, t_done, ...}
(hfr_set_trace).  The summary prints, per rank and pass, the summed wait and
work time and the span, which tells whether a tree launch is limited by
transfer work, by waiting on tree neighbours, or by pipeline fill/drain.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PH = {1: "up", 2: "down", 3: "pair_wait"}


def analyze(d):
    out = {}
    files = sorted(glob.glob(os.path.join(d, "rank*.npy")))
    t_all0 = None
    for f in files:
        r = int(os.path.basename(f)[4:-4])
        tr = np.load(f)
        ev = tr.reshape(-1, 8)
        ev = ev[ev[:, 0] != 0]
        if ev.size == 0:
            continue
        ph = (ev[:, 0] >> 60).astype(int)
        t0, t1, ts, t2 = (ev[:, k].astype(np.int64) for k in (1, 2, 3, 4))
        base = t0.min()
        rep = {"span_us": (t2.max() - base) / 1e3, "events": int(len(ev))}
        # CTA parity = the tree a CTA works on (TMA tree kernel): split by role
        cta_of = np.repeat(np.arange(tr.shape[0]), tr.shape[1])[tr.reshape(-1, 8)[:, 0] != 0]
        for p, name in [(p, f"{nm}_tree{par}") for p, nm in PH.items() for par in (0, 1)]:
            m = (ph == p) & ((cta_of & 1) == int(name[-1]))
            if not m.any():
                continue
            rep[name] = {"n": int(m.sum()), "wait_us_sum": float((t1[m] - t0[m]).sum() / 1e3),
                         "work_us_sum": float((t2[m] - t1[m]).sum() / 1e3),
                         "work_us_mean": float((t2[m] - t1[m]).mean() / 1e3),
                         "issue_us_mean": float((ts[m] - t1[m]).mean() / 1e3),
                         "drain_us_mean": float((t2[m] - ts[m]).mean() / 1e3),
                         "first_done_us": float((t2[m].min() - base) / 1e3),
                         # TMA tree kernel only (slots 5/6: bulk-group wait done, fences done)
                         **({"bulk_wait_us_mean": float((ev[m, 5].astype(np.int64) - ts[m]).mean() / 1e3),
                             "fence_us_mean": float((ev[m, 6].astype(np.int64) - ev[m, 5].astype(np.int64)).mean() / 1e3)}
                            if (ev[m, 5] != 0).all() else {}),
                         "last_done_us": float((t2[m].max() - base) / 1e3)}
        # per-CTA busy fraction
        ctas = tr.shape[0]
        busy = []
        for cta in range(ctas):
            e = tr[cta]
            e = e[e[:, 0] != 0]
            if len(e):
                busy.append(float((e[:, 4].astype(np.int64) - e[:, 2].astype(np.int64)).sum()
                                  / max(1, (e[:, 4].max() - e[:, 1].min()))))
        rep["cta_busy_frac_mean"] = float(np.mean(busy)) if busy else None
        out[r] = rep
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--analyze", default="")
    ap.add_argument("--algo", default="dbt")
    ap.add_argument("--chunk", type=int, default=32768)
    ap.add_argument("--ctas", type=int, default=64)
    ap.add_argument("--bytes", type=int, default=186 << 20)
    ap.add_argument("--out", default="gpurun_out/trace")
    ap.add_argument("--staging", type=int, default=0, help="hfr_config.tree_staging")
    a = ap.parse_args()
    if a.analyze:
        print(json.dumps(analyze(a.analyze), indent=1))
        return
    import torch
    import torch.distributed as dist

    import paper_2408_14158_b200 as hfr
    from paper_2408_14158_b200 import _build
    _build.build()
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = hfr.Comm.init(device=local, config=hfr.Config(algo=a.algo, chunk_elems=a.chunk, max_ctas=a.ctas,
                                                        scale=1.0 / dist.get_world_size(),
                                                        tree_staging=a.staging))
    t = comm.empty(a.bytes // 4, torch.float32)
    t.normal_()
    for _ in range(3):
        comm.allreduce(t)
    cap = 512
    tb = torch.zeros(64 * 1024 * cap, dtype=torch.uint8, device=f"cuda:{local}")
    comm.set_trace(tb)
    dist.barrier()
    comm.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    comm.allreduce(t)
    e1.record()
    torch.cuda.synchronize()
    comm.set_trace(None)
    os.makedirs(a.out, exist_ok=True)
    arr = tb.view(torch.int64).view(1024, cap, 8)[: (a.ctas or 296)].cpu().numpy().view(np.uint64)
    np.save(os.path.join(a.out, f"rank{rank}.npy"), arr)
    ms = torch.tensor([e0.elapsed_time(e1)], device=f"cuda:{local}")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        n = dist.get_world_size()
        print(json.dumps({"algo": a.algo, "chunk": a.chunk, "ctas": a.ctas, "staging": a.staging,
                          "n": n, "ms": float(ms),
                          "busbw": a.bytes / (float(ms) / 1e3) * 2 * (n - 1) / n / 1e9}))
    comm.finalize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
