#!/usr/bin/env python
"""NVLink bytes per allreduce, per GPU and direction, from the NVML link
counters (SURVEY §8(d) "counter evidence"; ncu cannot profile a multi-rank
kernel — its replay would deadlock on the cross-GPU waits).

    torchrun --nproc-per-node N tools/nvlink_traffic.py [--count C] [--steps K]

For each schedule (FLAT, DBT, PAIR_DBT, NVLS, and NCCL's all_reduce on the
same buffer) every rank reads NVML_FI_DEV_NVLINK_COUNT_{XMIT,RCV}_{BYTES,PACKETS}
(summed over its links) and a GPM sample (NVLINK_TOTAL_{TX,RX}_PER_SEC) before and after K back-to-back
allreduces and reports bytes per allreduce.  The algorithmic figure it is set
against is DESIGN.md §6's: FLAT 2(n-1)/n*S per direction.  One JSON line per
(schedule, rank) on rank 0's stdout.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# NVML field -> (name, multiplier to bytes); the COUNT_* fields are the
# NVLink-5 counters (the THROUGHPUT_* ones report "not supported" on B200)
FIELDS = (("COUNT_XMIT_BYTES", "tx_bytes", 1), ("COUNT_RCV_BYTES", "rx_bytes", 1),
          ("COUNT_XMIT_PACKETS", "tx_packets", 1), ("COUNT_RCV_PACKETS", "rx_packets", 1),
          ("THROUGHPUT_DATA_TX", "data_tx_bytes", 1024), ("THROUGHPUT_DATA_RX", "data_rx_bytes", 1024))
NAMES = [n for _, n, _ in FIELDS] + ["gpm_tx_bytes", "gpm_rx_bytes"]


class LinkCounters:
    def __init__(self, device: int):
        import pynvml as p
        self.p = p
        p.nvmlInit()
        self.h = p.nvmlDeviceGetHandleByIndex(device)
        self.links = []
        for l in range(18):
            try:
                if p.nvmlDeviceGetNvLinkState(self.h, l) == p.NVML_FEATURE_ENABLED:
                    self.links.append(l)
            except p.NVMLError:
                pass

    def read(self) -> dict:
        """Counters summed over the active links, in bytes/packets (None
        where unsupported), plus a GPM sample (or None)."""
        p = self.p
        out = {}
        for f, name, mul in FIELDS:
            fid = getattr(p, f"NVML_FI_DEV_NVLINK_{f}")
            total, ok = 0, False
            try:
                vals = p.nvmlDeviceGetFieldValues(self.h, [(fid, l) for l in self.links])
                for v in vals:
                    if v.nvmlReturn == p.NVML_SUCCESS:
                        total += int(v.value.ullVal) * mul
                        ok = True
            except (p.NVMLError, TypeError):
                pass
            out[name] = total if ok else None
        try:
            smp = p.nvmlGpmSampleAlloc()
            p.nvmlGpmSampleGet(self.h, smp)
            out["_gpm"] = smp
        except Exception:  # GPM unsupported / not permitted
            out["_gpm"] = None
        return out

    def gpm_bytes(self, c0, c1, seconds):
        """(tx, rx) bytes between two GPM samples (metrics are MiB/s averages)."""
        p = self.p
        if c0["_gpm"] is None or c1["_gpm"] is None:
            return None, None
        try:
            mg = p.c_nvmlGpmMetricsGet_t()
            mg.version = p.NVML_GPM_METRICS_GET_VERSION
            mg.numMetrics = 2
            mg.sample1, mg.sample2 = c0["_gpm"], c1["_gpm"]
            mg.metrics[0].metricId = p.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
            mg.metrics[1].metricId = p.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
            p.nvmlGpmMetricsGet(mg)
            return (mg.metrics[0].value * (1 << 20) * seconds, mg.metrics[1].value * (1 << 20) * seconds)
        except Exception:
            return None, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=48_758_784, help="fp32 elements per rank (default C2)")
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()

    import torch
    import torch.distributed as dist

    import paper_2408_14158_b200 as hfr
    from paper_2408_14158_b200 import _build

    _build.build()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    S = a.count * 4
    comm = hfr.Comm.init(device=local, config=hfr.Config(algo="flat", nvls_bytes=S + (64 << 20)))
    t = comm.empty(a.count, torch.float32)
    t.normal_()
    ctr = LinkCounters(local)

    def measure(name, fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        c0 = ctr.read()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            fn()
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        c1 = ctr.read()
        dist.barrier()
        per = {f: (None if c0[f] is None or c1[f] is None else (c1[f] - c0[f]) / a.steps) for f in NAMES[:-2]}
        gt, gr = ctr.gpm_bytes(c0, c1, secs)
        per["gpm_tx_bytes"] = None if gt is None else gt / a.steps
        per["gpm_rx_bytes"] = None if gr is None else gr / a.steps
        rec = {"schedule": name, "rank": rank, "n": world, "bytes_per_rank": S, "links": len(ctr.links),
               "per_allreduce_bytes": per,
               "algorithmic_flat_per_direction": 2.0 * (world - 1) / world * S}
        for k in ("tx_bytes", "rx_bytes", "gpm_tx_bytes", "gpm_rx_bytes"):
            if per[k] is not None:
                rec[f"{k}_over_flat_algorithmic"] = per[k] / rec["algorithmic_flat_per_direction"]
        recs = [None] * world
        dist.all_gather_object(recs, rec)
        if rank == 0:
            for r in recs:
                print(json.dumps(r), flush=True)

    for algo in ("flat", "dbt", "pair_dbt", "nvls"):
        try:
            comm.set_config(hfr.Config(algo=algo, scale=1.0 / world))
            measure(algo, lambda: comm.allreduce(t))
        except hfr.HfrError as e:
            if rank == 0:
                print(json.dumps({"schedule": algo, "unavailable": str(e)}), flush=True)
    x = torch.empty(a.count, dtype=torch.float32, device=dev).normal_()
    measure("nccl", lambda: dist.all_reduce(x))
    if comm.status() != hfr.SUCCESS:
        raise SystemExit(hfr.status_string(comm.status()))
    comm.finalize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
