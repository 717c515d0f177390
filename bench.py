#!/usr/bin/env python
"""bench.py — HFReduce allreduce bus bandwidth on B200 (the BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

Workload (config 2 of BASELINE.json): an fp32 sum-allreduce of one 186 MiB
gradient buffer per rank (48,758,784 elements, N(0, 1e-3^2) values, seeds
rng(1000 + rank)), the FLAT schedule (fused reduce-scatter + all-gather, the
rank-ascending fold that is bit-exact to the oracle), in symmetric peer-mapped
memory (zero-copy), scale = 1/n (gradient averaging, fused into the epilogue).

  N = 1  8 VIRTUAL ranks on one B200 (hfr_init_virtual): the same kernel and
         protocol with HBM as the transport ("C2-virtual8").
  N > 1  one rank per GPU over NVLink/NVSwitch ("C2-nvlink"), n = N.

A step is one allreduce of the whole buffer.  value = busBW = S/t * 2(n-1)/n
(nccl-tests convention, reading R15) with t the per-step device time, max over
ranks; inputs (186 MiB per rank) exceed the 126 MB L2, so no flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "allreduce bus GB/s (max over ranks) at 2/4/8 B200 vs NCCL & 900 GB/s NVLink"
NVLINK_PEER_GBS = 770.0   # B200_PROFILING.md: measured peer copy per direction (900 nominal)
NVLINK_NOMINAL_GBS = 900.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["hfr", "reference"], default="hfr")
    p.add_argument("--algo", default="flat", choices=["flat", "dbt", "pair_dbt"])
    p.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    p.add_argument("--count", type=int, default=0, help="elements per rank (default: C2 = 186 MiB fp32)")
    p.add_argument("--virtual", type=int, default=8, help="virtual ranks at N=1")
    p.add_argument("--max-ctas", type=int, default=0)
    p.add_argument("--threads", type=int, default=0)
    p.add_argument("--soak", type=float, default=1.0, help="untimed seconds of load for the clock sampler")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-nccl", action="store_true")
    p.add_argument("--no-variants", action="store_true")
    p.add_argument("--e2e-chunks", type=int, default=8, help="pipeline depth of the e2e step (1 = sequential)")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json)"
    except OSError:
        return 6650.0, "fallback (B200_PROFILING.md)"


def busbw(bytes_per_rank: float, seconds: float, n: int) -> float:
    return bytes_per_rank / seconds * 2.0 * (n - 1) / n / 1e9 if n > 1 else 0.0


def algbw(bytes_per_rank: float, seconds: float) -> float:
    return bytes_per_rank / seconds / 1e9


# ---------------------------------------------------------------------------
# clock sampler (B200_PROFILING.md "clocks DURING the timed region")
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int, interval_ms: int = 100):
        self.device = device
        self.interval_ms = interval_ms
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-i", str(self.device), "-lms", str(self.interval_ms)],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
            out, _ = self.p.communicate()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# ---------------------------------------------------------------------------
# CPU baseline: the C oracle (oracle/fold.c) on the host cores
# ---------------------------------------------------------------------------
def cpu_oracle_run(n: int, count: int, dtype: str, budget_s: float, max_reps: int = 1000):
    import hfr_inputs as gen
    from oracle import cfold
    xs = gen.rank_inputs(n, count, dtype, "grad", seed_base=1000)
    cfold.fold_ascending(xs, 1.0 / n)  # warm (page in)
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < max_reps and (not times or time.perf_counter() < t_end):
        t0 = time.perf_counter()
        cfold.fold_ascending(xs, 1.0 / n)
        times.append(time.perf_counter() - t0)
    return times, cfold.threads()


def reference_arm(args):
    """--impl reference: the oracle as it stands (oracle/fold.c, the
    rank-ascending fold of PAPER.md:333-336) timed on the host cores for the
    same workload, metric and unit.  Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.gpus if args.gpus > 1 else args.virtual
    dtype = "bf16" if args.dtype == "bf16" else "f32"
    count = args.count or (186 << 20) // 4
    esz = 2 if dtype == "bf16" else 4
    S = count * esz
    import hfr_inputs as gen
    from oracle import cfold
    xs = gen.rank_inputs(n, count, dtype, "grad", seed_base=1000)
    for _ in range(args.warmup):
        cfold.fold_ascending(xs, 1.0 / n)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cfold.fold_ascending(xs, 1.0 / n)
    t = (time.perf_counter() - t0) / args.steps
    v = busbw(S, t, n)
    cores = cfold.threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
        "config": workload_config(args, n, count, dtype),
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "sample": f"full workload: rank-ascending fold of {n} x {count} {dtype} elements per step "
                                   f"(oracle/fold.c, OpenMP {cores} threads), busBW-equivalent S/t*2(n-1)/n"},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, n, count, dtype):
    esz = 2 if dtype == "bf16" else 4
    virtual = args.gpus <= 1
    return {
        "workload": ("C2-virtual%d" % n) if virtual else "C2-nvlink",
        "description": (f"{n} {'virtual ranks on one B200 (HBM transport)' if virtual else 'ranks, one per B200 (NVLink/NVSwitch)'}"
                        f" x {count * esz / 2**20:.0f} MiB {dtype} sum-allreduce, scale 1/n"),
        "ranks": n, "count_per_rank": count, "bytes_per_rank": count * esz, "algo": args.algo,
        "memory": "symmetric (hfr_mem_alloc, zero-copy)",
        "l2": "inputs larger than L2 (bytes_per_rank > 126 MB), no flush",
        "parallelism": f"dp{args.gpus}",
    }


# ---------------------------------------------------------------------------
# the HFReduce arm
# ---------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import hfr_inputs as gen
    import paper_2408_14158_b200 as hfr
    from paper_2408_14158_b200 import _build

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus or (world == 1 and args.gpus == 1), "launch N>1 under torchrun with --gpus N"
    _build.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    multi = world > 1
    if multi:
        dist.init_process_group("nccl", device_id=dev)
    dtype = args.dtype
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    esz = 2 if dtype == "bf16" else 4
    count = args.count or (186 << 20) // 4
    n = world if multi else args.virtual
    S = count * esz
    scale = 1.0 / n
    cfg = hfr.Config(algo=args.algo, scale=scale, max_ctas=args.max_ctas, threads=args.threads,
                     timeout_ms=30000)
    nvls_note = None
    if multi:
        # NVLS arena (order-relaxed variant) holds the bench buffer; FLAT runs on it zero-copy too
        try:
            comm = hfr.Comm.init(device=local, config=hfr.Config(**{**cfg.__dict__, "nvls_bytes": S + (64 << 20)}))
        except hfr.HfrError as e:
            nvls_note = f"no NVLS arena: {e}"
            comm = hfr.Comm.init(device=local, config=cfg)
    else:
        comm = hfr.Comm.virtual_ranks(n, local, cfg)
    stream = torch.cuda.current_stream()

    # inputs: this process's ranks
    my_ranks = [rank] if multi else list(range(n))
    host_in = []
    for r in my_ranks:
        x = gen.rank_input(r, count, dtype, "grad", seed_base=1000)
        t = torch.from_numpy(x.view(np.int16) if dtype == "bf16" else x)
        host_in.append(t.view(tdt).pin_memory())
    bufs = comm.empty(count, tdt)
    bufs = bufs if isinstance(bufs, list) else [bufs]
    for b, h in zip(bufs, host_in):
        b.copy_(h, non_blocking=True)
    torch.cuda.synchronize()

    def step():
        if multi:
            comm.allreduce(bufs[0])
        else:
            comm.allreduce_virtual(bufs)

    def max_over_ranks(v: float) -> float:
        if not multi:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, steps):
        """Device time per step of `steps` calls of fn on the current stream,
        after a host + device barrier; max over ranks."""
        if multi:
            dist.barrier()
        comm.barrier(stream)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        l0 = comm.launches
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        launches = comm.launches - l0
        return max_over_ranks(e0.elapsed_time(e1) / 1e3 / steps), launches

    # warm-up; the clock sampler runs over the timed region and an untimed soak
    # right after it (so it collects samples even when K steps take ~10 ms)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.15)
    t_step, launches = timed(step, args.steps)
    t_soak = time.perf_counter() + args.soak
    while time.perf_counter() < t_soak:
        for _ in range(10):
            step()
        torch.cuda.synchronize()
    ck = clocks.stop()
    if comm.status() != hfr.SUCCESS:
        raise SystemExit(f"hfr error: {hfr.status_string(comm.status())}")

    value = busbw(S, t_step, n)
    hbm_peak, hbm_src = peaks()
    # the step's one kernel: the TMA-staged FLAT kernel for n in {2,4,8}
    tma = os.environ.get("HFR_FLAT_TMA", "1") != "0" and n in (2, 4, 8)
    kname = ("hfr_flat_tma_kernel" if tma else "hfr_flat_kernel") if args.algo == "flat" else "hfr_tree_kernel"
    if multi:
        nv_bytes = 2.0 * (n - 1) / n * S   # per GPU per direction per launch (§8d)
        roof = {"bound": "nvlink", "achieved": nv_bytes / t_step / 1e9, "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                "frac": nv_bytes / t_step / 1e9 / NVLINK_PEER_GBS, "traffic": None,
                "kernel": kname,
                "algorithmic_bytes_per_launch": nv_bytes,
                "peak_source": "measured peer copy 770 GB/s/dir (B200_PROFILING.md); 900 nominal",
                "frac_of_nominal": nv_bytes / t_step / 1e9 / NVLINK_NOMINAL_GBS}
    else:
        hbm_bytes = 2.0 * n * S            # every rank's buffer read once and written once
        roof = {"bound": "hbm", "achieved": hbm_bytes / t_step / 1e9, "peak": hbm_peak, "unit": "GB/s",
                "frac": hbm_bytes / t_step / 1e9 / hbm_peak, "traffic": None,
                "kernel": kname,
                "algorithmic_bytes_per_launch": hbm_bytes, "peak_source": hbm_src}
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            tr = json.load(open(prof)).get(f"{roof['kernel']}:{args.algo}:{n}:{dtype}:{'virtual' if not multi else 'nvlink'}")
            if tr:
                roof["traffic"] = tr
        except (OSError, ValueError):
            pass

    # ---- e2e through the public API: H2D inputs, allreduce, D2H result ----
    # The copies dominate (PCIe), so the step is pipelined the way a user of
    # the public API would: the buffer is cut into 8 chunks; chunk i's H2D (one
    # stream), allreduce (the current stream) and D2H (a third stream) overlap
    # chunk i+1's.  Every byte of the inputs and of the result crosses PCIe
    # inside the timed region.
    # The step's result is the reduced buffer: every rank holds the same bits
    # (the parity tests check cross-rank identity), so a process reads back
    # one copy — its own rank's at N>1, local rank 0's for the n virtual ranks.
    e2e = None
    if not args.no_e2e:
        host_out = [torch.empty_like(host_in[0]).pin_memory()]
        nchunk = max(1, args.e2e_chunks)
        K = 8 if dtype == "bf16" else 4
        edges = [(count * i // nchunk) // K * K for i in range(nchunk)] + [count]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in range(nchunk)]
        ev_red = [torch.cuda.Event() for _ in range(nchunk)]

        def e2e_step():
            cur = torch.cuda.current_stream()
            s_in.wait_stream(cur)
            for i in range(nchunk):
                lo, hi = edges[i], edges[i + 1]
                with torch.cuda.stream(s_in):
                    for b, h in zip(bufs, host_in):
                        b[lo:hi].copy_(h[lo:hi], non_blocking=True)
                    ev_in[i].record(s_in)
                cur.wait_event(ev_in[i])
                if multi:
                    comm.allreduce(bufs[0][lo:hi])
                else:
                    comm.allreduce_virtual([b[lo:hi] for b in bufs])
                ev_red[i].record(cur)
                s_out.wait_event(ev_red[i])
                with torch.cuda.stream(s_out):
                    host_out[0][lo:hi].copy_(bufs[0][lo:hi], non_blocking=True)
            cur.wait_stream(s_out)

        e2e_step()
        torch.cuda.synchronize()
        t_e2e, e2e_launches = timed(e2e_step, max(1, min(args.steps, 10)))
        e2e = {"value": busbw(S, t_e2e, n), "unit": "GB/s", "ms_per_step": t_e2e * 1e3,
               "h2d_bytes_per_step": S * len(bufs), "d2h_bytes_per_step": S,
               "note": "per step: pinned H2D of each local rank's input, hfr_allreduce, D2H of the result "
                       "(one copy per process: the ranks' results are bitwise identical), "
                       f"pipelined over {nchunk} chunk(s) on 3 streams; PCIe-bound"}

    # ---- context: NCCL on the same buffer, and the tree schedules ----
    nccl = None
    if multi and not args.no_nccl:
        t = torch.empty(count, dtype=tdt, device=dev)
        t.copy_(host_in[0])

        def nccl_step():
            dist.all_reduce(t)

        for _ in range(args.warmup):
            nccl_step()
        if multi:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            nccl_step()
        e1.record()
        torch.cuda.synchronize()
        tn = max_over_ranks(e0.elapsed_time(e1) / 1e3 / args.steps)
        nccl = {"busbw": busbw(S, tn, n), "ms_per_step": tn * 1e3, "version": ".".join(map(str, torch.cuda.nccl.version())),
                "settings": "default (env: NCCL_ALGO=%s NCCL_NVLS_ENABLE=%s)" % (
                    os.environ.get("NCCL_ALGO", "-"), os.environ.get("NCCL_NVLS_ENABLE", "-")),
                "hfr_over_nccl": value / busbw(S, tn, n) if tn > 0 else None}
        del t
    variants = {}
    if multi and not args.no_variants:  # tree schedules over NVLink (virtual-rank trees are not meaningful)
        for algo in ("dbt", "pair_dbt", "nvls"):
            if algo == args.algo or (algo == "pair_dbt" and n % 2):
                continue
            comm.set_config(hfr.Config(algo=algo, scale=scale, max_ctas=args.max_ctas, threads=args.threads,
                                       timeout_ms=30000))
            try:
                for _ in range(2):
                    step()
                tv, _ = timed(step, max(3, args.steps // 2))
            except hfr.HfrError as e:  # context only: never lose the headline line over a variant
                variants[algo] = {"unavailable": (nvls_note if algo == "nvls" and nvls_note else str(e))}
                if comm.status() != hfr.SUCCESS:
                    break
                continue
            variants[algo] = {"busbw": busbw(S, tv, n), "ms_per_step": tv * 1e3}
            if algo == "nvls":
                variants[algo]["numerics"] = "order-relaxed (NVSwitch reduction), held to DESIGN.md R18, not bit-exact"
            else:
                variants[algo]["numerics"] = "bit-exact vs the tree-order / pair-first oracle"
        if comm.status() == hfr.SUCCESS:
            comm.set_config(cfg)

    cpu = None
    if rank == 0 and not multi and not args.no_cpu:
        times, cores = cpu_oracle_run(n, count, dtype, budget_s=10.0)
        tc = statistics.median(times)
        cpu = {"value": busbw(S, tc, n), "unit": "GB/s", "cores": cores, "kind": "oracle",
               "sample": f"full C2 workload ({n} x {count} {dtype}), oracle/fold.c rank-ascending fold, "
                         f"median of {len(times)} reps (~10 s), busBW-equivalent S/t*2(n-1)/n"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": dict(workload_config(args, n, count, dtype), clock_soak_s=args.soak),
            "algbw": algbw(S, t_step), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": ck, "nccl": nccl, "variants": variants,
        }
        print(json.dumps(line), flush=True)
    comm.finalize()
    if multi:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
