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

A step is one allreduce of the whole buffer, t its device time (max over
ranks); inputs (186 MiB per rank) exceed the 126 MB L2, so no flush is needed.
  N > 1  value = busBW = S/t * 2(n-1)/n (nccl-tests convention, reading R15),
         roofline against the per-direction NVLink peak MEASURED on this lease
         (tools/p2p_probe.cu, all GPUs moving at once) and against 900 nominal.
  N = 1  busBW is 0 for one GPU: value = algBW = S/t of the 8
         virtual-rank allreduce, roofline against the measured HBM bandwidth
         (2·n·S bytes per launch); the 8-rank busBW is kept as `busbw_virtual`.
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
NVLINK_GUIDE_GBS = 770.0  # B200_PROFILING.md: measured peer copy per direction (fallback only)
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
    p.add_argument("--no-probe", action="store_true", help="skip the NVLink probe (roofline peak falls back)")
    p.add_argument("--no-nvls", action="store_true", help="no NVLS arena (plain symmetric memory)")
    p.add_argument("--dist", default="nccl", choices=["nccl", "gloo"],
                   help="torch.distributed backend for the host plumbing (gloo under ncu: no NCCL kernels; "
                        "implies --no-nccl)")
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


def headline(bytes_per_rank: float, seconds: float, n: int, multi: bool) -> float:
    """The line's `value`: busBW over NVLink (N > 1); algBW of the virtual-rank
    allreduce on one GPU (N = 1, where busBW is 0 by definition)."""
    return busbw(bytes_per_rank, seconds, n) if multi else algbw(bytes_per_rank, seconds)


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
def host_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def cpu_oracle_run(n: int, count: int, dtype: str, budget_s: float, max_reps: int = 1000, threads: int = 0):
    import hfr_inputs as gen
    from oracle import cfold
    xs = gen.rank_inputs(n, count, dtype, "grad", seed_base=1000)
    cfold.set_threads(threads if threads > 0 else (os.cpu_count() or 1))
    cfold.fold_ascending(xs, 1.0 / n)  # warm (page in)
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < max_reps and (not times or time.perf_counter() < t_end):
        t0 = time.perf_counter()
        cfold.fold_ascending(xs, 1.0 / n)
        times.append(time.perf_counter() - t0)
    used = cfold.threads()
    cfold.set_threads(os.cpu_count() or 1)
    return times, used


def cpu_baseline(n: int, count: int, dtype: str, esz: int, multi: bool, budget_s: float = 10.0):
    """The oracle (oracle/fold.c, rank-ascending fold, as it stands) on the
    host cores: all cores on the full workload (n x count), plus one thread
    on a 1/16 sample; the line's own metric (busBW-equivalent
    at N > 1, algBW at N = 1), as if the CPU fold were the allreduce."""
    S = count * esz
    times, cores = cpu_oracle_run(n, count, dtype, budget_s=budget_s)
    tc = statistics.median(times)
    small = max(4096, count // 16)
    t1, _ = cpu_oracle_run(n, small, dtype, budget_s=budget_s / 2, max_reps=50, threads=1)
    t1m = statistics.median(t1)
    def metric(b, t):
        return headline(b, t, n, multi)
    # SURVEY §8(d) also asks for GB/s over the (n+1)*S bytes the fold touches
    # and the Python oracle's time on C1 (2 ranks x 4096 fp32)
    import hfr_inputs as gen
    from oracle import hfr_oracle as O
    c1 = gen.rank_inputs(2, 4096, gen.FP32, "normal", seed_base=1234)
    O.fold_ascending(c1)
    tp = []
    for _ in range(20):
        t0 = time.perf_counter()
        O.fold_ascending(c1)
        tp.append(time.perf_counter() - t0)
    return {"value": metric(S, tc), "unit": "GB/s", "cores": cores, "kind": "oracle",
            "touched_gbs": (n + 1) * S / tc / 1e9,
            "c1_python_oracle_ms": statistics.median(tp) * 1e3,
            "sample": f"full workload ({n} x {count} {dtype}), oracle/fold.c rank-ascending fold, median of "
                      f"{len(times)} reps (~{budget_s:.0f} s), {'busBW' if multi else 'algBW'}-equivalent",
            "one_thread": {"value": metric(small * esz, t1m), "unit": "GB/s", "cores": 1,
                           "sample": f"{n} x {small} {dtype} (1/16 of the workload), median of {len(t1)} reps"},
            "host": host_info()}


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
    # all host cores: torchrun sets OMP_NUM_THREADS=1 for its workers, which
    # would time the oracle on one core at N > 1
    cfold.set_threads(os.cpu_count() or 1)
    for _ in range(args.warmup):
        cfold.fold_ascending(xs, 1.0 / n)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cfold.fold_ascending(xs, 1.0 / n)
    t = (time.perf_counter() - t0) / args.steps
    multi = args.gpus > 1
    v = headline(S, t, n, multi)
    cores = cfold.threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
        "value_definition": value_definition(multi),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
        "config": workload_config(args, n, count, dtype),
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "sample": f"full workload: rank-ascending fold of {n} x {count} {dtype} elements per step "
                                   f"(oracle/fold.c, OpenMP {cores} threads), "
                                   f"{'busBW' if multi else 'algBW'}-equivalent", "host": host_info()},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def value_definition(multi: bool) -> str:
    if multi:
        return "busBW = S/t*2(n-1)/n, t = device time per allreduce, max over ranks (nccl-tests convention)"
    return ("algBW = S/t of the 8-virtual-rank allreduce on one B200 (busBW is 0 for one GPU, SURVEY §8(d)); "
            "the virtual-rank busBW is busbw_virtual")


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
# NVLink per-direction peak measured on this lease (the roofline
# denominator must not be a number copied from a guide)
# ---------------------------------------------------------------------------
PROBE_SRC = os.path.join(ROOT, "tools", "p2p_probe.cu")
PROBE_BIN = os.path.join(ROOT, "tools", "p2p_probe")


def nvlink_probe(n: int):
    """Run tools/p2p_probe.cu over GPUs 0..n-1 (all moving at once, 256 MiB per
    peer, 148 CTAs x 512 threads) and return {pattern: GB/s per GPU per
    direction}; None if it cannot run."""
    import re
    try:
        if not os.path.exists(PROBE_BIN) or os.path.getmtime(PROBE_BIN) < os.path.getmtime(PROBE_SRC):
            subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                            "-o", PROBE_BIN, PROBE_SRC], check=True, capture_output=True, timeout=300)
        out = subprocess.run([PROBE_BIN, str(n), "256", "148", "512"], check=True, capture_output=True,
                             text=True, timeout=300).stdout
    except (OSError, subprocess.SubprocessError):
        return None
    res = {}
    for line in out.splitlines():
        m = re.match(r"n=\d+ (.+?)\s+\d+ MiB/peer.*->\s+([\d.]+) GB/s", line)
        if m:
            res[m.group(1).strip()] = float(m.group(2))
    return res or None


def nvlink_peak(probe):
    """The roofline denominator: the best all-GPUs-at-once pattern (pull,
    push or mixed pull/push — FLAT's own traffic is the mixed one)."""
    if not probe:
        return NVLINK_GUIDE_GBS, "fallback: B200_PROFILING.md peer copy 770 GB/s/dir (probe unavailable)"
    # every all-GPUs-at-once pattern, SM-driven or bulk-copy (TMA) driven
    keys = [k for k in probe if k.startswith(("read  (pull", "write (push", "mixed", "tma push", "tma pull", "tma mixed"))]
    if not keys:
        return NVLINK_GUIDE_GBS, "fallback: B200_PROFILING.md peer copy 770 GB/s/dir (probe parse failed)"
    best = max(keys, key=lambda k: probe[k])
    return probe[best], f"measured on this lease: tools/p2p_probe.cu '{best}', all {len(keys)} all-GPU patterns"


def source_sha():
    """sha256 of the library sources (the .so itself embeds box-local paths)."""
    import hashlib
    from paper_2408_14158_b200 import _build
    h = hashlib.sha256()
    for p in _build.DEPS:
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def committed_traffic(key: str):
    """ncu DRAM (+ NVLink) bytes per launch for this kernel/config from
    profiles/traffic.json, only if captured from the current sources."""
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        rec = json.load(open(prof)).get(key)
    except (OSError, ValueError):
        return None, None
    if not isinstance(rec, dict):
        return None, None
    if rec.get("source_sha") != source_sha():
        return None, {"stale": rec.get("source"), "captured_sha": rec.get("source_sha"), "current_sha": source_sha()}
    return rec, {"source": rec.get("source"), "source_sha": rec.get("source_sha")}


def variant_dir_bytes(hfr, algo: str, n: int, S: int, esz: int) -> float:
    """Algorithmic NVLink bytes per direction of the busiest rank for one
    allreduce of S bytes per rank, from the trees the
    library builds (hfr_tree_query): up-pass partials fp32 (16-bit and FP8
    DBT leaves send their raw values), down pass in the buffer dtype; PAIR adds the pair
    reduce-scatter and all-gather halves; NVLS (n+1)/n·S."""
    if algo == "nvls":
        return (n + 1) / n * S
    N = S / esz
    pair = algo == "pair_dbt"
    m = n // 2 if pair else n
    data = N / 2 if pair else N             # elements each tree set covers
    eg = [0.0] * m
    ing = [0.0] * m
    for which in (0, 1):                    # half of the chunks ride each tree
        parent, children = hfr.tree_query(m, which)
        for v in range(m):
            for c in children[v]:
                up = (esz if (not pair and esz < 4 and not children[c]) else 4) * data / 2
                eg[c] += up
                ing[v] += up
                eg[v] += esz * data / 2     # final chunk down to the child
                ing[c] += esz * data / 2
    worst = max(max(e, i) for e, i in zip(eg, ing)) if m > 1 else 0.0
    if pair:
        worst += S / 2 + S / 2              # pair RS + pair AG (partner link, both directions)
    return worst


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
        if args.dist == "gloo":
            dist.init_process_group("gloo")
            args.no_nccl = True
        else:
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
    probe = None
    if multi:
        # the per-direction NVLink peak of this lease, before anything else runs
        if rank == 0 and not args.no_probe:
            probe = nvlink_probe(n)
        dist.barrier()
    nvls_note = None
    if multi and not args.no_nvls:
        # NVLS arena (order-relaxed variant) holds the bench buffer; FLAT runs on it zero-copy too
        try:
            comm = hfr.Comm.init(device=local, config=hfr.Config(**{**cfg.__dict__, "nvls_bytes": S + (64 << 20)}))
        except hfr.HfrError as e:
            nvls_note = f"no NVLS arena: {e}"
            comm = hfr.Comm.init(device=local, config=cfg)
    elif multi:
        nvls_note = "no NVLS arena (--no-nvls)"
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
        t = torch.tensor([v], dtype=torch.float64, device=dev if args.dist == "nccl" else "cpu")
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

    value = headline(S, t_step, n, multi)
    hbm_peak, hbm_src = peaks()
    # the step's one kernel: the TMA-staged FLAT kernel for n in {2,4,8}
    kname = ("hfr_flat_tma_kernel" if n in (2, 4, 8) else "hfr_flat_kernel") if args.algo == "flat" \
        else "hfr_tree_kernel"
    tkey = f"{kname}:{args.algo}:{n}:{dtype}:{count}:{'nvlink' if multi else 'virtual'}"
    trec, tprov = committed_traffic(tkey)
    if multi:
        nv_bytes = 2.0 * (n - 1) / n * S   # per GPU per direction per launch (§8d)
        peak, peak_src = nvlink_peak(probe)
        achieved = nv_bytes / t_step / 1e9
        roof = {"bound": "nvlink", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "frac_of_nominal": achieved / NVLINK_NOMINAL_GBS,
                "frac_of_guide": achieved / NVLINK_GUIDE_GBS,  # B200_PROFILING.md's measured peer copy
                "nominal": NVLINK_NOMINAL_GBS,
                # CUPTI PM-sampled NVLink bytes per launch (tools/pm_nvlink.py), the larger
                # direction of rank 0: the user payload (comparable with the algorithmic
                # bytes) and what crossed the wire incl. packet protocol
                "traffic": (max(trec.get("nvltx_user_bytes") or 0, trec.get("nvlrx_user_bytes") or 0)
                            or None) if trec else None,
                "traffic_kind": "NVLink user-payload bytes per launch (CUPTI PM sampling, nvltx/nvlrx "
                                "__bytes_data_user, larger direction, rank 0)",
                "traffic_wire": (max(trec.get("nvltx_bytes") or 0, trec.get("nvlrx_bytes") or 0) or None)
                if trec else None,
                "dram_traffic": trec.get("dram_bytes") if trec else None,
                "traffic_provenance": tprov,
                "kernel": kname, "algorithmic_bytes_per_launch": nv_bytes,
                "peak_source": peak_src, "probe_gbs": probe}
    else:
        hbm_bytes = 2.0 * n * S            # every rank's buffer read once and written once
        roof = {"bound": "hbm", "achieved": hbm_bytes / t_step / 1e9, "peak": hbm_peak, "unit": "GB/s",
                "frac": hbm_bytes / t_step / 1e9 / hbm_peak,
                "traffic": trec.get("dram_bytes") if trec else None,
                "traffic_kind": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch",
                "traffic_provenance": tprov,
                "kernel": kname, "algorithmic_bytes_per_launch": hbm_bytes, "peak_source": hbm_src}

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
        e2e = {"value": headline(S, t_e2e, n, multi), "unit": "GB/s", "ms_per_step": t_e2e * 1e3,
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
            vb = variant_dir_bytes(hfr, algo, n, S, esz)
            variants[algo] = {"busbw": busbw(S, tv, n), "ms_per_step": tv * 1e3,
                              "nvlink_bytes_per_dir": vb, "achieved_dir_gbs": vb / tv / 1e9,
                              "frac_of_peak": vb / tv / 1e9 / roof["peak"],
                              "busbw_ceiling_at_peak": busbw(S, vb / roof["peak"] / 1e9, n)}
            if algo == "nvls":
                variants[algo]["numerics"] = "order-relaxed (NVSwitch reduction), held to DESIGN.md R18, not bit-exact"
            else:
                variants[algo]["numerics"] = "bit-exact vs the tree-order / pair-first oracle"
        if comm.status() == hfr.SUCCESS:
            comm.set_config(cfg)

    cpu = None
    if rank == 0 and not args.no_cpu:  # every N: rank 0, after the GPU timing (the others wait)
        cpu = cpu_baseline(n, count, dtype, esz, multi)
    if multi:
        dist.barrier()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            # the same config object as the reference arm's (the driver compares them)
            "config": workload_config(args, n, count, dtype),
            "value_definition": value_definition(multi),
            "algbw": algbw(S, t_step), "busbw_virtual": None if multi else busbw(S, t_step, n),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": dict(ck or {}, soak_s=args.soak), "nccl": nccl, "variants": variants,
        }
        print(json.dumps(line), flush=True)
    comm.finalize()
    if multi:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
