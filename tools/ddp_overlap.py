#!/usr/bin/env python
"""Config 5: HaiScale-style DDP — 7.0e9 bf16 gradients in 64 MiB buckets,
allreduced by HFReduce while a synthetic LLaMA-7B-shaped backward runs
(PAPER.md:449-453).  torchrun --nproc-per-node N tools/ddp_overlap.py

Synthetic backward: 32 layers of (wq, wk, wv, wo: 4096x4096; w_gate, w_up:
11008x4096; w_down: 4096x11008; 2 norms) + embedding + lm_head (vocab sized so
the total is exactly 7.0e9 parameters) — per weight one wgrad GEMM
(dW = dY^T X, written straight into the parameter's view of the bucket arena)
and one dgrad GEMM (dX = dY W) over T tokens, in reverse layer order.

Reports (max over ranks, median of --reps):
  T_bwd  backward alone;  T_comm  all bucket allreduces alone;
  T_both backward with the bucketed async allreduce;
  overlap = (T_bwd + T_comm - T_both) / T_comm  (target >= 0.90);
  slowdown = T_both / T_bwd.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

D, FFN, LAYERS, TOTAL = 4096, 11008, 32, 7_000_000_000


def llama7b_layout():
    """(name, out, in) in BACKWARD order, total exactly 7.0e9 elements."""
    layer = [("w_down", D, FFN), ("w_up", FFN, D), ("w_gate", FFN, D), ("wo", D, D), ("wv", D, D),
             ("wk", D, D), ("wq", D, D), ("norm_ffn", 1, D), ("norm_attn", 1, D)]
    per_layer = sum(o * i for _, o, i in layer)
    rest = TOTAL - LAYERS * per_layer - D            # embedding + lm_head + final norm
    vocab = rest // (2 * D)
    pad = rest - 2 * vocab * D
    params = [("lm_head", vocab, D), ("norm_final", 1, D)]
    for li in reversed(range(LAYERS)):
        params += [(f"l{li}.{nm}", o, i) for nm, o, i in layer]
    params.append(("embed", vocab, D))
    if pad:
        params.append(("pad", 1, pad))
    assert sum(o * i for _, o, i in params) == TOTAL
    return params


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--bucket-mib", type=int, default=64)
    ap.add_argument("--max-ctas", type=int, default=32)
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--algo", default="flat")
    ap.add_argument("--layers", type=int, default=LAYERS, help="fewer layers for a quick run")
    ap.add_argument("--gate", type=int, default=1, help="hfr_config.stream_gate")
    ap.add_argument("--threads", type=int, default=256, help="threads per comm CTA (small CTAs can share an SM "
                                                          "with a GEMM CTA)")
    ap.add_argument("--staging", type=int, default=1, help="hfr_config.flat_staging (1 = registers)")
    ap.add_argument("--tail", type=int, default=1, help="1: buckets completed by the last gradient GEMM (embed) "
                                                       "use a full-width config (nothing left to overlap)")
    ap.add_argument("--tail-algo", default="flat")
    ap.add_argument("--clock-phases", type=int, default=0,
                    help="N > 0: afterwards, N backwards alone then N with the allreduces, each block under its own "
                         "clock sampler (does the comm lower the power-capped SM clock?)")
    a = ap.parse_args()

    import torch
    import torch.distributed as dist

    import paper_2408_14158_b200 as hfr
    from paper_2408_14158_b200 import _build
    from paper_2408_14158_b200.ddp import HaiScaleDDP

    _build.build()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    params = llama7b_layout()
    if a.layers != LAYERS:
        keep = {f"l{li}." for li in range(a.layers)}
        params = [p for p in params if not p[0].startswith("l") or p[0][:p[0].index(".") + 1] in keep
                  or p[0].startswith("lm_head")]
    numels = [o * i for _, o, i in params]
    nvls = (TOTAL * 2 + (256 << 20)) if a.algo == "nvls" else 0
    cfg = hfr.Config(algo=a.algo, max_ctas=a.max_ctas, scale=1.0 / world, stream_gate=a.gate, nvls_bytes=nvls,
                     threads=a.threads, flat_staging=a.staging)
    # the comm's own config is the full-width default (T_comm_full); the DDP
    # buckets that overlap the backward use `cfg`
    comm = hfr.Comm.init(device=local, config=hfr.Config(algo=a.algo, scale=1.0 / world, stream_gate=a.gate,
                                                         nvls_bytes=nvls))
    tail_cfg = hfr.Config(algo=a.tail_algo, scale=1.0 / world, stream_gate=a.gate) if a.tail else None
    tail_from = [nm for nm, _, _ in params].index("embed")
    ddp = HaiScaleDDP(comm, numels, torch.bfloat16, bucket_bytes=a.bucket_mib << 20, config=cfg,
                      tail_config=tail_cfg, tail_from=tail_from)
    T = a.tokens
    g = torch.Generator(device=dev).manual_seed(3000 + rank)
    gemm = [(o, i) for _, o, i in params if o > 1 and i <= 65536]
    dY = {o: torch.randn(T, o, device=dev, dtype=torch.bfloat16, generator=g) for o in sorted({o for o, _ in gemm})}
    X = {i: torch.randn(T, i, device=dev, dtype=torch.bfloat16, generator=g) for i in sorted({i for _, i in gemm})}
    W = {oi: torch.randn(*oi, device=dev, dtype=torch.bfloat16, generator=g) * 0.02 for oi in sorted(set(gemm))}
    dX = {i: torch.empty(T, i, device=dev, dtype=torch.bfloat16) for i in X}
    compute = torch.cuda.current_stream()

    def backward(with_comm: bool):
        for idx, (_, o, i) in enumerate(params):
            gv = ddp.grad(idx)
            if o > 1 and i <= 65536:
                torch.matmul(dY[o].t(), X[i], out=gv.view(o, i))      # wgrad into the bucket arena
                torch.matmul(dY[o], W[(o, i)], out=dX[i])              # dgrad (load)
            else:
                gv.fill_(1.0 / (idx + 1))                                      # norms / pad
            if with_comm:
                ddp.mark_ready(idx, compute)
        if with_comm:
            ddp.finish(compute)

    def comm_only():
        for idx in range(len(params)):
            ddp.mark_ready(idx, compute)
        ddp.finish(compute)

    def comm_full():
        """every bucket with the comm's full-width default config"""
        keep = ddp.config, ddp.tail_config
        ddp.config = ddp.tail_config = None
        try:
            comm_only()
        finally:
            ddp.config, ddp.tail_config = keep

    def timed(fn):
        dist.barrier()
        comm.barrier(compute)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(compute)
        fn()
        e1.record(compute)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    backward(True)  # warm-up (cuBLAS heuristics, IPC mappings)
    comm_only()
    from bench import Clocks
    res = {"bwd": [], "comm": [], "both": [], "comm_full": []}
    # interleaved repetitions (bwd, comm, both, bwd, ...) so slow drifts of the
    # power-capped clock hit all three alike; overlap also reported per rep
    ck = Clocks(local, interval_ms=20)
    ck.start()
    for _ in range(a.reps):
        for name, fn in (("bwd", lambda: backward(False)), ("comm", comm_only), ("both", lambda: backward(True)),
                         ("comm_full", comm_full)):
            res[name].append(timed(fn))
    clk = {"all": ck.stop()}
    if a.clock_phases:
        for name, fn in (("bwd_only", lambda: backward(False)), ("bwd_with_comm", lambda: backward(True))):
            c = Clocks(local, interval_ms=20)
            c.start()
            ts = [timed(fn) for _ in range(a.clock_phases)]
            clk[name] = dict(c.stop(), median_ms=statistics.median(ts) * 1e3)
    if comm.status() != hfr.SUCCESS:
        raise SystemExit(hfr.status_string(comm.status()))
    tb, tc, tt, tf = (statistics.median(res[k]) for k in ("bwd", "comm", "both", "comm_full"))
    S = ddp.total * 2
    n = world
    flops = sum(4 * T * o * i for _, o, i in params if o > 1 and i <= 65536)
    if rank == 0:
        print(json.dumps({
            "config": "C5 HaiScale DDP", "n": n, "params": ddp.total, "grad_bytes": S,
            "buckets": len(ddp.bucket_ranges), "bucket_mib": a.bucket_mib, "max_ctas": a.max_ctas, "algo": a.algo,
            "stream_gate": a.gate, "threads": a.threads, "flat_staging": a.staging,
            "tokens": T, "T_bwd_ms": tb * 1e3, "T_comm_ms": tc * 1e3, "T_both_ms": tt * 1e3,
            "overlap": (tb + tc - tt) / tc, "bwd_slowdown": tt / tb,
            "T_comm_full_ms": tf * 1e3,
            # against the full-width allreduce time: 1 - exposed / T_comm_full
            "overlap_vs_full": 1.0 - (tt - tb) / tf, "comm_full_busbw": S / tf * 2 * (n - 1) / n / 1e9,
            "overlap_paired_median": statistics.median((b + c - t) / c for b, c, t in zip(res["bwd"], res["comm"],
                                                                                            res["both"])),
            "overlap_min": (min(res["bwd"]) + min(res["comm"]) - min(res["both"])) / min(res["comm"]),
            "tail": a.tail, "tail_algo": a.tail_algo if a.tail else None, "tail_buckets": sum(1 for m in ddp.bucket_params if a.tail and max(m) >= tail_from),
            "reps_order": "interleaved",
            "comm_busbw": S / tc * 2 * (n - 1) / n / 1e9, "bwd_tflops": flops / tb / 1e12,
            "clocks": clk, "reps": res}), flush=True)
    comm.finalize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
