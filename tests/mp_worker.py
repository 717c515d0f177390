"""Worker body for the multi-process tests (one process per rank).

Run by tests/test_gpu_multi.py (GPU, nccl/gloo over NVLink box) and
tests/test_dist_cpu.py (CPU, gloo) through torch.multiprocessing.spawn.
Each case writes a JSON verdict per rank under `outdir`.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _setup(rank, world, port, backend):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group(backend, rank=rank, world_size=world)


def gpu_cases(rank, world, port, outdir):
    import numpy as np
    import torch
    import torch.distributed as dist

    import hfr_inputs as gen
    import paper_2408_14158_b200 as hfr
    from oracle import hfr_oracle as O
    from tests.gpu_util import assert_bit_exact, assert_within_r18, to_numpy, to_torch, torch_dtype

    torch.cuda.set_device(rank)
    _setup(rank, world, port, "gloo")
    res = {"rank": rank, "ok": [], "fail": []}
    try:
        comm = hfr.Comm.init(device=rank, config=hfr.Config(timeout_ms=8000, chunk_elems=512))
        for dtype in (gen.FP32, gen.BF16, gen.FP16, gen.E4M3, gen.E5M2):
            for algo in ("flat", "oneshot", "dbt", "pair_dbt", "auto", "ce"):
                if algo == "pair_dbt" and world % 2:
                    continue
                for N in (4096 + 13, 1_000_003):
                    for mem in ("symmetric", "plain", "registered"):
                        comm.set_config(hfr.Config(algo=algo, chunk_elems=512, scale=0.5))
                        if dtype in gen.FP8 and mem == "plain":
                            continue  # FP8: symmetric + registered only (keeps the case count down)
                        xs = gen.rank_inputs(world, N, dtype, "normal", seed_base=2000 + N)
                        dt = torch_dtype(dtype)
                        if mem == "symmetric":
                            t = comm.empty(N, dt)
                        else:
                            t = torch.empty(N, dtype=dt, device=f"cuda:{rank}")
                            if mem == "registered":
                                comm.register(t)
                        t.copy_(to_torch(xs[rank], t.device))
                        w = comm.allreduce(t, async_op=(mem != "plain"))
                        if w is not None:
                            w.wait(host=True)
                        torch.cuda.synchronize()
                        got = to_numpy(t)
                        if mem == "registered":
                            comm.deregister(t)
                        want = O.allreduce(xs, algo, chunk_elems=512, scale=0.5)[0]
                        name = f"{algo}/{dtype}/{N}/{mem}"
                        try:
                            assert_bit_exact(got, want, name)
                            # identical bytes on every rank
                            h = hashlib.sha256(got.tobytes()).hexdigest()
                            hs = [None] * world
                            dist.all_gather_object(hs, h)
                            assert len(set(hs)) == 1, f"{name}: ranks differ"
                            res["ok"].append(name)
                        except AssertionError as e:
                            res["fail"].append(str(e)[:500])
        # config 3's largest message (1 GiB bf16 per rank), FLAT, sampled check
        comm.set_config(hfr.Config(algo="flat", scale=1.0 / world))
        N = (1 << 30) // 2
        t = comm.empty(N, torch.bfloat16)
        t.copy_(gen.rank_input_torch(rank, N, gen.BF16, device=f"cuda:{rank}"))
        idx = torch.from_numpy(np.random.default_rng(5).integers(0, N, size=1 << 19)).to(t.device)
        col = to_numpy(t[idx])
        cols = [None] * world
        dist.all_gather_object(cols, col)
        comm.allreduce(t)
        torch.cuda.synchronize()
        try:
            assert_bit_exact(to_numpy(t[idx]), O.fold_ascending(cols, 1.0 / world), "1 GiB bf16 sampled")
            res["ok"].append("1gib")
        except AssertionError as e:
            res["fail"].append(str(e)[:500])
        del t
        # HaiScale DDP: bucketed async allreduce == fold of the arena
        from paper_2408_14158_b200.ddp import HaiScaleDDP
        comm.set_config(hfr.Config(algo="flat", scale=0.5))
        numels = [1000, 70000, 3, 250000, 4097]
        ddp = HaiScaleDDP(comm, numels, torch.bfloat16, bucket_bytes=64 << 10)
        stream = torch.cuda.current_stream()
        xs_all = [gen.rank_input(r, ddp.total, gen.BF16, "normal", seed_base=4000) for r in range(world)]
        for i, (s, e) in enumerate(ddp.param_ranges):
            ddp.grad(i).copy_(to_torch(xs_all[rank][s:e], ddp.arena.device))
            ddp.mark_ready(i, stream)
        ddp.finish(stream)
        torch.cuda.synchronize()
        try:
            assert ddp.stats.launched == len(ddp.bucket_ranges)
            assert_bit_exact(to_numpy(ddp.arena[:ddp.total]), O.fold_ascending(xs_all, 0.5), "ddp")
            res["ok"].append("ddp")
        except AssertionError as e:
            res["fail"].append(str(e)[:500])
        # the same with few small overlap CTAs behind the stream gate and a
        # full-width tail (buckets completed by parameter 3 onwards): the CTA
        # count changes between launches of one comm, bits do not
        ddp2 = HaiScaleDDP(comm, numels, torch.bfloat16, bucket_bytes=64 << 10,
                           config=hfr.Config(algo="flat", scale=0.5, max_ctas=4, threads=128, stream_gate=1,
                                             flat_staging=1),
                           tail_config=hfr.Config(algo="flat", scale=0.5), tail_from=3)
        for step in range(2):
            for i, (s, e) in enumerate(ddp2.param_ranges):
                ddp2.grad(i).copy_(to_torch(xs_all[rank][s:e], ddp2.arena.device))
                ddp2.mark_ready(i, stream)
            ddp2.finish(stream)
            torch.cuda.synchronize()
            try:
                assert 0 < ddp2.stats.tail < ddp2.stats.launched, (ddp2.stats.tail, ddp2.stats.launched)
                assert_bit_exact(to_numpy(ddp2.arena[:ddp2.total]), O.fold_ascending(xs_all, 0.5), "ddp tail")
                res["ok"].append(f"ddp-tail-{step}")
            except AssertionError as e:
                res["fail"].append(str(e)[:500])
        comm.set_config(hfr.Config(algo="flat", scale=0.5))
        # the other collectives (NEXT-3), one rank per GPU
        comm.set_config(hfr.Config(scale=0.5))
        for kind in ("reduce_scatter", "allgather", "reduce", "broadcast"):
            for dtype in (gen.FP32, gen.BF16):
                N = 200_003
                xs = gen.rank_inputs(world, N, dtype, "normal", seed_base=6000 + N)
                t = comm.empty(N, torch_dtype(dtype))
                t.copy_(to_torch(xs[rank], t.device))
                comm.collective(kind, t, root=1)
                torch.cuda.synchronize()
                want = {"reduce_scatter": lambda: O.reduce_scatter(xs, 0.5), "allgather": lambda: O.all_gather(xs),
                        "reduce": lambda: O.reduce(xs, 1, 0.5), "broadcast": lambda: O.broadcast(xs, 1)}[kind]()
                try:
                    assert_bit_exact(to_numpy(t), want[rank], f"{kind}/{dtype}")
                    res["ok"].append(f"{kind}/{dtype}")
                except AssertionError as e:
                    res["fail"].append(str(e)[:500])
        # protocol mismatch: different counts (same grid) -> PROTOCOL on every rank
        comm.set_config(hfr.Config(algo="flat"))
        t = comm.empty(8192, torch.float32)
        try:
            w = comm.allreduce(t[: 4096 + (rank % 2)], async_op=True)
            w.wait(host=True)
            res["fail"].append("protocol mismatch not detected")
        except hfr.HfrError as e:
            if e.status == hfr.ERR_PROTOCOL:
                res["ok"].append("protocol")
            else:
                res["fail"].append(f"protocol: got {e}")
        comm.finalize()
        # argument mismatches that change the grid (4096 vs 4 Mi elements) or
        # even the kernel (AUTO: LL ONESHOT on one rank, FLAT on the other):
        # PROTOCOL within a fraction of the timeout, never TIMEOUT
        import time
        for algo in ("flat", "auto"):
            pc = hfr.Comm.init(device=rank, config=hfr.Config(algo=algo, timeout_ms=20000))
            t = pc.empty(4 << 20, torch.float32)
            cnt = 4096 if rank % 2 == 0 else (4 << 20)
            t0 = time.time()
            try:
                pc.allreduce(t[:cnt], async_op=True).wait(host=True)
                res["fail"].append(f"protocol-{algo}: mismatch not detected")
            except hfr.HfrError as e:
                dt_s = time.time() - t0
                if e.status == hfr.ERR_PROTOCOL and dt_s < 10:
                    res["ok"].append(f"protocol-grid-{algo}")
                else:
                    res["fail"].append(f"protocol-{algo}: got {e} after {dt_s:.1f} s")
            dist.barrier()
            pc.finalize()
        # NVLS order-relaxed path (reading R18 bound), if the box has multicast
        comm = hfr.Comm.init(device=rank, config=hfr.Config(timeout_ms=8000, nvls_bytes=64 << 20, algo="nvls",
                                                            scale=0.5))
        for dtype in (gen.FP32, gen.BF16, gen.FP16):
            for N in (4096 + 13, 1_000_003):
                for dist_name in ("normal", "int"):
                    xs = gen.rank_inputs(world, N, dtype, dist_name, seed_base=5000 + N)
                    t = comm.empty(N, torch_dtype(dtype))
                    t.copy_(to_torch(xs[rank], t.device))
                    name = f"nvls/{dtype}/{N}/{dist_name}"
                    try:
                        comm.allreduce(t)
                    except hfr.HfrError as e:
                        if e.status == hfr.ERR_UNSUPPORTED:
                            res["ok"].append("nvls-unsupported")
                            break
                        raise
                    torch.cuda.synchronize()
                    got = to_numpy(t)
                    want = O.fold_ascending(xs, 0.5)
                    try:
                        if dist_name == "int" and dtype == gen.FP32:
                            assert_bit_exact(got, want, name)  # exact fp32 sums: every order agrees
                        else:
                            assert_within_r18(got, xs, want, 0.5, name)
                        h = hashlib.sha256(got.tobytes()).hexdigest()
                        hs = [None] * world
                        dist.all_gather_object(hs, h)
                        assert len(set(hs)) == 1, f"{name}: ranks differ"
                        res["ok"].append(name)
                    except AssertionError as e:
                        res["fail"].append(str(e)[:500])
        # the other collectives on the multicast object: all-gather and
        # broadcast move raw bits (bit-exact); reduce-scatter and reduce are
        # order-relaxed on their reduced region (R18) and bit-exact elsewhere
        if "nvls-unsupported" not in res["ok"]:
            for dtype in (gen.FP32, gen.BF16):
                for N in (4096 + 13, 1_000_003):
                    xs = gen.rank_inputs(world, N, dtype, "normal", seed_base=6100 + N)
                    t = comm.empty(N, torch_dtype(dtype))
                    for kind in ("reduce_scatter", "allgather", "reduce", "broadcast"):
                        for root in ((0, world - 1) if kind in ("reduce", "broadcast") else (0,)):
                            t.copy_(to_torch(xs[rank], t.device))
                            comm.collective(kind, t, root=root)
                            torch.cuda.synchronize()
                            got = to_numpy(t)
                            name = f"nvls-{kind}/{dtype}/{N}/root{root}"
                            try:
                                if kind == "allgather":
                                    assert_bit_exact(got, O.all_gather(xs)[rank], name)
                                elif kind == "broadcast":
                                    assert_bit_exact(got, O.broadcast(xs, root)[rank], name)
                                else:
                                    if kind == "reduce":
                                        lo, hi = (0, N) if rank == root else (0, 0)
                                    else:
                                        lo, hi = O.shard_bounds(N, world, 4 if dtype == gen.FP32 else 8)[rank]
                                    want = O.fold_ascending(xs, 0.5)
                                    keep = np.ones(N, bool)
                                    keep[lo:hi] = False
                                    assert_bit_exact(got[keep], xs[rank][keep], name + "/untouched")
                                    if hi > lo:
                                        assert_within_r18(got[lo:hi], [x[lo:hi] for x in xs], want[lo:hi], 0.5, name)
                                res["ok"].append(name)
                            except AssertionError as e:
                                res["fail"].append(str(e)[:500])
        # every other schedule also runs zero-copy on NVLS arena memory
        comm.set_config(hfr.Config(algo="flat", scale=0.5))
        xs = gen.rank_inputs(world, 100_000, gen.FP32, "normal", seed_base=77)
        t = comm.empty(100_000, torch.float32)
        t.copy_(to_torch(xs[rank], t.device))
        comm.allreduce(t)
        torch.cuda.synchronize()
        try:
            assert_bit_exact(to_numpy(t), O.fold_ascending(xs, 0.5), "flat-on-nvls-arena")
            res["ok"].append("flat-on-nvls-arena")
        except AssertionError as e:
            res["fail"].append(str(e)[:500])
        comm.finalize()
        # module-level API (hfr.init(group) / hfr.allreduce / hfr.finalize)
        m = hfr.init(device=rank, config=hfr.Config(scale=0.5))
        xs = gen.rank_inputs(world, 70_001, gen.BF16, "normal", seed_base=88)
        t = m.empty(70_001, torch.bfloat16)
        t.copy_(to_torch(xs[rank], t.device))
        hfr.allreduce(t, async_op=True).wait()
        torch.cuda.synchronize()
        try:
            assert_bit_exact(to_numpy(t), O.fold_ascending(xs, 0.5), "module-api")
            res["ok"].append("module-api")
        except AssertionError as e:
            res["fail"].append(str(e)[:500])
        hfr.finalize()
        # timeout: rank 0 calls alone
        comm = hfr.Comm.init(device=rank, config=hfr.Config(timeout_ms=1500))
        t = comm.empty(4096, torch.float32)
        if rank == 0:
            try:
                comm.allreduce(t, async_op=True).wait(host=True)
                res["fail"].append("timeout not detected")
            except hfr.HfrError as e:
                (res["ok"] if e.status == hfr.ERR_TIMEOUT else res["fail"]).append(f"timeout:{e.status}")
        else:
            res["ok"].append("timeout-skip")
        dist.barrier()
        comm.finalize()
    except Exception:  # noqa: BLE001
        res["fail"].append(traceback.format_exc()[-2000:])
    with open(os.path.join(outdir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)
    dist.destroy_process_group()


def cpu_exchange_case(rank, world, port, outdir):
    """Host-side logic of the N>1 path on CPU: the IPC-handle all-gather
    callback libhfr uses during hfr_init/hfr_mem_alloc, over gloo."""
    import ctypes

    import torch.distributed as dist

    import paper_2408_14158_b200 as hfr
    _setup(rank, world, port, "gloo")
    res = {"rank": rank, "ok": [], "fail": []}
    try:
        cb = hfr._AG_FN(hfr._torch_allgather(None))
        for nbytes in (1, 64, 80, 4096):
            send = (ctypes.c_uint8 * nbytes)(*[(rank * 31 + i) & 0xFF for i in range(nbytes)])
            recv = (ctypes.c_uint8 * (nbytes * world))()
            rc = cb(ctypes.addressof(send), ctypes.addressof(recv), nbytes, None)
            assert rc == 0
            for q in range(world):
                exp = [(q * 31 + i) & 0xFF for i in range(nbytes)]
                assert list(recv[q * nbytes:(q + 1) * nbytes]) == exp
            res["ok"].append(nbytes)
    except Exception:  # noqa: BLE001
        res["fail"].append(traceback.format_exc()[-2000:])
    with open(os.path.join(outdir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)
    dist.destroy_process_group()


def entry(rank, world, port, outdir, case):
    {"gpu": gpu_cases, "cpu_exchange": cpu_exchange_case}[case](rank, world, port, outdir)
