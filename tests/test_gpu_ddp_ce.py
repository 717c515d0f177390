"""GPU parity on ONE B200 for the §8 rows that round 1 only exercised across
several GPUs (VERDICT r01 "next round" 1a/1b):

  a6  HaiScale-DDP bucketed overlap on a VIRTUAL comm:
      one arena per virtual rank, every bucket reduced by
      hfr_allreduce_virtual as the "backward" marks its gradients ready,
      with separate overlap / tail configs — bit-exact against the oracle's
      rank-ascending fold on every bucket, two steps;
  NEXT-2  the copy-engine schedule ("No GPU Kernel Overhead")
      for real on virtual ranks: cudaMemcpyAsync pulls between the ranks'
      buffers, stream-memop flags, the local fold kernel;
  a real nranks = 1 comm (hfr_init without peers): the PDL launch path of the
      latency-bound kernels, barrier, back-to-back calls on several streams;
  issue order (include/hfr.h): calls on different streams never overlap.
"""
from __future__ import annotations

import numpy as np
import pytest

import hfr_inputs as gen
from oracle import hfr_oracle as O
from tests.gpu_util import assert_bit_exact, to_numpy, to_torch, torch_dtype

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def hfr():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2408_14158_b200 as m
    from paper_2408_14158_b200 import _build
    _build.build()
    return m


def _layout(layers=3, d=256, ffn=688):
    """A LLaMA-shaped parameter list in backward order (C5's structure at
    small width): per layer down/up/gate/o/v/k/q projections and two norms,
    then the embedding; sizes are deliberately not bucket multiples."""
    numels = []
    for _ in range(layers):
        numels += [ffn * d, ffn * d, ffn * d, d * d, d * d, d * d, d * d, d, d]
    numels += [d, 1000 * d + 3]  # final norm, embedding (ragged)
    return numels


def _fill_grads(ddp, xs, stream):
    """The synthetic 'backward': write each parameter's gradient (all virtual
    ranks) on `stream` in backward order and mark it ready."""
    with torch.cuda.stream(stream):
        for i, (s, e) in enumerate(ddp.param_ranges):
            views = ddp.grad(i)
            views = views if isinstance(views, list) else [views]
            for v, x in zip(views, xs):
                v.copy_(to_torch(x[s:e], v.device), non_blocking=False)
            ddp.mark_ready(i, stream)
        ddp.finish(stream)


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("overlap_algo", ["flat", "ce", "dbt"])
def test_ddp_virtual_bit_exact(hfr, n, overlap_algo):
    """a6 on one GPU: C5-shaped bucket plan (ragged parameters and a ragged
    last bucket), small register-staged overlap CTAs behind the overlap
    config, a full-width tail config from the embedding on, two steps; every
    bucket bit-exact vs the oracle's fold of that bucket (FLAT / CE: the
    rank-ascending fold; DBT: the tree-order fold of the bucket)."""
    from paper_2408_14158_b200.ddp import HaiScaleDDP
    comm = hfr.Comm.virtual_ranks(n, 0, hfr.Config(scale=1.0 / n, timeout_ms=10000))
    try:
        numels = _layout()
        overlap = HaiScaleDDP.derive(comm, algo=overlap_algo, max_ctas=8, threads=128, flat_staging=1,
                                     chunk_elems=1024)
        tail = HaiScaleDDP.derive(comm, algo="flat")
        ddp = HaiScaleDDP(comm, numels, torch.bfloat16, bucket_bytes=256 << 10, config=overlap,
                          tail_config=tail, tail_from=len(numels) - 1)
        assert ddp.virtual and len(ddp.arenas) == n
        assert len(ddp.bucket_ranges) > 8 and ddp.bucket_ranges[-1][1] - ddp.bucket_ranges[-1][0] < ddp.bucket_elems
        stream = torch.cuda.Stream()
        for step in range(2):
            xs = gen.rank_inputs(n, ddp.total, gen.BF16, "normal", seed_base=4000 + 17 * step)
            _fill_grads(ddp, xs, stream)
            torch.cuda.synchronize()
            assert comm.status() == hfr.SUCCESS, hfr.status_string(comm.status())
            assert comm.config is ddp.base
            assert 0 < ddp.stats.tail < ddp.stats.launched
            outs = [to_numpy(a[:ddp.total]) for a in ddp.arenas]
            for k, (s, e) in enumerate(ddp.bucket_ranges):
                tail_bucket = max(ddp.bucket_params[k]) >= ddp.tail_from
                algo = "flat" if tail_bucket else overlap_algo
                want = O.allreduce([x[s:e] for x in xs], "flat" if algo == "ce" else algo, chunk_elems=1024,
                                   scale=1.0 / n)[0]
                for r in range(n):
                    assert_bit_exact(outs[r][s:e], want, f"step {step} bucket {k} ({algo}) rank {r}")
        comm.free_all()
    finally:
        comm.finalize()


def test_ddp_c5_full_size_sampled(hfr):
    """C5 at full size (7e9 bf16 gradients per rank in 64 MiB buckets: 208
    full + 1 ragged) on 8 virtual ranks (4 if the GPU lacks the memory),
    the tools/ddp_overlap.py layout and tail; 2^20 sampled elements per step
    bit-exact vs the oracle, and every rank's arena byte-identical."""
    import tools.ddp_overlap as d
    from paper_2408_14158_b200.ddp import HaiScaleDDP
    free, _ = torch.cuda.mem_get_info()
    n = 8 if free > 8 * 14.2e9 + 6e9 else 4
    if free < 4 * 14.2e9 + 4e9:
        pytest.skip(f"needs ~61 GB free, have {free / 1e9:.0f} GB")
    params = d.llama7b_layout()
    numels = [o * i for _, o, i in params]
    tail_from = [nm for nm, _, _ in params].index("embed")
    comm = hfr.Comm.virtual_ranks(n, 0, hfr.Config(scale=1.0 / n, timeout_ms=20000))
    try:
        overlap = HaiScaleDDP.derive(comm, algo="flat", max_ctas=32, threads=128, flat_staging=1)
        ddp = HaiScaleDDP(comm, numels, torch.bfloat16, bucket_bytes=gen.C5_BUCKET_BYTES, config=overlap,
                          tail_config=HaiScaleDDP.derive(comm, algo="flat"), tail_from=tail_from)
        assert ddp.total == gen.C5_PARAMS and len(ddp.bucket_ranges) == 209
        idx = torch.from_numpy(np.random.default_rng(11).integers(0, ddp.total, size=1 << 20)).cuda()
        idx[:4] = torch.tensor([0, ddp.total - 1, ddp.bucket_elems - 1, ddp.bucket_elems], device="cuda")
        CH = 1 << 28
        stream = torch.cuda.current_stream()
        for step in range(2):
            for r, a in enumerate(ddp.arenas):  # seeded synthetic gradients, generated on the device in chunks
                g = torch.Generator(device="cuda")
                for c0 in range(0, ddp.total, CH):
                    g.manual_seed(90_000 + 1000 * step + 31 * r + c0 // CH)
                    m = min(CH, ddp.total - c0)
                    x = torch.randn(m, generator=g, device="cuda", dtype=torch.float32)
                    a[c0:c0 + m].copy_((x.view(torch.int32) >> 16).to(torch.int16).view(torch.bfloat16))
                    del x
            cols = [to_numpy(a[idx]) for a in ddp.arenas]
            for i in range(len(numels)):
                ddp.mark_ready(i, stream)
            ddp.finish(stream)
            torch.cuda.synchronize()
            assert comm.status() == hfr.SUCCESS, hfr.status_string(comm.status())
            assert ddp.stats.tail == 9 * (step + 1)
            want = O.fold_ascending(cols, 1.0 / n)
            for r, a in enumerate(ddp.arenas):
                assert_bit_exact(to_numpy(a[idx]), want, f"C5 step {step} rank {r}")
            for a in ddp.arenas[1:]:
                assert torch.equal(a.view(torch.int16), ddp.arenas[0].view(torch.int16))
        comm.free_all()
    finally:
        comm.finalize()


# ---------------------------------------------------------------------------
# NEXT-2: the copy-engine schedule on virtual ranks
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype", [gen.FP32, gen.BF16, gen.FP16])
@pytest.mark.parametrize("N", [16_384 * 8 + 13, 1_000_003, 9_437_201])
@pytest.mark.parametrize("mem", ["symmetric", "unaligned"])
def test_ce_virtual(hfr, n, dtype, N, mem):
    """CE: copy-engine pulls (one cudaMemcpyAsync per copy), stream-memop
    ready/done/exit flags, local fold — bit-exact vs the rank-ascending fold.
    9.4 M fp32 elements at n=2 give 2 pipeline chunks per shard; 'unaligned'
    buffers (one element off 16 B) are staged through the scratch first."""
    comm = hfr.Comm.virtual_ranks(n, 0, hfr.Config(algo="ce", scale=0.5, timeout_ms=10000))
    try:
        launches0 = comm.launches
        xs = gen.rank_inputs(n, N, dtype, "normal", seed_base=800 + N)
        dt = torch_dtype(dtype)
        if mem == "symmetric":
            bufs = comm.empty(N, dt)
        else:
            bufs = [torch.empty(N + 1, dtype=dt, device="cuda:0")[1:] for _ in range(n)]
        for b, x in zip(bufs, xs):
            b.copy_(to_torch(x, "cuda:0"))
        comm.allreduce_virtual(bufs)
        torch.cuda.synchronize()
        assert comm.status() == hfr.SUCCESS, hfr.status_string(comm.status())
        want = O.fold_ascending(xs, 0.5)
        for r, b in enumerate(bufs):
            assert_bit_exact(to_numpy(b), want, f"ce n={n} rank {r}")
        # the SMs ran one fold kernel per rank and pipeline chunk (+ the
        # staging copies for plain memory), not the single FLAT launch
        launched = comm.launches - launches0 - (2 * n if mem == "unaligned" else 0)
        assert launched >= n, launched
    finally:
        comm.finalize()


def test_ce_virtual_async_and_repeated(hfr):
    """CE asynchronous (side stream) and 5 back-to-back calls in place: the
    result is the oracle applied 5 times (stream-memop epochs advance)."""
    n, N = 4, 300_001
    comm = hfr.Comm.virtual_ranks(n, 0, hfr.Config(algo="ce", scale=0.25, timeout_ms=10000))
    try:
        xs = gen.rank_inputs(n, N, gen.FP32, "normal", seed_base=5)
        bufs = comm.empty(N, torch.float32)
        for b, x in zip(bufs, xs):
            b.copy_(to_torch(x, "cuda:0"))
        want = xs
        for _ in range(5):
            comm.allreduce_virtual(bufs, async_op=True).wait()
            want = [O.fold_ascending(want, 0.25)] * n
        torch.cuda.synchronize()
        assert comm.status() == hfr.SUCCESS
        for r, b in enumerate(bufs):
            assert_bit_exact(to_numpy(b), want[0], f"ce repeated rank {r}")
    finally:
        comm.finalize()


# ---------------------------------------------------------------------------
# a real comm with nranks = 1 (PDL launches, barrier, DDP tail) — ADVICE r01
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("pdl_off", [0, 1])
def test_real_single_rank_sequence(hfr, pdl_off):
    """hfr_init with nranks = 1: AUTO (LL ONESHOT, programmatic dependent
    launch), explicit ONESHOT (fenced form), FLAT, DBT, CE (-> FLAT at n=1),
    barriers in between, on two streams, sync and async, back to back; every
    result bit-exact vs the oracle (n = 1: scale and cast), and the same with
    PDL off."""
    comm = hfr.Comm.single(0, hfr.Config(scale=0.5, pdl_off=pdl_off, timeout_ms=10000))
    try:
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        plan = [("auto", 3001, s1, False), ("oneshot", 200_003, s2, True), ("flat", 1_000_003, s1, False),
                ("dbt", 77_777, s2, True), ("ce", 400_001, s1, True), ("auto", 17, s2, False),
                ("pair_dbt", 5000, s1, False)]
        outs = []
        for i, (algo, N, st, async_op) in enumerate(plan):
            comm.set_config(hfr.Config(algo=algo, scale=0.5, pdl_off=pdl_off, timeout_ms=10000, chunk_elems=512))
            x = gen.rank_input(0, N, gen.BF16, "normal", seed_base=60 + i)
            t = comm.empty(N, torch.bfloat16) if i % 2 else torch.empty(N, dtype=torch.bfloat16, device="cuda:0")
            t.copy_(to_torch(x, "cuda:0"))
            torch.cuda.synchronize()
            try:
                w = comm.allreduce(t, async_op=async_op, stream=st)
            except hfr.HfrError as e:
                assert algo == "pair_dbt" and e.status == hfr.ERR_UNSUPPORTED  # pair-first needs even n
                continue
            if w is not None:
                w.wait(stream=st)
            comm.barrier(s2)
            outs.append((t, x, algo))
        torch.cuda.synchronize()
        assert comm.status() == hfr.SUCCESS
        for t, x, algo in outs:
            assert_bit_exact(to_numpy(t), O.fold_ascending([x], 0.5), f"n=1 {algo}")
        comm.free_all()
    finally:
        comm.finalize()


def test_real_single_rank_ddp_tail(hfr):
    """HaiScaleDDP on a real nranks = 1 comm with overlap and tail configs."""
    from paper_2408_14158_b200.ddp import HaiScaleDDP
    comm = hfr.Comm.single(0, hfr.Config(scale=0.5))
    try:
        numels = _layout(layers=1)
        ddp = HaiScaleDDP(comm, numels, torch.bfloat16, bucket_bytes=64 << 10,
                          config=HaiScaleDDP.derive(comm, max_ctas=4, threads=128, flat_staging=1),
                          tail_config=HaiScaleDDP.derive(comm), tail_from=len(numels) - 2)
        stream = torch.cuda.Stream()
        for step in range(2):
            xs = gen.rank_inputs(1, ddp.total, gen.BF16, "normal", seed_base=70 + step)
            _fill_grads(ddp, xs, stream)
            torch.cuda.synchronize()
            assert_bit_exact(to_numpy(ddp.arena[:ddp.total]), O.fold_ascending(xs, 0.5), f"n=1 ddp step {step}")
        assert 0 < ddp.stats.tail < ddp.stats.launched
        assert comm.status() == hfr.SUCCESS
    finally:
        comm.finalize()


# ---------------------------------------------------------------------------
# issue order across streams
# ---------------------------------------------------------------------------
def test_calls_on_different_streams_never_overlap(hfr):
    """Two synchronous allreduces on two streams, then an async one and a
    barrier, enqueued without any user synchronisation: include/hfr.h promises
    issue order, so each result is exact (overlapping kernels would share the
    pad's epoch, tile counter and scratch and corrupt each other)."""
    n = 4
    comm = hfr.Comm.virtual_ranks(n, 0, hfr.Config(algo="flat", scale=0.25, timeout_ms=10000))
    try:
        streams = [torch.cuda.Stream() for _ in range(3)]
        sizes = [3_000_017, 2_500_001, 4_000_037, 999_999]
        cases = []
        for j, N in enumerate(sizes):
            xs = gen.rank_inputs(n, N, gen.FP32, "normal", seed_base=900 + j)
            bufs = comm.empty(N, torch.float32)
            for b, x in zip(bufs, xs):
                b.copy_(to_torch(x, "cuda:0"))
            cases.append((bufs, xs))
        torch.cuda.synchronize()
        for rep in range(3):
            for j, (bufs, xs) in enumerate(cases):
                st = streams[j % 3]
                w = comm.allreduce_virtual(bufs, async_op=(j == 2), stream=st)
                if j == 2:
                    comm.barrier(streams[(j + 1) % 3])
                    w.wait(stream=st)
        torch.cuda.synchronize()
        assert comm.status() == hfr.SUCCESS
        for j, (bufs, xs) in enumerate(cases):
            want = xs
            for _ in range(3):
                want = [O.fold_ascending(want, 0.25)] * n
            for r, b in enumerate(bufs):
                assert_bit_exact(to_numpy(b), want[0], f"stream-order case {j} rank {r}")
    finally:
        comm.finalize()
