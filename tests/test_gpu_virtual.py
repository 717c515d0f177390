"""GPU parity tests, one B200, n VIRTUAL ranks (hfr_init_virtual): the same
kernels and cross-rank protocol as the multi-GPU path, with every rank's CTAs
in one cooperative launch.  Every result is compared element by element with
the CPU oracle on the same seeded inputs: bit-exact (NaN payloads excepted,
reading R5) for the order the schedule implements (FLAT -> rank-ascending
fold, DBT -> tree-order fold, PAIR_DBT -> pair-first fold)."""
from __future__ import annotations

import numpy as np
import pytest

import hfr_inputs as gen
from oracle import hfr_oracle as O
from tests.gpu_util import assert_bit_exact, dtype_of, to_numpy, to_torch, torch_dtype

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


_COMMS = {}


def comm_for(hfr, n):
    if n not in _COMMS:
        _COMMS[n] = hfr.Comm.virtual_ranks(n, 0, hfr.Config(timeout_ms=10000))
    return _COMMS[n]


def run(hfr, n, xs, algo, chunk=512, scale=1.0, symmetric=True, offset=0, async_op=False):
    comm = comm_for(hfr, n)
    comm.set_config(hfr.Config(algo=algo, chunk_elems=chunk, scale=scale))
    dt = torch_dtype(dtype_of(xs[0]))
    N = xs[0].shape[0]
    if symmetric:
        bufs = [b[offset:offset + N] for b in comm.empty(N + offset, dt)]
    else:
        bufs = [torch.empty(N + offset, dtype=dt, device="cuda:0")[offset:] for _ in range(n)]
    for b, x in zip(bufs, xs):
        b.copy_(to_torch(x, "cuda:0"))
    w = comm.allreduce_virtual(bufs, async_op=async_op)
    if w is not None:
        w.wait(host=True)
    torch.cuda.synchronize()
    assert comm.status() == hfr.SUCCESS, hfr.status_string(comm.status())
    return [to_numpy(b) for b in bufs]


def check(outs, want, what):
    for r, g in enumerate(outs):
        assert_bit_exact(g, want, f"{what} rank {r}")


ALGOS = ["flat", "oneshot", "dbt", "pair_dbt"]


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("dtype", [gen.FP32, gen.BF16, gen.FP16])
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("N", [1, 7, 4096, 4096 + 13, 100_003])
def test_parity_sizes(hfr, n, dtype, algo, N):
    if algo == "pair_dbt" and n % 2:
        pytest.skip("pair-first needs even n")
    xs = gen.rank_inputs(n, N, dtype, "normal", seed_base=1000 + N)
    outs = run(hfr, n, xs, algo, chunk=512)
    check(outs, O.allreduce(xs, algo, chunk_elems=512)[0], f"{algo} n={n} {dtype} N={N}")


@pytest.mark.parametrize("dist", ["specials", "int", "loguniform", "grad"])
@pytest.mark.parametrize("dtype", [gen.FP32, gen.BF16, gen.FP16])
@pytest.mark.parametrize("algo", ALGOS)
def test_parity_distributions(hfr, dist, dtype, algo):
    n, N = 8, 3 * 4096 + 5
    xs = gen.rank_inputs(n, N, dtype, dist, seed_base=77)
    outs = run(hfr, n, xs, algo, chunk=256, scale=0.125)
    check(outs, O.allreduce(xs, algo, chunk_elems=256, scale=0.125)[0], f"{algo} {dist} {dtype}")


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("scale", [0.1, 3.0, -0.5, 0.0, float("inf")])
def test_parity_scale(hfr, algo, scale):
    xs = gen.rank_inputs(4, 20_000, gen.FP32, "normal", seed_base=5)
    outs = run(hfr, 4, xs, algo, chunk=1024, scale=scale)
    check(outs, O.allreduce(xs, algo, chunk_elems=1024, scale=scale)[0], f"{algo} scale={scale}")


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("dtype", [gen.FP32, gen.BF16])
def test_staged_unaligned_and_plain_memory(hfr, algo, dtype):
    """Buffers outside symmetric memory or not 16-B aligned take the staged path."""
    xs = gen.rank_inputs(4, 10_001, dtype, "normal", seed_base=9)
    want = O.allreduce(xs, algo, chunk_elems=512)[0]
    check(run(hfr, 4, xs, algo, symmetric=False), want, "plain torch memory")
    check(run(hfr, 4, xs, algo, symmetric=True, offset=1), want, "unaligned")


@pytest.mark.parametrize("algo", ALGOS)
def test_async_request(hfr, algo):
    xs = gen.rank_inputs(2, 50_000, gen.BF16, "loguniform", seed_base=3)
    outs = run(hfr, 2, xs, algo, async_op=True)
    check(outs, O.allreduce(xs, algo, chunk_elems=512)[0], "async")


def test_zero_count_is_noop(hfr):
    comm = comm_for(hfr, 2)
    comm.set_config(hfr.Config())
    bufs = comm.empty(16, torch.float32)
    before = comm.launches
    comm.allreduce_virtual([b[:0] for b in bufs])
    assert comm.launches == before


@pytest.mark.parametrize("algo", ALGOS)
def test_golden_order_examples_on_gpu(hfr, algo):
    """The hand-derived order examples of tests/golden/order_examples.json,
    run through the kernels (chunk_elems is 256-aligned on the GPU, so each
    example is replicated to 256-element chunks)."""
    import json
    import os
    cases = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "order_examples.json")))["cases"]
    for case in cases:
        if case["algo"] != algo and not (algo == "oneshot" and case["algo"] == "flat"):
            continue
        xs0 = [np.array(v, dtype=np.float32) for v in case["inputs"]]
        # element j of the example -> chunk j (256 elements each, all equal)
        xs = [np.repeat(x, 256) for x in xs0]
        outs = run(hfr, len(xs), xs, algo, chunk=256, scale=case.get("scale", 1.0))
        want = np.repeat(np.array(case["expected"], dtype=np.float32), 256)
        if algo == "pair_dbt":
            # the pair split puts the second half at H; chunks restart there
            want = O.allreduce(xs, algo, chunk_elems=256, scale=case.get("scale", 1.0))[0]
        check(outs, want, case["name"])


@pytest.mark.parametrize("algo", ALGOS)
def test_c2_full_size(hfr, algo):
    """Config 2 at full size: 8 ranks x 186 MiB fp32 (48,758,784 elements),
    gradient-like values, plus an odd N — bit-exact on every element."""
    n = 8
    for N in (gen.C2_COUNT, gen.C2_COUNT + 1):
        xs = gen.rank_inputs(n, N, gen.FP32, "grad", seed_base=1000)
        outs = run(hfr, n, xs, algo, chunk=8192)
        want = O.allreduce(xs, algo, chunk_elems=8192)[0]
        check(outs, want, f"C2 {algo} N={N}")
        for o in outs[1:]:
            assert np.array_equal(o.view(np.uint32), outs[0].view(np.uint32))
        del outs, xs
        comm_for(hfr, n).free_all()


def test_bf16_exhaustive_n2_sample(hfr):
    """n=2 bf16: result = RNE_bf16(fl32(a)+fl32(b)) (library case) over a
    2^24 sample of (a, b) bit pairs incl. specials."""
    rng = np.random.default_rng(0)
    a = rng.integers(0, 1 << 16, size=1 << 24, dtype=np.uint32).astype(np.uint16)
    b = rng.integers(0, 1 << 16, size=1 << 24, dtype=np.uint32).astype(np.uint16)
    outs = run(hfr, 2, [a, b], "flat")
    fa, fb = O.widen(a), O.widen(b)
    want = torch.from_numpy(fa + fb).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    check(outs, want, "bf16 n=2")


def test_bf16_exhaustive_n2_all_pairs(hfr):
    """SURVEY §8(c) "bf16 exhaustive": at n=2 EVERY (a, b) pair of bf16 bit
    patterns (2^32 pairs, incl. NaN/Inf/subnormals/signed zeros) through the
    FLAT kernel bench.py times, against the C oracle's rank-ascending fold,
    in 16 slices of 2^28 pairs (512 MiB per rank each).  NaN payloads are
    not compared (reading R5)."""
    from oracle import cfold
    comm = comm_for(hfr, 2)
    comm.set_config(hfr.Config(algo="flat"))
    M = 1 << 28
    bufs = comm.empty(M, torch.bfloat16)

    def isnan16(u):
        return ((u & 0x7F80) == 0x7F80) & ((u & 0x7F) != 0)

    idx = np.arange(M, dtype=np.uint32)
    for sl in range(16):
        i = idx + np.uint32(sl * M)
        a = (i >> np.uint32(16)).astype(np.uint16)
        b = (i & np.uint32(0xFFFF)).astype(np.uint16)
        for buf, x in zip(bufs, (a, b)):
            buf.copy_(to_torch(x, "cuda:0"))
        comm.allreduce_virtual(bufs)
        torch.cuda.synchronize()
        assert comm.status() == hfr.SUCCESS
        want = cfold.fold_ascending([a, b])
        for r, buf in enumerate(bufs):
            got = to_numpy(buf)
            ok = (got == want) | (isnan16(got) & isnan16(want))
            bad = np.flatnonzero(~ok)
            assert bad.size == 0, (f"slice {sl} rank {r}: {bad.size} pairs differ, first (a,b)="
                                   f"{[(int(a[k]), int(b[k])) for k in bad[:4]]}")
    comm.free_all()


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("N", [2_003, 20_003])
def test_cuda_graph_replay(hfr, algo, N):
    """Captured allreduces replay correctly (device-side launch epochs): k
    replays of one captured in-place allreduce == the oracle applied k times.
    N=2003 runs ONESHOT's LL (flag-in-data) form, N=20003 the fenced form."""
    n = 4
    comm = comm_for(hfr, n)
    comm.set_config(hfr.Config(algo=algo, chunk_elems=512, scale=0.25))
    xs = gen.rank_inputs(n, N, gen.FP32, "normal", seed_base=66)
    bufs = comm.empty(N, torch.float32)
    for b, x in zip(bufs, xs):
        b.copy_(to_torch(x, "cuda:0"))
    comm.allreduce_virtual(bufs)          # uncaptured first call (sizes the scratch)
    torch.cuda.synchronize()
    want = O.allreduce(xs, algo, chunk_elems=512, scale=0.25)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            comm.allreduce_virtual(bufs)
    for _ in range(3):
        g.replay()
        want = O.allreduce(want, algo, chunk_elems=512, scale=0.25)
    torch.cuda.synchronize()
    assert comm.status() == hfr.SUCCESS
    check([to_numpy(b) for b in bufs], want[0], f"graph {algo}")


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("dtype", [gen.FP32, gen.BF16, gen.FP16])
@pytest.mark.parametrize("kind", ["reduce_scatter", "allgather", "reduce", "broadcast", "allreduce"])
@pytest.mark.parametrize("N", [5, 4096 + 13, 300_007])
def test_collectives(hfr, n, dtype, kind, N):
    """NEXT-3: the other collectives, bit-exact vs the oracle (whole buffers,
    including the parts a collective must leave unchanged)."""
    comm = comm_for(hfr, n)
    comm.set_config(hfr.Config(scale=0.5))
    root = n - 1
    xs = gen.rank_inputs(n, N, dtype, "normal", seed_base=300 + N)
    bufs = comm.empty(N, torch_dtype(dtype))
    for b, x in zip(bufs, xs):
        b.copy_(to_torch(x, "cuda:0"))
    comm.collective_virtual(kind, bufs, root=root)
    torch.cuda.synchronize()
    assert comm.status() == hfr.SUCCESS
    want = {"reduce_scatter": lambda: O.reduce_scatter(xs, 0.5), "allgather": lambda: O.all_gather(xs),
            "reduce": lambda: O.reduce(xs, root, 0.5), "broadcast": lambda: O.broadcast(xs, root),
            "allreduce": lambda: O.allreduce(xs, "flat", scale=0.5)}[kind]()
    for r, b in enumerate(bufs):
        assert_bit_exact(to_numpy(b), want[r], f"{kind} n={n} rank {r}")


def test_c3_max_size_sampled(hfr):
    """Config 3's largest message at the bench's launch configuration: 8
    virtual ranks x 1 GiB bf16 (536,870,912 elements) with scale 1/8, FLAT
    (TMA-staged) — 2^20 sampled outputs against the oracle on the sampled
    input columns, and byte-identity of all 8 outputs."""
    n, N = 8, (1 << 30) // 2
    comm = comm_for(hfr, n)
    comm.set_config(hfr.Config(algo="flat", scale=0.125))
    bufs = comm.empty(N, torch.bfloat16)
    for r, b in enumerate(bufs):
        b.copy_(gen.rank_input_torch(r, N, gen.BF16, device="cuda:0"))
    idx = torch.from_numpy(np.random.default_rng(5).integers(0, N, size=1 << 20)).cuda()
    idx[:8] = torch.arange(N - 8, N, device="cuda")  # the ragged end
    cols = [to_numpy(b[idx]) for b in bufs]
    comm.allreduce_virtual(bufs)
    torch.cuda.synchronize()
    assert comm.status() == hfr.SUCCESS
    want = O.fold_ascending(cols, 0.125)
    for r, b in enumerate(bufs):
        assert_bit_exact(to_numpy(b[idx]), want, f"1 GiB bf16 rank {r}")
    h0 = bufs[0].view(torch.int16).sum(dtype=torch.int64)
    for b in bufs[1:]:
        assert torch.equal(b.view(torch.int16), bufs[0].view(torch.int16))
    del bufs, h0
    comm.free_all()


def test_c2_bench_configuration(hfr):
    """C2 exactly as bench.py times it: 8 virtual ranks x 186 MiB fp32,
    gradient-like inputs (seeds 1000 + rank), FLAT, scale 1/8, symmetric
    memory — every element bit-exact."""
    n, N = 8, gen.C2_COUNT
    xs = gen.rank_inputs(n, N, gen.FP32, "grad", seed_base=1000)
    outs = run(hfr, n, xs, "flat", scale=1.0 / n)
    check(outs, O.fold_ascending(xs, 1.0 / n), "C2 bench configuration")
    comm_for(hfr, n).free_all()


_FUZZ = np.random.default_rng(20261018)
_FUZZ_CASES = []
for _i in range(48):
    _n = int(_FUZZ.integers(1, 9))
    _algo = str(_FUZZ.choice(["flat", "oneshot", "dbt", "pair_dbt", "auto", "ce"]))
    if _algo == "pair_dbt" and _n % 2:
        _n += 1 if _n < 8 else -1
    _FUZZ_CASES.append(dict(
        n=_n, algo=_algo, dtype=str(_FUZZ.choice([gen.FP32, gen.BF16, gen.FP16])),
        count=int(_FUZZ.choice([int(_FUZZ.integers(0, 64)), int(_FUZZ.integers(64, 20_000)),
                                int(_FUZZ.integers(20_000, 400_000))])),
        chunk=256 * int(_FUZZ.integers(1, 33)), scale=float(_FUZZ.choice([1.0, 0.5, 1.0 / 3, 2.0])),
        mem=str(_FUZZ.choice(["symmetric", "plain", "offset"])), async_op=bool(_FUZZ.integers(0, 2)),
        dist=str(_FUZZ.choice(["normal", "loguniform", "specials", "int"])), seed=int(_FUZZ.integers(0, 1 << 30))))


@pytest.mark.parametrize("case", _FUZZ_CASES, ids=lambda c: f"{c['algo']}-n{c['n']}-{c['dtype']}-{c['count']}-{c['mem']}")
def test_fuzz_configs(hfr, case):
    """Seeded random configurations (rank count, schedule, dtype, size, chunk,
    scale, memory kind, sync/async, value mix), each bit-exact vs the oracle."""
    c = case
    xs = gen.rank_inputs(c["n"], c["count"], c["dtype"], c["dist"], seed_base=c["seed"])
    outs = run(hfr, c["n"], xs, c["algo"], chunk=c["chunk"], scale=c["scale"],
               symmetric=c["mem"] != "plain", offset=1 if c["mem"] == "offset" else 0, async_op=c["async_op"])
    want = O.allreduce(xs, c["algo"], chunk_elems=c["chunk"], scale=c["scale"])[0]
    check(outs, want, str(c))


@pytest.mark.parametrize("n", [2, 8])
@pytest.mark.parametrize("dtype", [gen.FP32, gen.BF16])
def test_oneshot_fenced_form(hfr, n, dtype):
    """Explicit ONESHOT above the LL threshold runs the fenced push form
    ((n-1) * count * 8 bytes > 6 MiB, message still within the inbox slot)."""
    N = 450_001 if n == 8 else 1_000_003
    xs = gen.rank_inputs(n, N, dtype, "normal", seed_base=91)
    outs = run(hfr, n, xs, "oneshot", scale=0.5)
    check(outs, O.allreduce(xs, "flat", scale=0.5)[0], f"fenced oneshot n={n}")


FP8S = [gen.E4M3, gen.E5M2]


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("dtype", FP8S)
@pytest.mark.parametrize("algo", ALGOS + ["ce", "auto"])
@pytest.mark.parametrize("N", [7, 4096 + 13, 100_003, 1_000_001])
def test_parity_fp8(hfr, n, dtype, algo, N):
    """FP8 (reading R20): E4M3 / E5M2 inputs widened exactly,
    fp32 accumulate in the schedule's order, one RNE rounding with the R20
    overflow rule — bit-exact vs the oracle for every schedule."""
    if algo == "pair_dbt" and n % 2:
        pytest.skip("pair-first needs even n")
    xs = gen.rank_inputs(n, N, dtype, "normal", seed_base=2100 + N)
    outs = run(hfr, n, xs, algo, chunk=512, scale=0.5)
    check(outs, O.allreduce(xs, algo, chunk_elems=512, scale=0.5)[0], f"{algo} n={n} {dtype} N={N}")


@pytest.mark.parametrize("dtype", FP8S)
@pytest.mark.parametrize("dist", ["specials", "int", "loguniform", "grad"])
@pytest.mark.parametrize("algo", ALGOS + ["ce"])
@pytest.mark.parametrize("scale", [1.0, 0.125, 40.0])
def test_parity_fp8_distributions(hfr, dtype, dist, algo, scale):
    """FP8 value mixes incl. NaN/Inf/subnormals/signed zeros, and a scale of
    40 that drives sums past the largest finite value (E4M3 -> NaN, E5M2 ->
    Inf under R20)."""
    n, N = 8, 3 * 16384 + 5
    xs = gen.rank_inputs(n, N, dtype, dist, seed_base=88)
    outs = run(hfr, n, xs, algo, chunk=256, scale=scale)
    check(outs, O.allreduce(xs, algo, chunk_elems=256, scale=scale)[0], f"{algo} {dist} {dtype} x{scale}")


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("dtype", FP8S)
@pytest.mark.parametrize("kind", ["reduce_scatter", "allgather", "reduce", "broadcast"])
def test_collectives_fp8(hfr, n, dtype, kind):
    comm = comm_for(hfr, n)
    comm.set_config(hfr.Config(scale=0.5))
    N = 300_007
    xs = gen.rank_inputs(n, N, dtype, "normal", seed_base=400)
    bufs = comm.empty(N, torch_dtype(dtype))
    for b, x in zip(bufs, xs):
        b.copy_(to_torch(x, "cuda:0"))
    comm.collective_virtual(kind, bufs, root=1)
    torch.cuda.synchronize()
    assert comm.status() == hfr.SUCCESS
    want = {"reduce_scatter": lambda: O.reduce_scatter(xs, 0.5), "allgather": lambda: O.all_gather(xs),
            "reduce": lambda: O.reduce(xs, 1, 0.5), "broadcast": lambda: O.broadcast(xs, 1)}[kind]()
    for r, b in enumerate(bufs):
        assert_bit_exact(to_numpy(b), want[r], f"{kind} fp8 n={n} rank {r}")


def run_cfg(hfr, n, xs, cfg):
    """run() with an explicit Config (the tree kernels' staging modes)."""
    comm = comm_for(hfr, n)
    comm.set_config(cfg)
    N = xs[0].shape[0]
    bufs = comm.empty(N, torch_dtype(dtype_of(xs[0])))
    for b, x in zip(bufs, xs):
        b.copy_(to_torch(x, "cuda:0"))
    comm.allreduce_virtual(bufs)
    torch.cuda.synchronize()
    assert comm.status() == hfr.SUCCESS, hfr.status_string(comm.status())
    return [to_numpy(b) for b in bufs]


@pytest.mark.parametrize("staging", [1, 2])
@pytest.mark.parametrize("algo", ["dbt", "pair_dbt"])
@pytest.mark.parametrize("n", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype", [gen.FP32, gen.BF16, gen.E4M3])
@pytest.mark.parametrize("chunk,N", [(4096, 300_007), (8192, 1_000_003), (24576, 123_457), (256, 4096 + 13)])
def test_tree_staging_modes(hfr, staging, algo, n, dtype, chunk, N):
    """Both tree data paths (1: SM loads/stores + per-chunk fence; 2: TMA bulk
    copies with per-tile flags, several tiles per chunk when chunk > 2048)
    give the tree-order oracle's bits, incl. ragged half ends."""
    if algo == "pair_dbt" and n % 2:
        pytest.skip("pair-first needs even n")
    xs = gen.rank_inputs(n, N, dtype, "normal", seed_base=3300 + N)
    outs = run_cfg(hfr, n, xs, hfr.Config(algo=algo, chunk_elems=chunk, scale=0.25, tree_staging=staging))
    check(outs, O.allreduce(xs, algo, chunk_elems=chunk, scale=0.25)[0], f"{algo} staging={staging} n={n}")


@pytest.mark.parametrize("algo", ["dbt", "pair_dbt"])
def test_tree_many_tiles_segments(hfr, algo):
    """More tiles than one launch's flag array (2^18): the schedule splits
    into several launches (segments) — bf16, n=2, 256-element chunks."""
    n, N = 2, (1 << 18) * 256 * (2 if algo == "pair_dbt" else 1) + 1001
    xs = gen.rank_inputs(n, N, gen.BF16, "normal", seed_base=12)
    comm = comm_for(hfr, n)
    launches = comm.launches
    outs = run_cfg(hfr, n, xs, hfr.Config(algo=algo, chunk_elems=256, scale=0.5))
    assert comm.launches - launches >= 2
    check(outs, O.allreduce(xs, algo, chunk_elems=256, scale=0.5)[0], f"{algo} segments")
    del outs
    comm.free_all()


@pytest.mark.parametrize("staging", [1, 2])
@pytest.mark.parametrize("n", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype", [gen.FP32, gen.BF16, gen.E5M2])
@pytest.mark.parametrize("N", [7, 4096 + 13, 1_000_003])
def test_flat_staging_modes(hfr, staging, n, dtype, N):
    """FLAT with register staging (1) and TMA-staged loads (2; n = 3 has no
    TMA instantiation and falls back to registers): the rank-ascending
    fold's bits either way."""
    xs = gen.rank_inputs(n, N, dtype, "normal", seed_base=4400 + N)
    outs = run_cfg(hfr, n, xs, hfr.Config(algo="flat", scale=0.5, flat_staging=staging))
    check(outs, O.fold_ascending(xs, 0.5), f"flat staging={staging} n={n} {dtype} N={N}")


@pytest.mark.parametrize("n", [11, 16])
@pytest.mark.parametrize("algo", ["flat", "oneshot", "dbt", "pair_dbt", "ce", "auto"])
@pytest.mark.parametrize("dtype", [gen.FP32, gen.BF16, gen.E4M3])
def test_parity_beyond_one_box(hfr, n, algo, dtype):
    """More ranks than one 8-GPU box (the library allows up to 16): the
    generic-n kernels (no compile-time rank count), deeper double binary
    trees (odd n: rank 0 interior in both trees, reading R9) — bit-exact."""
    if algo == "pair_dbt" and n % 2:
        pytest.skip("pair-first needs even n")
    N = 100_003
    xs = gen.rank_inputs(n, N, dtype, "normal", seed_base=5100 + n)
    comm = comm_for(hfr, n)
    comm.set_config(hfr.Config(algo=algo, chunk_elems=1024, scale=1.0 / n, timeout_ms=20000))
    bufs = comm.empty(N, torch_dtype(dtype))
    for b, x in zip(bufs, xs):
        b.copy_(to_torch(x, "cuda:0"))
    comm.allreduce_virtual(bufs)
    torch.cuda.synchronize()
    assert comm.status() == hfr.SUCCESS, hfr.status_string(comm.status())
    want = O.allreduce(xs, algo, chunk_elems=1024, scale=1.0 / n)[0]
    check([to_numpy(b) for b in bufs], want, f"{algo} n={n} {dtype}")
