"""Pins for the oracle's other collectives ("general reduce and
broadcast") and the shard layout (reading R19)."""
import numpy as np
import pytest

import hfr_inputs as gen
from oracle import hfr_oracle as O


@pytest.mark.parametrize("count", [0, 1, 7, 8, 9, 4096, 4097, 100_003])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("K", [4, 8])
def test_shard_bounds_partition(count, n, K):
    b = O.shard_bounds(count, n, K)
    assert len(b) == n and b[0][0] == 0 and b[-1][1] == count
    for (lo, hi), (lo2, _) in zip(b, b[1:]):
        assert hi == lo2 and lo <= hi and lo % K == 0
    # balanced to within one vector (plus the tail on the last shard)
    sizes = [hi - lo for lo, hi in b[:-1]]
    if sizes:
        assert max(sizes) - min(sizes) <= K


def test_library_shard_range_matches_oracle():
    import paper_2408_14158_b200 as hfr
    from paper_2408_14158_b200 import _build
    _build.build()
    for n in (1, 2, 3, 4, 5, 8, 16):
        for count in (0, 1, 9, 1000, 4097, 1 << 20):
            for dt, K in (("f32", 4), ("bf16", 8)):
                want = O.shard_bounds(count, n, K)
                got = [hfr.shard_range(n, count, dt, g) for g in range(n)]
                assert got == want, (n, count, dt)


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_reduce_scatter_integer_closed_form(n):
    xs = gen.rank_inputs(n, 5003, gen.FP32, "int", seed_base=8)
    out = O.reduce_scatter(xs)
    total = sum(x.astype(np.int64) for x in xs)
    for g, (lo, hi) in enumerate(O.shard_bounds(5003, n, 4)):
        assert np.array_equal(out[g][lo:hi].astype(np.int64), total[lo:hi])
        rest = np.ones(5003, bool)
        rest[lo:hi] = False
        assert np.array_equal(out[g][rest], xs[g][rest])


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("dtype", [gen.FP32, gen.BF16])
def test_allgather_of_reduce_scatter_is_allreduce(n, dtype):
    """all_gather(reduce_scatter(x)) == allreduce(x) bit for bit (ZeRO identity)."""
    xs = gen.rank_inputs(n, 10_007, dtype, "normal", seed_base=9)
    composed = O.all_gather(O.reduce_scatter(xs, 0.25))
    want = O.fold_ascending(xs, 0.25)
    for c in composed:
        assert np.array_equal(c.view(np.uint8), want.view(np.uint8))


def test_allgather_explicit_values():
    n, N = 4, 1030
    xs = [np.full(N, 10.0 * (g + 1), dtype=np.float32) for g in range(n)]
    out = O.all_gather(xs)
    for r in range(n):
        for g, (lo, hi) in enumerate(O.shard_bounds(N, n, 4)):
            assert np.all(out[r][lo:hi] == 10.0 * (g + 1))


@pytest.mark.parametrize("root", [0, 2])
def test_reduce_and_broadcast(root):
    xs = gen.rank_inputs(3, 777, gen.FP32, "int", seed_base=10)
    red = O.reduce(xs, root)
    total = sum(x.astype(np.int64) for x in xs)
    for r in range(3):
        if r == root:
            assert np.array_equal(red[r].astype(np.int64), total)
        else:
            assert np.array_equal(red[r], xs[r])
    bc = O.broadcast(xs, root)
    for r in range(3):
        assert np.array_equal(bc[r], xs[root])
