"""Property tests (hypothesis) of the oracle: for random rank counts, sizes,
chunkings, scales and dtypes, every order agrees with the exact integer sum on
integer inputs, every order stays within Higham's bound of the exact sum on
real inputs, n=2 reduces to one library add, and the collectives compose
(all_gather o reduce_scatter == allreduce)."""
from fractions import Fraction

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

import hfr_inputs as gen
from oracle import hfr_oracle as O

ALGOS = ("flat", "dbt", "pair_dbt")


@settings(max_examples=60, deadline=None)
@given(n=st.integers(1, 8), count=st.integers(0, 3000), chunk=st.sampled_from([256, 512, 768, 1024]),
       algo=st.sampled_from(ALGOS), seed=st.integers(0, 10_000))
def test_integer_inputs_exact_in_every_order(n, count, chunk, algo, seed):
    if algo == "pair_dbt" and n % 2:
        n += 1
    xs = gen.rank_inputs(n, count, gen.FP32, "int", seed_base=seed)
    got = O.allreduce(xs, algo, chunk_elems=chunk)[0]
    want = sum((x.astype(np.int64) for x in xs), np.zeros(count, np.int64))
    assert np.array_equal(got.astype(np.int64), want)


@settings(max_examples=40, deadline=None)
@given(n=st.integers(2, 8), chunk=st.sampled_from([256, 512, 1024]), algo=st.sampled_from(ALGOS),
       seed=st.integers(0, 10_000), dist=st.sampled_from(["normal", "loguniform", "grad"]))
def test_every_order_within_higham_bound(n, chunk, algo, seed, dist):
    if algo == "pair_dbt" and n % 2:
        n += 1
    count = 600
    xs = gen.rank_inputs(n, count, gen.FP32, dist, seed_base=seed)
    got = O.allreduce(xs, algo, chunk_elems=chunk)[0]
    u = Fraction(1, 1 << 24)
    gamma = (n - 1) * u / (1 - (n - 1) * u)
    for i in range(0, count, 37):
        exact = sum(Fraction(float(x[i])) for x in xs)
        A = sum(abs(Fraction(float(x[i]))) for x in xs)
        assert abs(Fraction(float(got[i])) - exact) <= gamma * A


@settings(max_examples=40, deadline=None)
@given(count=st.integers(0, 5000), algo=st.sampled_from(ALGOS), seed=st.integers(0, 10_000),
       dtype=st.sampled_from([gen.FP32, gen.BF16, gen.FP16]))
def test_two_ranks_is_one_library_add(count, algo, seed, dtype):
    a, b = gen.rank_inputs(2, count, dtype, "normal", seed_base=seed)
    got = O.allreduce([a, b], algo, chunk_elems=256)[0]
    s = np.add(O.widen(a), O.widen(b), dtype=np.float32)
    want = O._finish(s, 1.0, O._out_dtype([a]))
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


@settings(max_examples=40, deadline=None)
@given(n=st.integers(1, 8), count=st.integers(0, 4000), seed=st.integers(0, 10_000),
       dtype=st.sampled_from([gen.FP32, gen.BF16, gen.FP16]),
       scale=st.sampled_from([1.0, 0.5, 0.125, 0.1]))
def test_allgather_of_reduce_scatter(n, count, seed, dtype, scale):
    xs = gen.rank_inputs(n, count, dtype, "normal", seed_base=seed)
    composed = O.all_gather(O.reduce_scatter(xs, scale))
    want = O.fold_ascending(xs, scale)
    for c in composed:
        assert np.array_equal(c.view(np.uint8), want.view(np.uint8))
