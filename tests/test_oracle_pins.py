"""Pins for the CPU oracle (oracle/hfr_oracle.py) against things other than itself.

Each pin is chosen so that a plausible mistake in the oracle — a dropped term,
a wrong sign or index, a transposed operand, a wrong grouping, FTZ, a double
rounding, scaling at the wrong place — fails at least one test:

* exact-rational brute force: every fp32 add / multiply / bf16 cast is
  re-derived from exact rationals with a hand-written IEEE round-to-nearest-
  even (subnormals and overflow included) — independent of numpy's float math;
* closed forms: integer inputs whose every partial sum is exact, for which any
  order must give the int64 sum;
* library special cases: n=2 is ``np.float32(a) + np.float32(b)`` (commutative,
  so every order agrees); bf16 RNE vs ``torch.Tensor.to(torch.bfloat16)``;
* golden worked examples (tests/golden/), each cited;
* invariants: n*x with low mantissa bits cleared, all-zero rank identity,
  Higham's summation error bound against the exact sum;
* tree invariants of SPEC.md:146-148 for n = 1..1024.
"""
from __future__ import annotations

import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import hfr_inputs as gen
from oracle import hfr_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------------------
# exact-rational IEEE model (independent of numpy float arithmetic)
# ----------------------------------------------------------------------------

def _round_binary(q: Fraction, p: int, emin: int, emax: int):
    """Round rational q to the binary format with p significand bits (incl.
    hidden bit), min normal exponent emin, max exponent emax, RNE.  Returns a
    Fraction or +-math.inf; zero sign is handled by the caller."""
    if q == 0:
        return Fraction(0)
    s = -1 if q < 0 else 1
    a = abs(q)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    e = max(e, emin)
    ulp = Fraction(2) ** (e - (p - 1))
    m = a / ulp
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    r = fl * ulp
    if r >= Fraction(2) ** (emax + 1):
        return s * math.inf
    return s * r


def f32_round(q: Fraction):
    return _round_binary(q, 24, -126, 127)


def bf16_round(q: Fraction):
    return _round_binary(q, 8, -126, 127)


def exact_add(a: float, b: float) -> float:
    """fl32(a + b) from exact rationals, with IEEE signed-zero rules."""
    if math.isnan(a) or math.isnan(b):
        return math.nan
    if math.isinf(a) or math.isinf(b):
        if math.isinf(a) and math.isinf(b) and (a > 0) != (b > 0):
            return math.nan
        return a if math.isinf(a) else b
    q = Fraction(a) + Fraction(b)
    if q == 0:
        # x + (-x) = +0 under RNE; (-0) + (-0) = -0
        return -0.0 if (math.copysign(1, a) < 0 and math.copysign(1, b) < 0) else 0.0
    r = f32_round(q)
    return float(r)


def exact_mul(a: float, b: float) -> float:
    if math.isnan(a) or math.isnan(b):
        return math.nan
    if math.isinf(a) or math.isinf(b):
        if a == 0 or b == 0:
            return math.nan
        return math.copysign(math.inf, a) * math.copysign(1, b)
    q = Fraction(a) * Fraction(b)
    if q == 0:
        return math.copysign(0.0, math.copysign(1, a) * math.copysign(1, b))
    return float(f32_round(q))


def exact_bf16(y: float) -> float:
    if math.isnan(y) or math.isinf(y) or y == 0:
        return y
    return math.copysign(float(bf16_round(Fraction(y))), y)  # an underflow to zero keeps the sign


def bits32(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float32).view(np.uint32)


def brute_ascending(cols, scale=1.0, bf16=False):
    """Rank-ascending fold, element by element, via exact_add."""
    out = []
    for vals in cols:
        acc = float(vals[0])
        for v in vals[1:]:
            acc = exact_add(acc, float(v))
        acc = exact_mul(acc, float(np.float32(scale)))
        out.append(exact_bf16(acc) if bf16 else acc)
    return out


def _same_f32(got: np.ndarray, want) -> bool:
    want = np.asarray(want, dtype=np.float32)
    g, w = np.asarray(got, dtype=np.float32), want
    nan_ok = np.array_equal(np.isnan(g), np.isnan(w))
    m = ~np.isnan(w)
    return nan_ok and np.array_equal(bits32(g[m]), bits32(w[m]))


# ----------------------------------------------------------------------------
# the brute-force model itself is sane (pins the pin)
# ----------------------------------------------------------------------------

def test_exact_model_matches_known_ieee_facts():
    assert exact_add(16777216.0, 1.0) == 16777216.0          # tie to even
    assert exact_add(16777216.0, 3.0) == 16777220.0          # 16777219 -> tie -> even (…20)
    assert exact_add(1.0, 2.0 ** -24) == 1.0                 # half ulp of 1.0 ties to 1.0
    assert exact_add(1.0, 2.0 ** -23) == 1.0 + 2.0 ** -23
    assert math.copysign(1, exact_add(-0.0, -0.0)) < 0
    assert math.copysign(1, exact_add(-0.0, 0.0)) > 0
    assert exact_add(2.0 ** -149, 2.0 ** -149) == 2.0 ** -148  # subnormals, no FTZ
    assert exact_add(3.4e38, 3.4e38) == math.inf
    assert exact_bf16(257.0) == 256.0
    assert exact_bf16(1.0 + 2.0 ** -8) == 1.0                # tie -> even
    assert exact_bf16(1.0 + 3 * 2.0 ** -8) == 1.0 + 2.0 ** -6


# ----------------------------------------------------------------------------
# fold_ascending
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("dist", ["normal", "loguniform", "specials"])
def test_fold_ascending_fp32_brute_force(n, dist):
    xs = gen.rank_inputs(n, 64, gen.FP32, dist, seed_base=77 + n)
    got = O.fold_ascending(xs)
    want = brute_ascending(list(zip(*[x.tolist() for x in xs])))
    assert _same_f32(got, want)


@pytest.mark.parametrize("scale", [0.125, 0.1, 3.0])
def test_fold_ascending_scale_brute_force(scale):
    xs = gen.rank_inputs(4, 64, gen.FP32, "normal", seed_base=5)
    got = O.fold_ascending(xs, scale=scale)
    want = brute_ascending(list(zip(*[x.tolist() for x in xs])), scale=scale)
    assert _same_f32(got, want)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("dist", ["normal", "loguniform", "specials"])
def test_fold_ascending_bf16_brute_force(n, dist):
    xs = gen.rank_inputs(n, 64, gen.BF16, dist, seed_base=99 + n)
    got = O.bf16_to_f32(O.fold_ascending(xs, scale=0.5 if n > 2 else 1.0))
    cols = list(zip(*[O.bf16_to_f32(x).tolist() for x in xs]))
    want = brute_ascending(cols, scale=0.5 if n > 2 else 1.0, bf16=True)
    assert _same_f32(got, want)


@pytest.mark.parametrize("n", [2, 3, 4, 7, 8])
@pytest.mark.parametrize("algo", ["flat", "dbt", "pair_dbt"])
def test_integer_closed_form(n, algo):
    """|x| < 2^20, n <= 8: every partial sum is exact, so any order = int64 sum."""
    if algo == "pair_dbt" and n % 2:
        pytest.skip("pair-first needs even n")
    xs = gen.rank_inputs(n, 3000, gen.FP32, "int", seed_base=11)
    want = np.zeros(3000, dtype=np.int64)
    for x in xs:
        want += x.astype(np.int64)
    got = O.allreduce(xs, algo, chunk_elems=256)[0]
    assert np.array_equal(got.astype(np.int64), want)


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("algo", ["flat", "dbt", "pair_dbt"])
def test_integer_closed_form_bf16(n, algo):
    """bf16 integers |x| <= 256: fp32 sums exact in any order; output =
    RNE_bf16(int sum), the RNE taken by torch (a library routine)."""
    import torch
    xs = gen.rank_inputs(n, 2000, gen.BF16, "int", seed_base=12)
    s = np.zeros(2000, dtype=np.int64)
    for x in xs:
        s += O.bf16_to_f32(x).astype(np.int64)
    want = torch.tensor(s.astype(np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = O.allreduce(xs, algo, chunk_elems=256)[0]
    assert np.array_equal(got, want)


@pytest.mark.parametrize("algo", ["flat", "dbt", "pair_dbt"])
def test_n2_is_library_add(algo):
    a, b = gen.rank_inputs(2, 5000, gen.FP32, "specials", seed_base=3)
    got = O.allreduce([a, b], algo, chunk_elems=256)[0]
    assert _same_f32(got, a + b)
    import torch
    a16, b16 = gen.rank_inputs(2, 5000, gen.BF16, "loguniform", seed_base=4)
    fa, fb = O.bf16_to_f32(a16), O.bf16_to_f32(b16)
    want = torch.tensor(fa + fb).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = O.allreduce([a16, b16], algo, chunk_elems=256)[0]
    nan = np.isnan(fa + fb)
    assert np.array_equal(np.isnan(O.bf16_to_f32(got)), nan)
    assert np.array_equal(got[~nan], want[~nan])


def test_n1_identity():
    x = gen.rank_input(0, 1000, gen.FP32, "specials")
    assert _same_f32(O.fold_ascending([x]), x)
    xb = gen.rank_input(0, 1000, gen.BF16, "specials")
    y = O.fold_ascending([xb])
    nan = np.isnan(O.bf16_to_f32(xb))
    assert np.array_equal(y[~nan], xb[~nan])
    assert np.all(np.isnan(O.bf16_to_f32(y[nan])))


@pytest.mark.parametrize("n", [3, 5, 6, 7, 8])
def test_n_times_x_invariant(n):
    """Sum of n identical buffers = n*x (exact) when x's low ceil(log2 n)
    mantissa bits are clear (SURVEY.md §8c 'n·x invariant')."""
    x = gen.low_bits_cleared(gen.rank_input(0, 20000, gen.FP32, "normal"), 3)
    got = O.fold_ascending([x] * n)
    want = (x.astype(np.float64) * n).astype(np.float32)
    assert np.array_equal(bits32(got), bits32(want))


@pytest.mark.parametrize("algo", ["flat", "dbt", "pair_dbt"])
def test_zero_rank_is_identity(algo):
    """A rank of +0.0 leaves the fold over the others unchanged (compare by
    value: -0.0 + +0.0 = +0.0 is the documented exception)."""
    n = 8
    xs = gen.rank_inputs(n, 4096, gen.FP32, "normal", seed_base=21)
    zs = [x.copy() for x in xs]
    zs[5] = np.zeros_like(xs[5])
    got = O.allreduce(zs, algo, chunk_elems=256)[0]
    if algo == "flat":
        want = O.fold_ascending(xs[:5] + xs[6:])
        assert np.array_equal(got, want)
    # independent check for every order: within Higham's bound of the exact sum
    _assert_within_higham(got, zs)


def _assert_within_higham(got, xs):
    n = len(xs)
    u = 2.0 ** -24
    gamma = (n - 1) * u / (1 - (n - 1) * u)
    # exact sum in long double via fractions on a sample, float64 bound elsewhere
    X = np.stack([O.widen(x).astype(np.float64) for x in xs])
    A = np.abs(X).sum(axis=0)
    idx = np.linspace(0, X.shape[1] - 1, 97).astype(int)
    for i in idx:
        exact = sum(Fraction(float(v)) for v in X[:, i])
        err = abs(Fraction(float(got[i])) - exact)
        assert err <= Fraction(gamma) * Fraction(float(A[i])) * (1 + Fraction(1, 1 << 20)), i


@pytest.mark.parametrize("algo", ["flat", "dbt", "pair_dbt"])
@pytest.mark.parametrize("n", [2, 4, 8])
def test_higham_bound(algo, n):
    xs = gen.rank_inputs(n, 8192, gen.FP32, "normal", seed_base=31)
    got = O.allreduce(xs, algo, chunk_elems=512)[0]
    _assert_within_higham(got, xs)


# ----------------------------------------------------------------------------
# bf16 RNE cast
# ----------------------------------------------------------------------------

def test_bf16_rne_matches_torch():
    import torch
    rng = np.random.default_rng(0)
    u = rng.integers(0, 2 ** 32, size=1 << 20, dtype=np.uint64).astype(np.uint32)
    f = u.view(np.float32)
    got = O.bf16_rne(f)
    want = torch.tensor(f).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    nan = np.isnan(f)
    assert np.array_equal(got[~nan], want[~nan])
    assert np.all(np.isnan(O.bf16_to_f32(got[nan])))
    # low-payload NaNs must not become Inf (reading R5)
    low_nan = np.array([0x7F800001, 0xFF800001, 0x7F80FFFF], dtype=np.uint32).view(np.float32)
    assert np.all(np.isnan(O.bf16_to_f32(O.bf16_rne(low_nan))))


def test_bf16_rne_hand_cases():
    cases = [(1.0 + 2.0 ** -8, 0x3F80), (1.0 + 3 * 2.0 ** -8, 0x3F82), (257.0, 0x4380),
             (-257.0, 0xC380), (259.0, 0x4382), (0.0, 0x0000), (-0.0, 0x8000), (np.inf, 0x7F80)]
    for v, bits in cases:
        assert int(O.bf16_rne(np.array([v], dtype=np.float32))[0]) == bits, v


# ----------------------------------------------------------------------------
# golden worked examples
# ----------------------------------------------------------------------------

def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _as_inputs(case):
    xs = [np.array(v, dtype=np.float32) for v in case["inputs"]]
    if case["dtype"] == "bf16":
        xs = [(x.view(np.uint32) >> 16).astype(np.uint16) for x in xs]
    return xs


@pytest.mark.parametrize("case", _load("spec_examples.json")["cases"], ids=lambda c: c["cite"][:24])
def test_spec_examples(case):
    xs = _as_inputs(case)
    algos = ["flat", "dbt"] + (["pair_dbt"] if len(xs) % 2 == 0 else [])
    for algo in algos:
        got = O.allreduce(xs, algo, chunk_elems=256)
        want = np.array(case["expected"], dtype=np.float32)
        for g in got:
            g32 = O.bf16_to_f32(g) if case["dtype"] == "bf16" else g
            assert _same_f32(g32, want), (algo, case["cite"])


@pytest.mark.parametrize("case", _load("order_examples.json")["cases"], ids=lambda c: c["name"])
def test_order_examples(case):
    xs = [np.array(v, dtype=np.float32) for v in case["inputs"]]
    got = O.allreduce(xs, case["algo"], chunk_elems=case["chunk_elems"], scale=case.get("scale", 1.0))
    want = np.array(case["expected"], dtype=np.float32)
    for g in got:
        assert _same_f32(g, want), case["name"]


# ----------------------------------------------------------------------------
# tree-order folds: brute force from the tree TABLE (not the oracle's builder)
# ----------------------------------------------------------------------------

def _golden_tree(n, which):
    t = _load("trees.json")["trees"][str(n)][which]
    return t["root"], {int(k): v for k, v in t["children"].items()}


def _brute_tree_elem(root, children, vals):
    def E(v):
        kids = children.get(v, [])
        acc = None
        for c in [k for k in kids if k < v]:
            e = E(c)
            acc = e if acc is None else exact_add(acc, e)
        acc = float(vals[v]) if acc is None else exact_add(acc, float(vals[v]))
        for c in [k for k in kids if k > v]:
            acc = exact_add(acc, E(c))
        return acc
    return E(root)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_fold_tree_brute_force(n):
    C = 4
    xs = gen.rank_inputs(n, 40, gen.FP32, "loguniform", seed_base=41)
    got = O.fold_tree(xs, C)
    trees = [_golden_tree(n, "A"), _golden_tree(n, "B")]
    want = []
    for i in range(40):
        root, ch = trees[(i // C) % 2]
        want.append(_brute_tree_elem(root, ch, [float(x[i]) for x in xs]))
    assert _same_f32(got, want)


@pytest.mark.parametrize("n", [4, 8])
def test_fold_pairfirst_brute_force(n):
    C = 3
    N = 1100  # > 512, so the split H = 768 is exercised with a ragged half
    xs = gen.rank_inputs(n, N, gen.FP32, "loguniform", seed_base=51)
    got = O.fold_pairfirst(xs, C, scale=0.25)
    m = n // 2
    trees = [_golden_tree(m, "A"), _golden_tree(m, "B")] if m > 1 else None
    H = 768
    assert O.pair_split(N) == H
    want = []
    for i in range(N):
        lo = 0 if i < H else H
        p = [exact_add(float(xs[2 * k][i]), float(xs[2 * k + 1][i])) for k in range(m)]
        root, ch = trees[((i - lo) // C) % 2]
        want.append(exact_mul(_brute_tree_elem(root, ch, p), 0.25))
    assert _same_f32(got, want)


def test_pair_split_reading():
    assert O.pair_split(0) == 0
    assert O.pair_split(1) == 1
    assert O.pair_split(4096) == 2048
    assert O.pair_split(4097) == 2304
    for N in range(0, 5000, 37):
        H = O.pair_split(N)
        assert 0 <= H <= N and (H == N or H % 256 == 0) and H >= (N + 1) // 2


# ----------------------------------------------------------------------------
# tree construction (SPEC.md:146-148 invariants, golden tables)
# ----------------------------------------------------------------------------

def _depth(parent, v):
    d = 0
    while parent[v] >= 0:
        v = parent[v]
        d += 1
        assert d <= len(parent)
    return d


@pytest.mark.parametrize("n", list(range(1, 129)) + [255, 256, 257, 511, 512, 1000, 1023, 1024])
def test_tree_invariants(n):
    trees = O.build_double_binary_tree(n)
    interior = []
    for parent, children in trees:
        roots = [v for v in range(n) if parent[v] < 0]
        assert len(roots) == 1
        # spanning: every node reaches the root; children consistent with parents
        for v in range(n):
            assert _depth(parent, v) <= int(math.floor(math.log2(n))) + 2
            for c in children[v]:
                assert parent[c] == v
            assert len(children[v]) <= 2
        assert sum(len(c) for c in children) == n - 1
        interior.append({v for v in range(n) if children[v]})
    both = interior[0] & interior[1]
    if n % 2 == 0:
        assert not both, both          # interior in at most one tree
    else:
        assert both <= {0}, both       # documented odd-n exception (reading R9)
    assert O.build_double_binary_tree(n) == trees  # deterministic


@pytest.mark.parametrize("n", [2, 4, 8])
def test_tree_golden_tables(n):
    for which, (parent, children) in zip("AB", O.build_double_binary_tree(n)):
        root, ch = _golden_tree(n, which)
        assert parent[root] == -1
        assert {v: c for v, c in enumerate(children) if c} == ch


def test_tree_n1_degenerate():
    (pa, ca), (pb, cb) = O.build_double_binary_tree(1)
    assert pa == [-1] and pb == [-1] and ca == [[]] and cb == [[]]
    with pytest.raises(ValueError):
        O.build_double_binary_tree(0)


# ----------------------------------------------------------------------------
# fp16 (PAPER.md:404 lists FP16): fp32 accumulate, one RNE rounding to binary16
# ----------------------------------------------------------------------------

def f16_round(q: Fraction):
    return _round_binary(q, 11, -14, 15)


def exact_f16(y: float) -> float:
    if math.isnan(y) or math.isinf(y) or y == 0:
        return y
    return math.copysign(float(f16_round(Fraction(y))), y)  # an underflow to zero keeps the sign


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("dist", ["normal", "loguniform", "specials"])
def test_fold_ascending_fp16_brute_force(n, dist):
    xs = gen.rank_inputs(n, 64, gen.FP16, dist, seed_base=199 + n)
    scale = 0.5 if n > 2 else 1.0
    got = O.fold_ascending(xs, scale=scale).astype(np.float32)
    cols = list(zip(*[x.astype(np.float32).tolist() for x in xs]))
    want = []
    for vals in cols:
        acc = float(vals[0])
        for v in vals[1:]:
            acc = exact_add(acc, float(v))
        want.append(exact_f16(exact_mul(acc, scale)))
    assert _same_f32(got, want)


def test_fp16_rne_matches_torch_and_hand_cases():
    import torch
    rng = np.random.default_rng(1)
    f = rng.integers(0, 2 ** 32, size=1 << 20, dtype=np.uint64).astype(np.uint32).view(np.float32)
    got = O._finish(f, 1.0, O.F16)
    want = torch.tensor(f).to(torch.float16).numpy()
    nan = np.isnan(f)
    assert np.array_equal(got[~nan].view(np.uint16), want[~nan].view(np.uint16))
    assert np.all(np.isnan(got[nan]))
    # hand cases: 2049 ties to 2048, 2051 ties to 2052, 65520 overflows to inf, 2^-25 ties to 0
    cases = [(2049.0, 2048.0), (2051.0, 2052.0), (65519.0, 65504.0), (65520.0, np.inf), (2.0 ** -25, 0.0),
             (3 * 2.0 ** -25, 2.0 ** -23)]
    for v, w in cases:
        assert float(O._finish(np.array([v], np.float32), 1.0, O.F16)[0]) == w, v


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("algo", ["flat", "dbt", "pair_dbt"])
def test_integer_closed_form_fp16(n, algo):
    """|x| <= 256, n <= 8: sums <= 2048 are exact in fp32 and in binary16."""
    xs = gen.rank_inputs(n, 2000, gen.FP16, "int", seed_base=13)
    want = sum(x.astype(np.int64) for x in xs)
    got = O.allreduce(xs, algo, chunk_elems=256)[0]
    assert np.array_equal(got.astype(np.int64), want)


# ----------------------------------------------------------------------------
# FP8 (PAPER.md:404 lists FP8; reading R20): E4M3 (OCP "FN") and E5M2, fp32
# accumulate, one RNE rounding; overflow -> NaN (E4M3) / Inf (E5M2)
# ----------------------------------------------------------------------------

FP8_FORMATS = [(gen.E4M3, "float8_e4m3fn"), (gen.E5M2, "float8_e5m2")]


def exact_fp8(y: float, fmt: str) -> float:
    """RNE of a float to the FP8 format from exact rationals (independent of
    the oracle's ladder search): E4M3 p=4, emin=-6, largest finite 448 (the
    binary grid's 480 is the NaN code); E5M2 p=3, emin=-14, emax=15."""
    if math.isnan(y):
        return math.nan
    if fmt == gen.E4M3:
        if math.isinf(y):
            return math.nan
        if y == 0:
            return y
        r = _round_binary(Fraction(y), 4, -6, 8)
        return math.nan if (math.isinf(r) or abs(r) > 448) else math.copysign(float(r), y)
    if math.isinf(y) or y == 0:
        return y
    return math.copysign(float(_round_binary(Fraction(y), 3, -14, 15)), y)  # signed zero on underflow


def _torch_fp8_values(codes: np.ndarray, tname: str) -> np.ndarray:
    import torch
    return torch.from_numpy(np.ascontiguousarray(codes).view(np.uint8)).view(getattr(torch, tname)).float().numpy()


@pytest.mark.parametrize("fmt,tname", FP8_FORMATS)
def test_fp8_decode_matches_torch(fmt, tname):
    codes = np.arange(256, dtype=np.uint8)
    want = _torch_fp8_values(codes, tname)
    got = O.fp8_decode_table(fmt).astype(np.float32)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    m = ~np.isnan(want)
    assert np.array_equal(bits32(got[m]), bits32(want[m]))


@pytest.mark.parametrize("fmt,tname", FP8_FORMATS)
def test_fp8_rne_matches_torch_and_hand_cases(fmt, tname):
    import torch
    rng = np.random.default_rng(3)
    f = rng.integers(0, 2 ** 32, size=1 << 20, dtype=np.uint64).astype(np.uint32).view(np.float32)
    f2 = (rng.standard_normal(1 << 20) * np.exp2(rng.uniform(-20, 18, 1 << 20))).astype(np.float32)
    for y in (f, f2):
        got = O.fp8_rne(y, fmt).view(np.uint8)
        want = torch.from_numpy(y).to(getattr(torch, tname)).view(torch.uint8).numpy()
        gv, wv = O.fp8_decode_table(fmt)[got], O.fp8_decode_table(fmt)[want]
        assert np.array_equal(np.isnan(gv), np.isnan(wv))
        m = ~np.isnan(wv)
        assert np.array_equal(got[m], want[m])
    if fmt == gen.E4M3:  # ties to even code, the 464 tie stays finite, past it NaN; subnormal ties
        cases = [(464.0, 448.0), (465.0, math.nan), (1e9, math.nan), (math.inf, math.nan), (2.0 ** -10, 0.0),
                 (1.5 * 2.0 ** -9, 2.0 ** -8), (17.0, 16.0), (19.0, 20.0)]
    else:
        cases = [(61439.0, 57344.0), (61440.0, math.inf), (-math.inf, -math.inf), (2.0 ** -17, 0.0),
                 (1.5 * 2.0 ** -16, 2.0 ** -15), (9.0, 8.0), (11.0, 12.0)]
    for v, w in cases:
        g = float(O.widen(O.fp8_rne(np.array([v], np.float32), fmt))[0])
        assert (math.isnan(g) and math.isnan(w)) or g == w, (fmt, v, g, w)
        e = exact_fp8(v, fmt)
        assert (math.isnan(e) and math.isnan(w)) or e == w, (fmt, v, e, w)


@pytest.mark.parametrize("fmt,tname", FP8_FORMATS)
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("dist", ["normal", "loguniform", "specials", "int"])
def test_fold_ascending_fp8_brute_force(fmt, tname, n, dist):
    """Exact-rational brute force of the rank-ascending fold
    with FP8 inputs decoded by PyTorch (not the oracle's table) and the final
    rounding by exact_fp8."""
    xs = gen.rank_inputs(n, 96, fmt, dist, seed_base=311 + n)
    scale = 0.25 if n > 2 else 1.0
    got = O.fold_ascending(xs, scale=scale)
    assert O.fp8_format(got.dtype) == fmt
    cols = list(zip(*[_torch_fp8_values(x, tname).tolist() for x in xs]))
    want = []
    for vals in cols:
        acc = float(vals[0])
        for v in vals[1:]:
            acc = exact_add(acc, float(v))
        want.append(exact_fp8(exact_mul(acc, scale), fmt))
    assert _same_f32(O.widen(got), want)


@pytest.mark.parametrize("fmt,tname", FP8_FORMATS)
@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("algo", ["flat", "dbt", "pair_dbt"])
def test_integer_closed_form_fp8(fmt, tname, n, algo):
    """|x| <= 8, n <= 8: every fp32 partial sum is an exact integer (<= 64) in
    any order, so every schedule gives RNE_fp8(integer sum) — computed here by
    PyTorch's conversion of the int64 sum."""
    import torch
    xs = gen.rank_inputs(n, 3000, fmt, "int", seed_base=17)
    ints = [_torch_fp8_values(x, tname).astype(np.int64) for x in xs]
    total = sum(ints)
    want = torch.from_numpy(total.astype(np.float32)).to(getattr(torch, tname)).view(torch.uint8).numpy()
    got = O.allreduce(xs, algo, chunk_elems=256)[0]
    assert np.array_equal(got.view(np.uint8), want)
