"""Plain, slow, obviously-correct CPU oracle for HFReduce (arXiv 2408.14158 §4).

TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.  Imported only by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs.

What HFReduce computes (§4 intro): an allreduce — every rank ends
with the elementwise sum of all ranks' gradient buffers.  The paper's two
algorithms reach that sum in a fixed order:

* Algorithm 1 "Intra Node Reduce": ``Dc_i += GPU-j's Dc_i``
  for j in GPU_Count — a left fold over sources in ascending index order.
  ``fold_ascending`` writes that definition out (reading R1).
* Algorithm 2 "Inter Node Reduce": pass 1 reduces up a
  double binary tree (``DL_i += DR_i``), pass 2 gathers the result down;
  chunks alternate between the two trees.  ``fold_tree`` evaluates exactly the
  per-element expression that schedule produces (readings R8-R11).
* "HFReduce with NVLink": pair pre-reduce over NVLink, then
  the tree over pair partials, split result returned to the pair and
  all-gathered.  ``fold_pairfirst`` (reading R13).

Numerics (readings R2-R6): every add and the one scale multiply are IEEE-754
binary32 round-to-nearest-even with no FTZ/DAZ and no FMA; bf16 inputs are
widened exactly to fp32, accumulated in fp32 and rounded ONCE to bf16 (RNE,
NaN kept NaN) after the scale.

fp32 arrays are ``np.float32``; bf16 arrays are ``np.uint16`` bit patterns;
fp16 arrays are ``np.float16``; FP8 arrays (PAPER.md:404 lists FP8; OCP E4M3
"FN" and E5M2, reading R20) are ``np.uint8`` bit patterns whose dtype carries
the format in its metadata (``E4M3_DT`` / ``E5M2_DT``).
"""
from __future__ import annotations

import numpy as np

F32 = "f32"
BF16 = "bf16"
F16 = "f16"
E4M3 = "e4m3"
E5M2 = "e5m2"

# FP8 bit-pattern arrays: uint8 tagged with the format (numpy has no fp8 type)
E4M3_DT = np.dtype(np.uint8, metadata={"hfr": E4M3})
E5M2_DT = np.dtype(np.uint8, metadata={"hfr": E5M2})

PAIR_SPLIT_ALIGN = 256  # elements; reading R13 (half boundary alignment)


# ----------------------------------------------------------------------------
# dtype helpers
# ----------------------------------------------------------------------------

def fp8_format(dt) -> str | None:
    """'e4m3' / 'e5m2' for a tagged FP8 dtype, else None."""
    md = getattr(dt, "metadata", None)
    return md.get("hfr") if md else None


# FP8 formats (reading R20): (exponent bits, mantissa bits, bias).  E4M3 is
# OCP "E4M3FN": no infinities, S.1111.111 is NaN, largest finite 448; E5M2 is
# IEEE-like: exponent 11111 holds +-Inf (mantissa 0) and NaN, largest 57344.
_FP8 = {E4M3: (4, 3, 7), E5M2: (5, 2, 15)}


def fp8_decode_table(fmt: str) -> np.ndarray:
    """float64 value of each of the 256 codes, straight from the format
    definition: normal (-1)^s 2^(e-bias) (1 + m/2^M); subnormal (e = 0)
    (-1)^s 2^(1-bias) (m/2^M); E4M3 code S.1111.111 = NaN; E5M2 e = 2^E-1:
    m = 0 Inf, else NaN."""
    E, M, bias = _FP8[fmt]
    out = np.empty(256, dtype=np.float64)
    for code in range(256):
        s = -1.0 if code >> 7 else 1.0
        e = (code >> M) & ((1 << E) - 1)
        m = code & ((1 << M) - 1)
        if fmt == E4M3 and e == 15 and m == 7:
            v = np.nan
        elif fmt == E5M2 and e == 31:
            v = np.inf if m == 0 else np.nan
        elif e == 0:
            v = 2.0 ** (1 - bias) * (m / 2.0 ** M)
        else:
            v = 2.0 ** (e - bias) * (1.0 + m / 2.0 ** M)
        out[code] = s * v
    return out


def fp8_rne(y: np.ndarray, fmt: str) -> np.ndarray:
    """fp32 -> FP8 bits, round to nearest, ties to the even code (code LSB 0).

    Reading R20 (overflow, as torch.Tensor.to(float8_*): no saturation): the
    ladder of non-negative finite values is extended by one hypothetical step
    above the largest finite (448 + 32 = 480 for E4M3, 57344 + 8192 = 65536
    for E5M2, whose code there is +Inf); a magnitude that rounds onto that step
    overflows: E4M3 -> NaN (it has no Inf), E5M2 -> Inf.  NaN -> NaN;
    +-Inf -> E5M2 +-Inf, E4M3 NaN; the sign is kept (also on zero)."""
    E, M, bias = _FP8[fmt]
    table = fp8_decode_table(fmt)
    pos = [c for c in range(128) if np.isfinite(table[c])]   # 0x00.. ascending magnitudes
    ladder = np.array([table[c] for c in pos] + [table[pos[-1]] + 2.0 ** (((pos[-1] >> M) & ((1 << E) - 1)) - bias - M)])
    codes = np.array(pos + [pos[-1] + 1], dtype=np.int64)    # hypothetical step: next code
    nan_code = 0x7F if fmt == E4M3 else 0x7E
    inf_code = 0x7C
    y = np.ascontiguousarray(y, dtype=np.float32)
    a = np.abs(y.astype(np.float64))
    sign = (np.signbit(y)).astype(np.int64) << 7
    k = np.searchsorted(ladder, a, side="left")              # ladder[k-1] < a <= ladder[k]
    k = np.clip(k, 1, len(ladder) - 1)
    lo, hi = ladder[k - 1], ladder[k]
    pick_hi = (a - lo > hi - a) | ((a - lo == hi - a) & ((codes[k] & 1) == 0))
    idx = np.where(pick_hi, k, k - 1)
    idx = np.where(a == 0, 0, idx)
    code = codes[idx]
    over = (idx == len(ladder) - 1) | (a > ladder[-1])
    code = np.where(over, nan_code if fmt == E4M3 else inf_code, code)
    code = np.where(np.isinf(y), nan_code if fmt == E4M3 else inf_code, code)
    code = np.where(np.isnan(y), nan_code, code)
    return (code | sign).astype(np.uint8).view(E4M3_DT if fmt == E4M3 else E5M2_DT)


def widen(x: np.ndarray) -> np.ndarray:
    """Exact widening to fp32: bf16 bit patterns -> float32 (upper 16 bits);
    IEEE binary16 -> float32 (every half is a float); FP8 codes -> their
    value from the format definition (every FP8 value is a float)."""
    fmt = fp8_format(x.dtype)
    if fmt:
        return fp8_decode_table(fmt).astype(np.float32)[np.asarray(x).view(np.uint8)]
    if x.dtype == np.float32:
        return x
    if x.dtype == np.uint16:
        return (x.astype(np.uint32) << np.uint32(16)).view(np.float32)
    if x.dtype == np.float16:
        return x.astype(np.float32)
    raise TypeError(f"unsupported oracle dtype {x.dtype}")


def bf16_rne(y: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bits, round-to-nearest-even; NaN stays (quiet) NaN.

    Reading R5: the classic ``u + 0x7FFF + ((u >> 16) & 1)`` trick would turn
    low-payload NaNs into Inf, so NaNs are special-cased.
    """
    u = np.ascontiguousarray(y, dtype=np.float32).view(np.uint32).astype(np.uint64)
    is_nan = (u & 0x7FFFFFFF) > 0x7F800000
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) & 0xFFFF
    r = np.where(is_nan, ((u >> 16) | 0x0040) & 0xFFFF, r)
    return r.astype(np.uint16)


def bf16_to_f32(b: np.ndarray) -> np.ndarray:
    return widen(np.asarray(b, dtype=np.uint16))


def _finish(acc: np.ndarray, scale: float, out_dtype: str) -> np.ndarray:
    """Root/owner epilogue: one fp32 multiply by ``scale`` then the output cast
    (reading R3: gradient scale applied once to the fp32 total)."""
    y = np.multiply(acc, np.float32(scale), dtype=np.float32)
    if out_dtype == F32:
        return y
    if out_dtype == BF16:
        return bf16_rne(y)
    if out_dtype == F16:
        return y.astype(np.float16)  # numpy's float32 -> binary16 conversion rounds to nearest even
    if out_dtype in (E4M3, E5M2):
        return fp8_rne(y, out_dtype)
    raise ValueError(out_dtype)


def _out_dtype(xs) -> str:
    fmt = fp8_format(xs[0].dtype)
    if fmt:
        return fmt
    if xs[0].dtype == np.uint16:
        return BF16
    if xs[0].dtype == np.float16:
        return F16
    return F32


def _out_np(out_dtype: str):
    return {F32: np.float32, BF16: np.uint16, F16: np.float16, E4M3: E4M3_DT, E5M2: E5M2_DT}[out_dtype]


# ----------------------------------------------------------------------------
# Algorithm 1 order: rank-ascending left fold (the flat path's reference)
# ----------------------------------------------------------------------------

def fold_ascending(xs, scale: float = 1.0) -> np.ndarray:
    """``acc = x_0; for r in 1..n-1: acc = fl32(acc + x_r)``; then scale, cast.

    PAPER.md:333-336 (Alg. 1 inner loop "For j in GPU_Count: Dc_i += GPU-j's
    Dc_i"), starting the accumulator from source 0 (reading R6, keeps -0.0).
    Explicit loop over ranks — never ``np.sum(axis=0)``, whose order is an
    implementation detail.
    """
    if len(xs) == 0:
        raise ValueError("empty source set")
    acc = widen(xs[0]).astype(np.float32, copy=True)
    for r in range(1, len(xs)):
        acc = np.add(acc, widen(xs[r]), dtype=np.float32)
    return _finish(acc, scale, _out_dtype(xs))


# ----------------------------------------------------------------------------
# Double binary tree (reading R9) — PAPER.md:297, 315, 406 cite it, no
# construction is given (bibliography absent).
# ----------------------------------------------------------------------------

def _tree_a(n: int):
    """In-order binary tree over ranks 0..n-1 (NCCL-style, reading R9).

    Returns (parent, children) with parent[root] = -1 and children[v] a list of
    child ranks.  Root is 0 with the single child = highest power of two < n.
    Node r != 0 with lowest set bit b: parent = (r ^ b) | (b << 1), or r ^ b if
    that is >= n.  Children of r (b > 1): r - b/2, and r + h for the largest
    h in {b/2, b/4, ...} with r + h < n.
    """
    parent = [-1] * n
    children = [[] for _ in range(n)]
    for r in range(1, n):
        b = r & -r
        p = (r ^ b) | (b << 1)
        if p >= n:
            p = r ^ b
        parent[r] = p
    # derive children from parents (single source of truth), ascending rank
    for r in range(1, n):
        children[parent[r]].append(r)
    for c in children:
        c.sort()
    return parent, children


def build_double_binary_tree(n: int):
    """Two trees (A, B), each as (parent list, children lists).

    Tree B is tree A relabelled by f(r) = n-1-r for even n (mirror) and
    f(r) = (r+1) mod n for odd n (shift).  Reading R9.
    """
    if n < 1:
        raise ValueError("n must be >= 1")
    pa, ca = _tree_a(n)
    if n % 2 == 0:
        f = lambda r: n - 1 - r  # noqa: E731
    else:
        f = lambda r: (r + 1) % n  # noqa: E731
    pb = [-1] * n
    cb = [[] for _ in range(n)]
    for r in range(n):
        pb[f(r)] = -1 if pa[r] < 0 else f(pa[r])
    for r in range(n):
        if pb[r] >= 0:
            cb[pb[r]].append(r)
    for c in cb:
        c.sort()
    return (pa, ca), (pb, cb)


def tree_root(tree) -> int:
    parent, _ = tree
    return parent.index(-1)


def _eval_tree(tree, v: int, vals) -> np.ndarray:
    """E(v) = ((E(children < v) + x_v) + E(children > v)), each child subtree
    added in ascending rank order (reading R10: fixed in-order combination at
    a tree node, ``DL_i += DR_i`` of PAPER.md:354 made arrival-independent)."""
    _, children = tree
    below = [c for c in children[v] if c < v]
    above = [c for c in children[v] if c > v]
    acc = None
    for c in below:
        e = _eval_tree(tree, c, vals)
        acc = e if acc is None else np.add(acc, e, dtype=np.float32)
    acc = vals[v] if acc is None else np.add(acc, vals[v], dtype=np.float32)
    for c in above:
        acc = np.add(acc, _eval_tree(tree, c, vals), dtype=np.float32)
    return acc


def fold_tree(xs, chunk_elems: int, scale: float = 1.0) -> np.ndarray:
    """Per-element result of the double-binary-tree allreduce (Alg. 2).

    Chunk c = elements [c*C, (c+1)*C) rides tree A if c is even, tree B if odd
    (reading R8).  Within a chunk the root's value is E(root) (pass 1,
    PAPER.md:350-362); pass 2 copies it unchanged to every
    rank, so the result is E(root) after the root's scale and cast.
    """
    n = len(xs)
    count = xs[0].shape[0]
    trees = build_double_binary_tree(n)
    out_dtype = _out_dtype(xs)
    out = np.empty(count, dtype=_out_np(out_dtype))
    for c0 in range(0, count, chunk_elems):
        c = c0 // chunk_elems
        sl = slice(c0, min(c0 + chunk_elems, count))
        tree = trees[c % 2]
        vals = [widen(x[sl]) for x in xs]
        out[sl] = _finish(_eval_tree(tree, tree_root(tree), vals), scale, out_dtype)
    return out


def pair_split(count: int) -> int:
    """Start of the second half for the pair-first variant (reading R13):
    H = min(N, 256 * ceil(N / 512)) — ceil(N/2) rounded up to 256 elements."""
    return min(count, PAIR_SPLIT_ALIGN * ((count + 2 * PAIR_SPLIT_ALIGN - 1) // (2 * PAIR_SPLIT_ALIGN)))


def fold_pairfirst(xs, chunk_elems: int, scale: float = 1.0) -> np.ndarray:
    """"HFReduce with NVLink", reading R13.

    1. pair partials p_k = fl32(x_{2k} + x_{2k+1}), k = 0..n/2-1 (NVLink pair
       reduce before the inter-node stage);
    2. the buffer is split into halves [0, H) and [H, N); within each half,
       chunk c (counted from the half's start) rides tree T_{c mod 2} of the
       double binary tree over the n/2 pair partials;
    3. root scale + cast; the result is returned to the pairs and all-gathered
       unchanged.
    """
    n = len(xs)
    if n % 2:
        raise ValueError("pair-first needs an even number of ranks")
    count = xs[0].shape[0]
    m = n // 2
    trees = build_double_binary_tree(m)
    out_dtype = _out_dtype(xs)
    out = np.empty(count, dtype=_out_np(out_dtype))
    H = pair_split(count)
    for lo, hi in ((0, H), (H, count)):
        for c0 in range(lo, hi, chunk_elems):
            c = (c0 - lo) // chunk_elems
            sl = slice(c0, min(c0 + chunk_elems, hi))
            p = [np.add(widen(xs[2 * k][sl]), widen(xs[2 * k + 1][sl]), dtype=np.float32)
                 for k in range(m)]
            tree = trees[c % 2]
            out[sl] = _finish(_eval_tree(tree, tree_root(tree), p), scale, out_dtype)
    return out


# ----------------------------------------------------------------------------
# The other collectives ("general reduce and broadcast", PAPER.md:297;
# SURVEY NEXT-3).  Shard layout = reading R19.
# ----------------------------------------------------------------------------

def shard_bounds(count: int, n: int, elems_per_vec: int):
    """Reading R19: shard g = [K*floor(V*g/n), K*floor(V*(g+1)/n)) with K the
    elements per 16 bytes and V = floor(count/K); the last shard also takes the
    ragged tail [K*V, count)."""
    V = count // elems_per_vec
    lo = [elems_per_vec * (V * g // n) for g in range(n)]
    hi = lo[1:] + [count]
    return list(zip(lo, hi))


def _k(xs):
    """Elements per 16-byte vector."""
    return 16 // xs[0].dtype.itemsize


def reduce_scatter(xs, scale: float = 1.0):
    """Rank g's shard g := rank-ascending fold of shard g (Alg. 1 order),
    scaled and cast; everything else of rank g's buffer unchanged."""
    n = len(xs)
    out = [x.copy() for x in xs]
    for g, (lo, hi) in enumerate(shard_bounds(xs[0].shape[0], n, _k(xs))):
        out[g][lo:hi] = fold_ascending([x[lo:hi] for x in xs], scale)
    return out


def all_gather(xs):
    """Every rank's shard g := rank g's shard g (raw values)."""
    n = len(xs)
    out = [x.copy() for x in xs]
    for g, (lo, hi) in enumerate(shard_bounds(xs[0].shape[0], n, _k(xs))):
        for r in range(n):
            out[r][lo:hi] = xs[g][lo:hi]
    return out


def reduce(xs, root: int, scale: float = 1.0):
    """Root's buffer := the allreduce result; the others unchanged."""
    out = [x.copy() for x in xs]
    out[root] = fold_ascending(xs, scale)
    return out


def broadcast(xs, root: int):
    """Every rank's buffer := root's buffer."""
    return [xs[root].copy() for _ in xs]


def allreduce(xs, algo: str = "flat", chunk_elems: int = 1 << 16, scale: float = 1.0):
    """Every rank's output (identical bytes on all ranks) for the given order."""
    if algo in ("flat", "oneshot", "auto", "ce"):
        y = fold_ascending(xs, scale)
    elif algo == "dbt":
        y = fold_tree(xs, chunk_elems, scale)
    elif algo == "pair_dbt":
        y = fold_pairfirst(xs, chunk_elems, scale)
    else:
        raise ValueError(algo)
    return [y.copy() for _ in xs]

