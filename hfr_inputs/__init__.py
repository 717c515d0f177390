"""Seeded synthetic input generators shared by tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic: it only draws random
per-rank gradient buffers (numpy) with the shapes and value distributions
DESIGN.md §"Input recipe" lists. Both the oracle (oracle/) and the CUDA path
(paper_2408_14158_b200/) consume these arrays; neither side imports the other.

Dtype encoding: fp32 buffers are ``np.float32`` arrays; bf16 buffers are
``np.uint16`` arrays holding the raw bfloat16 bit patterns; fp16 buffers are
``np.float16``.  bf16 values are obtained by TRUNCATING a float32 draw to its
top 16 bits (round-toward-zero bit slicing); fp16 values by numpy's
float32 -> float16 conversion of the draw (input generation only).

Seeds follow SURVEY.md §8d: ``np.random.default_rng(base + rank)``.
"""
from __future__ import annotations

import numpy as np

FP32 = "f32"
BF16 = "bf16"
FP16 = "f16"
E4M3 = "e4m3"
E5M2 = "e5m2"
FP8 = (E4M3, E5M2)

# FP8 bit-pattern arrays: uint8 tagged with the format in the dtype metadata
# (numpy has no fp8 type; the oracle reads the same tag)
E4M3_DT = np.dtype(np.uint8, metadata={"hfr": E4M3})
E5M2_DT = np.dtype(np.uint8, metadata={"hfr": E5M2})

# Distribution names:
#   normal     N(0, 1)
#   grad       N(0, 1e-3^2)  gradient-like (C2)
#   int        integers, |x| < 2^20 for fp32 (every partial sum exact for n <= 8),
#              |x| <= 256 for bf16 (bf16-exact, fp32 sums exact in any order)
#   loguniform magnitudes log-uniform in [2^-20, 2^4], random sign (C3)
#   specials   mixture of +-0, subnormals, +-Inf, NaN, 2^24 and 1 (C1 (iii))
DISTS = ("normal", "grad", "int", "loguniform", "specials")


def _draw_f32(rng: np.random.Generator, dist: str, count: int, dtype: str) -> np.ndarray:
    if dist == "normal":
        return rng.standard_normal(count, dtype=np.float32)
    if dist == "grad":
        return (rng.standard_normal(count, dtype=np.float32) * np.float32(1e-3)).astype(np.float32)
    if dist == "int":
        # bf16/fp16: |x| <= 256 exact, sums exact in fp32; FP8: |x| <= 8 exact in both formats
        lim = (1 << 20) - 1 if dtype == FP32 else (8 if dtype in FP8 else 256)
        return rng.integers(-lim, lim + 1, size=count, dtype=np.int64).astype(np.float32)
    if dist == "loguniform":
        e = rng.uniform(-20.0, 4.0, size=count)
        s = rng.choice(np.array([-1.0, 1.0]), size=count)
        return (s * np.exp2(e)).astype(np.float32)
    if dist == "specials":
        pool = np.array(
            [0.0, -0.0, 1.0, -1.0, 2.0 ** 24, 1.5, np.inf, -np.inf, np.nan,
             np.float32(1e-40), np.float32(-1e-40), np.float32(1.17549435e-38),
             np.float32(3.4e38), np.float32(-3.4e38), np.float32(2.0 ** -149)],
            dtype=np.float32)
        pick = rng.integers(0, len(pool), size=count)
        out = pool[pick]
        # a third of the entries are ordinary normals so the mix is not all-special
        mask = rng.random(count) < 0.33
        out[mask] = rng.standard_normal(int(mask.sum()), dtype=np.float32)
        return out
    raise ValueError(f"unknown distribution {dist!r}")


def _to_dtype(x: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == FP32:
        return np.ascontiguousarray(x, dtype=np.float32)
    if dtype == BF16:
        return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)
    if dtype == FP16:
        with np.errstate(over="ignore"):
            return np.ascontiguousarray(x, dtype=np.float32).astype(np.float16)
    if dtype in FP8:
        # input generation only: PyTorch's float32 -> float8 conversion of the draw
        import torch
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
        t = t.to(torch.float8_e4m3fn if dtype == E4M3 else torch.float8_e5m2)
        return t.view(torch.uint8).numpy().view(E4M3_DT if dtype == E4M3 else E5M2_DT)
    raise ValueError(f"unknown dtype {dtype!r}")


def rank_input(rank: int, count: int, dtype: str = FP32, dist: str = "normal",
               seed_base: int = 1234) -> np.ndarray:
    """One rank's buffer: ``count`` elements drawn with ``default_rng(seed_base + rank)``."""
    rng = np.random.default_rng(seed_base + rank)
    return _to_dtype(_draw_f32(rng, dist, count, dtype), dtype)


def rank_inputs(nranks: int, count: int, dtype: str = FP32, dist: str = "normal",
                seed_base: int = 1234) -> list[np.ndarray]:
    """Buffers for all ranks of one allreduce (list index = communicator rank)."""
    return [rank_input(r, count, dtype, dist, seed_base) for r in range(nranks)]


def low_bits_cleared(x: np.ndarray, bits: int) -> np.ndarray:
    """fp32 array with the low ``bits`` mantissa bits zeroed (for the n*x invariant)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    return (u & np.uint32((0xFFFFFFFF << bits) & 0xFFFFFFFF)).view(np.float32)


# Paper-scale sizes.
C1_COUNT = 4096                      # config 1: 2 ranks x 4096 fp32
C2_COUNT = 186 * (1 << 20) // 4      # config 2: 186 MiB fp32 = 48,758,784 elements
C5_BUCKET_BYTES = 64 << 20           # config 5: 64 MiB buckets
C5_PARAMS = 7_000_000_000            # config 5: 7B bf16 gradient volume


def c3_sizes_bytes() -> list[int]:
    """config 3: message sizes 1 KiB .. 1 GiB (powers of two)."""
    return [1024 << k for k in range(21)]


def rank_input_torch(rank: int, count: int, dtype: str = FP32, seed_base: int = 7000, device="cuda"):
    """Large seeded N(0,1) buffer generated on the device (torch.Generator
    seeded with seed_base + rank), for full-size (1 GiB) cases whose host
    generation would be slow.  Tests read sampled input elements back from the
    device before the call and give those to the oracle."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed_base + rank)
    x = torch.randn(count, generator=g, device=device, dtype=torch.float32)
    if dtype == BF16:
        return (x.view(torch.int32) >> 16).to(torch.int16).view(torch.bfloat16)  # truncation, as rank_input
    if dtype == FP16:
        return x.to(torch.float16)
    if dtype in FP8:
        return x.to(torch.float8_e4m3fn if dtype == E4M3 else torch.float8_e5m2)
    return x
