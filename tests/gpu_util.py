"""Helpers shared by the GPU tests (host-side marshalling only)."""
from __future__ import annotations

import numpy as np

import hfr_inputs as gen


def _fp8(x: np.ndarray):
    md = x.dtype.metadata
    return md.get("hfr") if md else None


def to_torch(x: np.ndarray, device):
    import torch
    fmt = _fp8(x)
    if fmt:
        t = torch.from_numpy(np.ascontiguousarray(x).view(np.uint8))
        return t.view(torch.float8_e4m3fn if fmt == gen.E4M3 else torch.float8_e5m2).to(device)
    if x.dtype == np.uint16:
        return torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(device)
    return torch.from_numpy(x).to(device)


def dtype_of(x: np.ndarray) -> str:
    """The hfr_inputs dtype name of an input array."""
    fmt = _fp8(x)
    if fmt:
        return fmt
    return {np.dtype(np.uint16): gen.BF16, np.dtype(np.float16): gen.FP16}.get(x.dtype, gen.FP32)


def torch_dtype(dtype: str):
    import torch
    return {gen.BF16: torch.bfloat16, gen.FP16: torch.float16, gen.E4M3: torch.float8_e4m3fn,
            gen.E5M2: torch.float8_e5m2}.get(dtype, torch.float32)


def to_numpy(t) -> np.ndarray:
    import torch
    if t.dtype == torch.bfloat16:
        return t.detach().cpu().view(torch.int16).numpy().view(np.uint16)
    if t.dtype == torch.float8_e4m3fn:
        return t.detach().cpu().view(torch.uint8).numpy().view(gen.E4M3_DT)
    if t.dtype == torch.float8_e5m2:
        return t.detach().cpu().view(torch.uint8).numpy().view(gen.E5M2_DT)
    return t.detach().cpu().numpy()


def as_f32(x: np.ndarray) -> np.ndarray:
    fmt = _fp8(x)
    if fmt:
        import torch
        t = torch.from_numpy(np.ascontiguousarray(x).view(np.uint8))
        return t.view(torch.float8_e4m3fn if fmt == gen.E4M3 else torch.float8_e5m2).float().numpy()
    if x.dtype == np.uint16:
        return (x.astype(np.uint32) << np.uint32(16)).view(np.float32)
    if x.dtype == np.float16:
        return x.astype(np.float32)
    return x


def _bits(x: np.ndarray) -> np.ndarray:
    return x.view({1: np.uint8, 2: np.uint16}.get(x.dtype.itemsize, np.uint32))


def assert_bit_exact(got: np.ndarray, want: np.ndarray, what: str = ""):
    """Identical bits everywhere except NaN payloads (reading R5: compare NaN
    positions, not payloads)."""
    assert got.shape == want.shape and got.dtype == want.dtype, what
    g, w = as_f32(got), as_f32(want)
    gn, wn = np.isnan(g), np.isnan(w)
    if not np.array_equal(gn, wn):
        i = int(np.flatnonzero(gn != wn)[0])
        raise AssertionError(f"{what}: NaN mismatch at {i}: got {g[i]!r} want {w[i]!r}")
    m = ~wn
    gb = _bits(got[m])
    wb = _bits(want[m])
    if not np.array_equal(gb, wb):
        bad = np.flatnonzero(gb != wb)
        idx = np.flatnonzero(m)[bad[:5]]
        raise AssertionError(f"{what}: {bad.size} mismatching elements, first at {idx.tolist()}: "
                             f"got {g[idx].tolist()} want {w[idx].tolist()}")


def assert_within_r18(got: np.ndarray, xs, want: np.ndarray, scale: float, what: str = ""):
    """DESIGN.md reading R18 (order-relaxed paths): with A = sum_r |x_r| per
    element, fp32 |got - want| <= 1e-6 * scale * A; bf16 |got - want| <=
    max(1 ulp(want), 8.3e-7 * scale * A + 1/2 ulp(want)).  NaN/Inf positions
    must match."""
    g = as_f32(got).astype(np.float64)
    w = as_f32(want).astype(np.float64)
    A = np.zeros_like(w)
    for x in xs:
        A += np.abs(as_f32(x).astype(np.float64))
    A *= abs(scale)
    fin = np.isfinite(w)
    assert np.array_equal(np.isnan(g), np.isnan(w)), f"{what}: NaN positions"
    assert np.array_equal(g[~fin], w[~fin]) or not (~fin).any(), f"{what}: Inf mismatch"
    d = np.abs(g[fin] - w[fin])
    if got.dtype.itemsize == 2:
        bits, emin = (7, -126) if got.dtype == np.uint16 else (10, -14)
        ex = np.floor(np.log2(np.maximum(np.abs(w[fin]), 2.0 ** emin)))
        ulp = 2.0 ** (ex - bits)
        lim = np.maximum(ulp, 8.3e-7 * A[fin] + 0.5 * ulp)
    else:
        lim = 1e-6 * A[fin]
    bad = np.flatnonzero(d > lim)
    assert bad.size == 0, f"{what}: {bad.size} elements beyond R18, worst {float((d - lim).max())}"
