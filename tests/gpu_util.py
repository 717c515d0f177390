"""Helpers shared by the GPU tests (host-side marshalling only)."""
from __future__ import annotations

import numpy as np

import hfr_inputs as gen


def to_torch(x: np.ndarray, device):
    import torch
    if x.dtype == np.uint16:
        return torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(device)
    return torch.from_numpy(x).to(device)


def torch_dtype(dtype: str):
    import torch
    return torch.bfloat16 if dtype == gen.BF16 else torch.float32


def to_numpy(t) -> np.ndarray:
    import torch
    if t.dtype == torch.bfloat16:
        return t.detach().cpu().view(torch.int16).numpy().view(np.uint16)
    return t.detach().cpu().numpy()


def as_f32(x: np.ndarray) -> np.ndarray:
    if x.dtype == np.uint16:
        return (x.astype(np.uint32) << np.uint32(16)).view(np.float32)
    return x


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
    gb = got[m].view(np.uint16 if got.dtype == np.uint16 else np.uint32)
    wb = want[m].view(np.uint16 if want.dtype == np.uint16 else np.uint32)
    if not np.array_equal(gb, wb):
        bad = np.flatnonzero(gb != wb)
        idx = np.flatnonzero(m)[bad[:5]]
        raise AssertionError(f"{what}: {bad.size} mismatching elements, first at {idx.tolist()}: "
                             f"got {g[idx].tolist()} want {w[idx].tolist()}")
