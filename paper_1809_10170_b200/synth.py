"""Seeded synthetic data (BASELINE.json: i.i.d. uniform[-1, 1]).

Counter-based splitmix64 -> 24-bit mantissa, identical on CPU and GPU tensors
and bit-identical to the CPU checker's generator (oracle/oracle.c), so host-generated
inputs (bench e2e) and device-generated ones (bench value, tests) agree, and
the CPU oracle can regenerate any tensor from (seed, stream)."""
from __future__ import annotations

import torch


def _u64(v: int) -> int:
    """uint64 constant as the int64 with the same bits."""
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


_G = _u64(0x9E3779B97F4A7C15)
_C1 = _u64(0xBF58476D1CE4E5B9)
_C2 = _u64(0x94D049BB133111EB)
_S1 = _u64(0xD1B54A32D192ED03)
_S2 = _u64(0x8CB92BA72F3D8DD7)


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    return (x >> k) & ((1 << (64 - k)) - 1)


def uniform_values(numel: int, seed: int, stream: int, device, offset: int = 0,
                   chunk: int = 1 << 24) -> torch.Tensor:
    base = _u64(_u64(seed * _S1) ^ _u64(stream * _S2))
    out = torch.empty(numel, dtype=torch.float32, device=device)
    for lo in range(0, numel, chunk):
        hi = min(numel, lo + chunk)
        x = torch.arange(lo + offset, hi + offset, dtype=torch.int64, device=device)
        x = x + base
        x = x + _G
        x = (x ^ _srl(x, 30)) * _C1
        x = (x ^ _srl(x, 27)) * _C2
        x = x ^ _srl(x, 31)
        r = _srl(x, 40).to(torch.float32)
        out[lo:hi] = r * (1.0 / 8388608.0) - 1.0
    return out


def fill_uniform_(t: torch.Tensor, seed: int, stream: int, scale: float = 1.0) -> torch.Tensor:
    v = uniform_values(t.numel(), seed, stream, t.device)
    if scale != 1.0:
        v = v * scale
    t.copy_(v.view(t.shape))
    return t
