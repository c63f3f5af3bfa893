"""Counter-hash input generator (SURVEY.md §8(d) "Inputs").

value(seed, stream, i) = ((splitmix64(seed ^ (stream << 40) ^ i) >> 56) - 128) * 2**-shift

The top byte gives an integer k in [-128, 127]; k * 2**-shift has at most 8
significant bits, so it is exact in bf16 (8-bit significand) and in fp32.

Streams (fixed recipe):
  * STREAM_PARAM = 1,       shift 12: |x| <= 0.031, std ~0.018 (LLM init ~0.02)
  * STREAM_GRAD0 + r,       shift 14: gradient of rank r; one element in 1024
                            (selected by hash bits 20..29 == 0) is scaled by 64
                            (still exact) so quantization blocks see outliers.
  * STREAM_MCODE/VCODE/ABS: synthetic "warm" 8-bit Adam state for large
                            benchmarks (codes and per-block absmax); small
                            parity tests instead warm the state with oracle
                            steps.

Indices are *logical* flat indices (tensor order, no padding), so the logical
parameters do not depend on the layout or on the world size.

Two implementations with identical output: numpy (host) and torch (any
device, used to fill HBM quickly for the benchmark).  tests/test_synth.py
checks that they agree.
"""
from __future__ import annotations

import numpy as np

STREAM_PARAM = 1
STREAM_GRAD0 = 16
STREAM_MCODE = 64
STREAM_VCODE = 65
STREAM_ABSM = 66
STREAM_ABSV = 67
PARAM_SHIFT = 12
GRAD_SHIFT = 14
OUTLIER_SCALE = 64.0

_C0 = 0x9E3779B97F4A7C15
_C1 = 0xBF58476D1CE4E5B9
_C2 = 0x94D049BB133111EB


# ----------------------------------------------------------------------------
# numpy
# ----------------------------------------------------------------------------
def splitmix64_np(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64, copy=False)
    with np.errstate(over="ignore"):
        z = x + np.uint64(_C0)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_C1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_C2)
        return z ^ (z >> np.uint64(31))


def _raw_np(seed: int, stream: int, start: int, n: int) -> np.ndarray:
    i = np.arange(start, start + n, dtype=np.uint64)
    key = np.uint64((seed ^ (stream << 40)) & 0xFFFFFFFFFFFFFFFF)
    return splitmix64_np(i ^ key)


def values_np(seed: int, stream: int, start: int, n: int, shift: int,
              outliers: bool = False) -> np.ndarray:
    """float32 array of n values for logical indices [start, start+n)."""
    h = _raw_np(seed, stream, start, n)
    k = (h >> np.uint64(56)).astype(np.int64) - 128
    x = k.astype(np.float32) * np.float32(2.0 ** -shift)
    if outliers:
        sel = ((h >> np.uint64(20)) & np.uint64(1023)) == 0
        x[sel] *= np.float32(OUTLIER_SCALE)
    return x


def params_np(seed: int, start: int, n: int) -> np.ndarray:
    return values_np(seed, STREAM_PARAM, start, n, PARAM_SHIFT)


def grads_np(seed: int, rank: int, start: int, n: int) -> np.ndarray:
    return values_np(seed, STREAM_GRAD0 + rank, start, n, GRAD_SHIFT, outliers=True)


def codes_np(seed: int, stream: int, start: int, n: int, signed: bool) -> np.ndarray:
    """Uniform 8-bit codes: int8 in [-127, 127] or uint8 in [0, 255]."""
    h = _raw_np(seed, stream, start, n)
    b = (h >> np.uint64(56)).astype(np.int64)
    if signed:
        return ((b % 255) - 127).astype(np.int8)
    return b.astype(np.uint8)


def absmax_np(seed: int, stream: int, start: int, n: int, shift: int) -> np.ndarray:
    """Positive per-block absmax values (k+1) * 2**-shift, k in [0, 255]."""
    h = _raw_np(seed, stream, start, n)
    k = (h >> np.uint64(56)).astype(np.int64) + 1
    return k.astype(np.float32) * np.float32(2.0 ** -shift)


# ----------------------------------------------------------------------------
# torch (same values; int64 arithmetic wraps like uint64, shifts made logical)
# ----------------------------------------------------------------------------
def _s64(c: int) -> int:
    return c - (1 << 64) if c >= (1 << 63) else c


def _srl(x, k: int):
    import torch  # noqa: F401
    return (x >> k) & ((1 << (64 - k)) - 1)


def _raw_torch(seed: int, stream: int, start: int, n: int, device):
    import torch
    i = torch.arange(start, start + n, dtype=torch.int64, device=device)
    key = _s64((seed ^ (stream << 40)) & 0xFFFFFFFFFFFFFFFF)
    z = (i ^ key) + _s64(_C0)
    z = (z ^ _srl(z, 30)) * _s64(_C1)
    z = (z ^ _srl(z, 27)) * _s64(_C2)
    return z ^ _srl(z, 31)


def values_torch(seed: int, stream: int, start: int, n: int, shift: int,
                 outliers: bool = False, device="cpu", chunk: int = 1 << 26):
    """float32 tensor on `device`, identical to values_np; built in chunks."""
    import torch
    out = torch.empty(n, dtype=torch.float32, device=device)
    for c0 in range(0, n, chunk):
        c = min(chunk, n - c0)
        h = _raw_torch(seed, stream, start + c0, c, device)
        k = _srl(h, 56) - 128
        x = k.to(torch.float32) * (2.0 ** -shift)
        if outliers:
            sel = (_srl(h, 20) & 1023) == 0
            x = torch.where(sel, x * OUTLIER_SCALE, x)
        out[c0:c0 + c] = x
        del h, k, x
    return out


def params_torch(seed: int, start: int, n: int, device="cpu"):
    return values_torch(seed, STREAM_PARAM, start, n, PARAM_SHIFT, device=device)


def grads_torch(seed: int, rank: int, start: int, n: int, device="cpu"):
    return values_torch(seed, STREAM_GRAD0 + rank, start, n, GRAD_SHIFT,
                        outliers=True, device=device)


def codes_torch(seed: int, stream: int, start: int, n: int, signed: bool,
                device="cpu", chunk: int = 1 << 26):
    import torch
    out = torch.empty(n, dtype=torch.int8 if signed else torch.uint8, device=device)
    for c0 in range(0, n, chunk):
        c = min(chunk, n - c0)
        b = _srl(_raw_torch(seed, stream, start + c0, c, device), 56)
        out[c0:c0 + c] = ((b % 255) - 127).to(torch.int8) if signed else b.to(torch.uint8)
    return out


def absmax_torch(seed: int, stream: int, start: int, n: int, shift: int, device="cpu"):
    import torch
    k = _srl(_raw_torch(seed, stream, start, n, device), 56) + 1
    return k.to(torch.float32) * (2.0 ** -shift)
