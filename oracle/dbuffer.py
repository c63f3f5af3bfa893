"""Oracle DBuffer: steps a4 (AllGather), a5 (views), a6 (grouped cast/scale),
a7 (ReduceScatter).  SURVEY.md §8(c) O2/O3.  TEST INFRASTRUCTURE ONLY.

Semantics from PAPER.md:
  * device k owns [k*S, (k+1)*S) of the m*S global buffer;
  * tensors are zero-copy views at [l_t, l_t + e_t);
  * group-level ops: "identical kernels across tensors are fused before
    communication" -- the gradient cast bf16->fp32 and the 1/m
    scale are applied to the whole buffer in one pass *before* the
    ReduceScatter; padding is written 0 (O2 deviation);
  * ReduceScatter sums the m ranks' buffers; rank k receives slice k.  The
    oracle sums in rank order 0..m-1 in fp32 (R12); ``reduce_scatter_f64`` is
    the once-rounded reference used for the error bound.

Parity pins (tests/test_oracle_dbuffer.py): AG o shard = identity (bit exact),
views alias the buffer, RS = per-rank sum (closed form on dyadic inputs where
fp32 sums are exact), error bound (m-1)*2^-24*sum|x| vs the fp64 sum, bf16
once-rounding.
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

from .planner import Layout


def to_bf16_rne(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (round to nearest even), returned as uint16 bit patterns.
    NaN is kept NaN (quiet)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    r = ((u + rounding) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        r[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return r


def bf16_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def place_logical(lay: Layout, flat: np.ndarray, fill=0) -> np.ndarray:
    """Global m*S buffer holding the logical (padding-free, tensor-order) flat
    vector at each tensor's interval; padding = fill.  This is what writing
    through the zero-copy views produces."""
    buf = np.full(lay.m * lay.S, fill, dtype=flat.dtype)
    off = 0
    for l, e in zip(lay.starts, lay.numel):
        buf[l:l + e] = flat[off:off + e]
        off += e
    return buf


def views(lay: Layout, buf: np.ndarray) -> List[np.ndarray]:
    """a5: tensor t = buf[l_t : l_t + e_t] (numpy slices alias the buffer)."""
    return [buf[l:l + e] for l, e in zip(lay.starts, lay.numel)]


def shard(lay: Layout, buf: np.ndarray, rank: int) -> np.ndarray:
    return buf[rank * lay.S:(rank + 1) * lay.S]


def all_gather(shards: Sequence[np.ndarray]) -> np.ndarray:
    """a4: every rank receives the concatenation of all shards in rank order."""
    return np.concatenate([np.asarray(s) for s in shards])


def grouped_cast_scale(lay: Layout, grad: np.ndarray, src_is_bf16: bool) -> np.ndarray:
    """a6: one pass over the unit's gradient buffer: fp32(grad) * fl32(1/m);
    padding positions are written 0."""
    g = bf16_to_f32(grad) if src_is_bf16 else np.asarray(grad, dtype=np.float32)
    out = g * np.float32(1.0 / lay.m)
    for a, b in lay.padding_intervals():
        out[a:b] = 0
    return out.astype(np.float32)


def reduce_scatter(lay: Layout, bufs: Sequence[np.ndarray]) -> List[np.ndarray]:
    """a7: y_k = sum_{r=0..m-1} bufs[r][kS:(k+1)S], fp32, rank order."""
    assert len(bufs) == lay.m
    S = lay.S
    out = []
    for k in range(lay.m):
        acc = np.zeros(S, dtype=np.float32)
        for r in range(lay.m):
            acc = (acc + np.asarray(bufs[r][k * S:(k + 1) * S], dtype=np.float32)).astype(np.float32)
        out.append(acc)
    return out


def reduce_scatter_f64(lay: Layout, bufs: Sequence[np.ndarray]) -> List[np.ndarray]:
    """Exact-sum reference: fp64 accumulation (exact for <= 2^29 fp32 terms of
    bounded exponent range here), returned in fp64."""
    S = lay.S
    return [sum(np.asarray(bufs[r][k * S:(k + 1) * S], dtype=np.float64)
                for r in range(lay.m)) for k in range(lay.m)]


def f64_to_bf16_rne(x: np.ndarray) -> np.ndarray:
    """fp64 -> bf16 with ONE rounding (RNE): fp64 -> fp32 round-to-odd, then
    fp32 -> bf16 RNE (exact because fp32 carries >= 2 extra bits)."""
    x = np.asarray(x, dtype=np.float64)
    t = x.astype(np.float32)
    inexact = t.astype(np.float64) != x
    over = inexact & (np.abs(t.astype(np.float64)) > np.abs(x))
    t[over] = np.nextafter(t[over], np.float32(0))
    bits = t.view(np.uint32).copy()
    bits[inexact] |= np.uint32(1)
    return to_bf16_rne(bits.view(np.float32))


def reduce_scatter_bf16(lay: Layout, grads_bf16: Sequence[np.ndarray]) -> List[np.ndarray]:
    """bf16 mode: y16 = bf16_RNE(exact sum of fp32(G_r) * 1/m),
    rounded once.  The fp64 sum of m <= 8 bf16 values is exact."""
    S = lay.S
    out = []
    for k in range(lay.m):
        acc = np.zeros(S, dtype=np.float64)
        for r in range(lay.m):
            acc += bf16_to_f32(grads_bf16[r][k * S:(k + 1) * S]).astype(np.float64)
        out.append(f64_to_bf16_rne(acc / lay.m))
    return out
