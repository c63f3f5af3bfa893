"""Oracle FP8 (E4M3) block quantization of the parameters before the
AllGather: SURVEY.md §8(f) N2, "128x128 FP8 block quantization before AG
(1 B/elem AG for BJ config 4)".  TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py): only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference arm may import it.

Paper passages:
  P:42   "Block-wise Quantization. Quantizing model weights [DeepSeek-V3] ...
          per-block scaling factors ... communication-free block-wise
          quantization requires each quantization block to reside entirely
          on a single device."
  P:474  "Following a DeepSeek-style quantization scheme, we quantize only the
          FFN weights (most parameters) ... The 128-row setting reproduces
          DeepSeek's 128x128 tiling (i.e., weights can be sliced into 128x128
          blocks)."
  P:344  FP32 master weights.
The paper prints neither the FP8 format nor the scaling rule; the readings
(R18-R20) are:
  R18  Format: OCP FP8 E4M3 ("e4m3fn": 1 sign, 4 exponent bits with bias 7, 3
       mantissa bits, no infinities, largest finite 448 = S.1111.110, NaN =
       S.1111.111), round to nearest with ties to the even code, saturating
       to +-448; the sign of zero is kept.
  R19  Per tile of a 2-D weight viewed as [rows, cols] (128 x 128 tiles, edge
       tiles smaller), from the fp32 master weights:
           A     = max |x| over the tile
           inv   = fl32(448 / A)
           code  = E4M3(fl32(x * inv))          (RNE, saturating)
           scale = fl32(A / 448)                (dequantization factor)
       and x ~= decode(code) * scale.  A = 0: every code 0, scale 0.
  R20  The quantized unit holds the 2-D FFN weights only planned at
       128-row granularity, so every tile lies on one rank and
       the scales need no communication to compute.  Tile slots are numbered
       in buffer order (tensors in order, tiles row-major); rank r's tiles are
       a contiguous run of slots.
The AllGather of the codes (1 byte per element) and of the per-tile scales
is the concatenation of the ranks' shards (O2), bit exact.

Pins (tests/test_oracle_fp8.py): the decode table against the format's
landmarks (0x7E = 448, 0x38 = 1, 0x08 = 2^-6, 0x01 = 2^-9, NaN codes) and
torch's float8_e4m3fn view (library routine); encode against torch's
float8_e4m3fn cast on every finite value, every midpoint (ties) and random
inputs, and against a brute-force nearest search; the tile's max element
maps to +-448; the rounding bound |y - decode(code)| <= 2^-4 |y| + 2^-10 for
y = fl(x * inv); values already on a tile's grid round-trip exactly; rank
sharded quantization == unsharded per-tensor quantization (containment).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

from .planner import Layout, rank_tiles

f32 = np.float32
E4M3_MAX = 448.0
E4M3_NAN = 0x7F


def e4m3_value(code: int) -> float:
    """Decode one E4M3 code from the bit fields (R18)."""
    s = -1.0 if code & 0x80 else 1.0
    e = (code >> 3) & 0xF
    m = code & 0x7
    if e == 0xF and m == 0x7:
        return float("nan")
    if e == 0:
        return s * (m / 8.0) * 2.0 ** -6
    return s * (1.0 + m / 8.0) * 2.0 ** (e - 7)


def e4m3_table() -> np.ndarray:
    """All 256 codes decoded (fp32; NaN for 0x7F / 0xFF)."""
    return np.array([e4m3_value(c) for c in range(256)], dtype=f32)


def e4m3_decode(codes: np.ndarray) -> np.ndarray:
    return e4m3_table()[np.asarray(codes, dtype=np.uint8)]


def e4m3_encode(x: np.ndarray) -> np.ndarray:
    """fp32 -> E4M3 code, round to nearest, ties to the even code, saturating
    at +-448, sign of zero kept, NaN -> 0x7F (R18).  Nearest of the 127
    non-negative finite values by an explicit comparison with both
    neighbours."""
    x = np.asarray(x, dtype=f32)
    pos = e4m3_table()[:0x7F].astype(np.float64)  # codes 0x00..0x7E, increasing
    a = np.minimum(np.abs(x).astype(np.float64), E4M3_MAX)
    hi = np.searchsorted(pos, a, side="left")  # first value >= a
    hi = np.clip(hi, 0, 0x7E)
    lo = np.clip(hi - 1, 0, 0x7E)
    d_lo = a - pos[lo]
    d_hi = pos[hi] - a
    pick_hi = (d_hi < d_lo) | ((d_hi == d_lo) & (hi % 2 == 0))
    exact = pos[hi] == a
    code = np.where(exact | pick_hi, hi, lo).astype(np.uint8)
    code = np.where(np.signbit(x), code | 0x80, code).astype(np.uint8)
    return np.where(np.isnan(x), np.uint8(E4M3_NAN), code).astype(np.uint8)


def quantize_tile(x: np.ndarray) -> Tuple[np.ndarray, np.float32]:
    """One tile (any shape) of fp32 weights -> (codes, scale) per R19, made
    total by R28: A is the NaN-propagating max; inv = min(fl(448 / A),
    FLT_MAX), so a tile with A < 448 / FLT_MAX (fl(448/A) = inf) still maps
    every x to a finite fl(x * inv) (|x| <= A); a tile whose A is NaN or +inf
    gets the NaN code 0x7F everywhere and scale A (poisoned, visible)."""
    x = np.asarray(x, dtype=f32)
    A = f32(np.max(np.abs(x))) if x.size else f32(0)  # numpy's max propagates NaN
    if A == 0:
        return np.zeros(x.shape, np.uint8), f32(0)
    if not np.isfinite(A):
        return np.full(x.shape, E4M3_NAN, np.uint8), A
    with np.errstate(over="ignore", under="ignore"):
        inv = f32(min(f32(f32(E4M3_MAX) / A), np.finfo(f32).max))
        codes = e4m3_encode((x * inv).astype(f32))
        return codes, f32(A / f32(E4M3_MAX))


def tile_specs(row_len: Sequence[int], tile: int = 128) -> List[Tuple]:
    """("tile", C, tile, tile) for every tensor of row length C (R20)."""
    return [("tile", int(c), tile, tile) for c in row_len]


def slot_base(lay: Layout, rank: int, specs) -> int:
    """First scale slot of `rank` (tiles numbered in buffer order, R20)."""
    return sum(len(rank_tiles(lay, r, specs)) for r in range(rank))


def quantize_shard(lay: Layout, rank: int, master_shard: np.ndarray, specs):
    """Rank-local step: every tile of the rank's shard of the fp32 master ->
    (codes shard of S bytes, padding 0; scales of the rank's tiles)."""
    codes = np.zeros(lay.S, np.uint8)
    scales = []
    for off, rows, cols, pitch in rank_tiles(lay, rank, specs):
        idx = off + (np.arange(rows)[:, None] * pitch + np.arange(cols)[None, :])
        q, s = quantize_tile(master_shard[idx])
        codes[idx] = q
        scales.append(s)
    return codes, np.array(scales, dtype=f32)


def quantize_all_gather(lay: Layout, master_full: np.ndarray, specs):
    """Every rank quantizes its shard, then the AllGather of codes and scales
    (concatenation in rank order, O2).  master_full: the m*S fp32 buffer."""
    cs, ss = [], []
    for r in range(lay.m):
        c, s = quantize_shard(lay, r, master_full[r * lay.S:(r + 1) * lay.S], specs)
        cs.append(c)
        ss.append(s)
    return np.concatenate(cs) if cs else np.zeros(0, np.uint8), \
        np.concatenate(ss) if ss else np.zeros(0, f32)
