"""Oracle dynamic (tree) code map for 8-bit Adam states: SURVEY.md §8(f) N2,
"Also the dynamic (Dettmers) code map".  TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py).

PAPER.md P:419: "8-bit Adam applies block-wise INT8 quantization to the
gradient statistics", citing Dettmers et al. ([dettmers8], 8-bit optimizers
via block-wise quantization), whose states use a *dynamic* code: 256 values in
[-1, 1] spread over decades, quantization = nearest value of x / absmax.  The
paper prints no table; reading R25 takes Dettmers' dynamic
tree construction with 7 exponent levels:

  signed map (first moment m):  for i = 0..6, n = 2^i + 1 boundaries
      b_j = 0.1 + j * 0.9 / (n - 1)  (j = 0..n-1), means
      mu_j = 0.1 + (j + 0.5) * (0.9 / (n - 1))  (j = 0..n-2, 2^i values),
      values +-D_i * mu_j with D_i = 1e-6, 1e-5, ..., 1e0;  plus 0 and 1.
  unsigned map (second moment v): the same with n = 2^(i+1) + 1 and only the
      positive values;  plus 0 and 1.
  Each value is computed in fp64 exactly as written and rounded once to fp32;
  256 values, sorted ascending (index = the 8-bit code).
  quantize:   A = max|x| over the block; y = fl32(x / A); hi = first code with
              map[hi] >= y (clamped to [1, 255]), lo = hi - 1;
              code = hi if fl32(map[hi] - y) < fl32(y - map[lo]) else lo
              (ties -> the lower code); A = 0 -> the code of 0.  A is the
              NaN-propagating max; a block whose A is NaN or +inf (a
              non-finite gradient) keeps A and gets the code of 0 everywhere
              (reading R27, as the linear codec).
  dequantize: x = fl32(map[code] * A).
Both sides decide the code in fp32 with the same operations, so codes are
comparable bit for bit.

Pins (tests/test_oracle_codemap.py): 256 distinct sorted values, 0 and 1
present, decade populations 2^i (signed: each sign) / 2^(i+1) (unsigned),
symmetry of the signed map, agreement with Dettmers' published construction
re-evaluated independently in float32 torch (linspace + midpoints) within
fp32 rounding; quantization = brute-force nearest value; round trip of
values on the grid; the Adam step with this codec equals the linear-codec
step when the states are exactly representable in both.
"""
from __future__ import annotations

from functools import lru_cache
from typing import Tuple

import numpy as np

f32 = np.float32
DECADES = (1e-6, 1e-5, 1e-4, 1e-3, 1e-2, 1e-1, 1e0)


@lru_cache(maxsize=2)
def dynamic_map(signed: bool) -> np.ndarray:
    vals = [0.0, 1.0]
    for i, D in enumerate(DECADES):
        n = (2 ** i if signed else 2 ** (i + 1)) + 1
        for j in range(n - 1):
            mu = 0.1 + (j + 0.5) * (0.9 / (n - 1))
            vals.append(D * mu)
            if signed:
                vals.append(-(D * mu))
    out = np.array(sorted(float(f32(v)) for v in vals), dtype=f32)
    assert out.size == 256
    return out


def zero_code(signed: bool) -> int:
    return int(np.nonzero(dynamic_map(signed) == 0)[0][0])


def dyn_dequantize(codes: np.ndarray, absmax, signed: bool) -> np.ndarray:
    return (dynamic_map(signed)[np.asarray(codes, np.uint8)] * f32(absmax)).astype(f32)


def dyn_code(y: np.ndarray, signed: bool) -> np.ndarray:
    """Nearest map value of y (fp32 comparisons, ties to the lower code)."""
    mp = dynamic_map(signed)
    y = np.asarray(y, f32)
    hi = np.clip(np.searchsorted(mp, y, side="left"), 1, 255)
    lo = hi - 1
    d_hi = (mp[hi] - y).astype(f32)
    d_lo = (y - mp[lo]).astype(f32)
    return np.where(d_hi < d_lo, hi, lo).astype(np.uint8)


def dyn_quantize(x: np.ndarray, signed: bool) -> Tuple[np.ndarray, f32]:
    """One block -> (codes uint8, absmax)."""
    x = np.asarray(x, f32)
    a = f32(np.max(np.abs(x))) if x.size else f32(0)
    if a == 0 or not np.isfinite(a):  # R27: a NaN / infinite block keeps A, codes of 0
        return np.full(x.shape, zero_code(signed), np.uint8), a
    with np.errstate(under="ignore"):
        return dyn_code((x / a).astype(f32), signed), a
