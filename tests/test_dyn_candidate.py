"""Host check (-m "not gpu") that the dynamic-codec kernel's branch-free code
decision (adam_dyn.cu: closed-form candidate c from R25's decade structure,
then hi in {c-1, c, c+1} from two comparisons on the exact map values) is the
oracle's nearest-value rule (oracle/codemap.py dyn_code).  The kernel's
candidate uses only plain fp32 operations, replayed here in numpy float32.
This test samples the places where a wrong candidate could matter -- every
map value and midpoint +-64 ulps, every decade boundary +-4096 ulps, 2 M
random values; tests/dyn_candidate_exhaustive.py runs all 2^31 fp32 values of
[-1, 1] (output: profiles/r2/dyn_candidate_exhaustive.txt)."""
import numpy as np
import pytest

from oracle import codemap as CM
from dyn_candidate_exhaustive import cand

f32 = np.float32


def _kernel_code(y, signed):
    """The kernel's decision, replayed: candidate, clamp, 4 map values."""
    mp = CM.dynamic_map(signed)
    a = np.abs(y)
    p = cand(a, signed)
    c = np.where(y < 0, 255 - p, p) if signed else p
    c = np.clip(c, 2, 254)
    v0, v1, v2, v3 = mp[c - 2], mp[c - 1], mp[c], mp[c + 1]
    a1, a2 = v1 >= y, v2 >= y
    hi = np.where(a1, c - 1, np.where(a2, c, c + 1))
    hv = np.where(a1, v1, np.where(a2, v2, v3))
    lv = np.where(a1, v0, np.where(a2, v1, v2))
    return np.where((hv - y).astype(f32) < (y - lv).astype(f32), hi, hi - 1).astype(np.uint8)


def _samples(signed):
    mp = CM.dynamic_map(signed)
    pts = np.concatenate([mp, ((mp[1:].astype(np.float64) + mp[:-1]) / 2).astype(f32),
                          np.array([10.0 ** -k for k in range(8)], f32), np.array([0.0, 1.0], f32)])
    bits = pts.view(np.int32)
    near = (bits[:, None] + np.arange(-64, 65, dtype=np.int32)[None, :]).ravel()
    dec = np.array([10.0 ** -k for k in range(8)], f32).view(np.int32)
    near_dec = (dec[:, None] + np.arange(-4096, 4097, dtype=np.int32)[None, :]).ravel()
    rng = np.random.default_rng(0)
    rnd = np.concatenate([rng.uniform(0, 1, 10 ** 6), 10 ** rng.uniform(-12, 0, 10 ** 6)]).astype(f32)
    y = np.concatenate([np.abs(np.concatenate([near, near_dec]).view(f32)), rnd])
    y = y[np.isfinite(y) & (y >= 0) & (y <= 1)]
    if signed:
        y = np.concatenate([y, -y])
    return y.astype(f32)


@pytest.mark.parametrize("signed", [True, False])
def test_branch_free_decision_equals_oracle(signed):
    y = _samples(signed)
    assert np.array_equal(_kernel_code(y, signed), CM.dyn_code(y, signed))
