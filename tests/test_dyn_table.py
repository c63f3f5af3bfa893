"""The dynamic codec's code decision (N2, reading R25) as the kernels take
it: a lookup in the tables rsdb_dynamic_code_tables exports (one entry per
sign / exponent / top-mantissa-bits bin, one comparison), replayed on the
host against the oracle's nearest-map-value rule (oracle/codemap.py
dyn_code) on every map value and midpoint and their 64 neighbouring floats,
the decade limits 1e-k with 4096 neighbours, the bin edges, and random
values; tests/dyn_table_exhaustive.py runs all 2^31 fp32 values of [-1, 1]
(output: profiles/r2/dyn_table_exhaustive.txt).  The GPU tests check the
kernel's codes against the oracle end to end."""
import numpy as np
import pytest

import paper_2602_22437_b200 as R
from oracle import codemap as CM

from dyn_table_exhaustive import table_code

f32 = np.float32


def _samples(signed):
    mp = CM.dynamic_map(signed)
    pts = np.concatenate([mp, ((mp[1:].astype(np.float64) + mp[:-1]) / 2).astype(f32),
                          np.array([10.0 ** -k for k in range(8)], f32), np.array([0.0, 1.0], f32)])
    bits = np.abs(pts).view(np.int32)
    near = (bits[:, None] + np.arange(-64, 65, dtype=np.int32)[None, :]).ravel()
    dec = np.array([10.0 ** -k for k in range(8)], f32).view(np.int32)
    near_dec = (dec[:, None] + np.arange(-4096, 4097, dtype=np.int32)[None, :]).ravel()
    mb = 6 if signed else 7
    edges = (np.arange(100 << mb, (128 << mb) + 1, dtype=np.int64) << (23 - mb)).astype(np.int32)
    near_edge = (edges[:, None] + np.arange(-2, 3, dtype=np.int32)[None, :]).ravel()
    rng = np.random.default_rng(0)
    rnd = np.concatenate([rng.uniform(0, 1, 10 ** 6), 10 ** rng.uniform(-12, 0, 10 ** 6)]).astype(f32)
    y = np.concatenate([np.concatenate([near, near_dec, near_edge]).view(f32), rnd,
                        np.array([0.0, 1e-30, 2.0 ** -27, 2.0 ** -126], f32)])
    y = y[np.isfinite(y) & (y >= 0) & (y <= 1)]
    if signed:
        y = np.concatenate([y, -y])
    return y.astype(f32)


@pytest.fixture(scope="module")
def tables():
    tm, tv = R.dynamic_code_tables()
    return np.array(tm, np.uint32), np.array(tv, np.uint32)


@pytest.mark.parametrize("signed", [True, False])
def test_table_decision_equals_oracle(tables, signed):
    y = _samples(signed)
    got = table_code(tables[0] if signed else tables[1], y, signed)
    assert np.array_equal(got, CM.dyn_code(y, signed))


def test_table_shape(tables):
    """Codes in range, every step of the rule appears once, negative zero
    decides like zero."""
    tm, tv = tables
    assert len(tm) == R._capi.RSDB_DYN_TABLE_M_LEN and len(tv) == R._capi.RSDB_DYN_TABLE_V_LEN
    for tab, signed in ((tm, True), (tv, False)):
        y = np.array([0.0, -0.0], f32)
        assert table_code(tab, y, signed)[0] == table_code(tab, y, signed)[1] == CM.zero_code(signed)
        assert table_code(tab, np.array([1.0], f32), signed)[0] == 255
