"""Pins of the dynamic (tree) code map oracle (oracle/codemap.py, SURVEY N2,
reading R25): the map's structure, Dettmers' published construction
re-evaluated in float32 torch, brute-force nearest quantization, grid round
trips, the error bound, and the codec inside the 8-bit Adam step."""
import numpy as np
import pytest
import torch

from oracle import adam8 as OA
from oracle import codemap as CM

f32 = np.float32


@pytest.mark.parametrize("signed", [True, False])
def test_map_structure(signed):
    mp = CM.dynamic_map(signed)
    assert mp.dtype == np.float32 and mp.size == 256
    assert np.all(np.diff(mp.astype(np.float64)) > 0)          # distinct, ascending
    assert 0.0 in mp and 1.0 in mp and mp.max() == 1.0
    for i, D in enumerate(CM.DECADES):
        pos = np.sum((mp > 0.1 * D) & (mp < D))
        assert pos == (2 ** i if signed else 2 ** (i + 1))
        if signed:
            assert np.sum((mp < -0.1 * D) & (mp > -D)) == 2 ** i
    if signed:
        neg = -mp[mp < 0][::-1]
        pos = mp[(mp > 0) & (mp < 1)]
        assert np.array_equal(neg, pos)
        assert CM.zero_code(True) == 127
    else:
        assert mp.min() == 0.0 and CM.zero_code(False) == 0


@pytest.mark.parametrize("signed", [True, False])
def test_map_matches_published_construction(signed):
    """Dettmers' construction (linspace(0.1, 1, n) boundaries, midpoints,
    scaled by 10^(i-6)) evaluated in float32 torch: the same values up to
    float32 rounding of the intermediate steps."""
    data = []
    for i in range(7):
        n = 2 ** i + 1 if signed else 2 ** (i + 1) + 1
        b = torch.linspace(0.1, 1, n, dtype=torch.float32)
        means = (b[:-1] + b[1:]) / 2.0
        data += ((10 ** (-6 + i)) * means).tolist()
        if signed:
            data += (-(10 ** (-6 + i)) * means).tolist()
    data += [0.0, 1.0]
    ref = np.array(sorted(data), dtype=np.float64)
    mp = CM.dynamic_map(signed).astype(np.float64)
    assert np.all(np.abs(mp - ref) <= 4e-7 * np.abs(ref))


@pytest.mark.parametrize("signed", [True, False])
def test_code_is_nearest_value(signed):
    mp = CM.dynamic_map(signed).astype(np.float64)
    rng = np.random.default_rng(0)
    y = np.concatenate([rng.uniform(-1 if signed else 0, 1, 20000),
                        10.0 ** rng.uniform(-8, 0, 20000) * (np.where(rng.random(20000) < 0.5, -1, 1)
                                                             if signed else 1)]).astype(f32)
    c = CM.dyn_code(y, signed)
    d = np.abs(y.astype(np.float64)[:, None] - mp[None, :])
    best = d.min(axis=1)
    got = d[np.arange(y.size), c]
    assert np.all(got <= best + 1e-7 * np.abs(y) + 1e-12)
    # grid values round-trip exactly; A = 0 -> the zero code
    assert np.array_equal(CM.dyn_code(CM.dynamic_map(signed), signed), np.arange(256))
    q, a = CM.dyn_quantize(np.zeros(7, f32), signed)
    assert a == 0 and np.all(q == CM.zero_code(signed))
    assert np.all(CM.dyn_dequantize(q, a, signed) == 0)


def test_quantization_error_bound():
    """|x - deq(q(x))| <= A * (half the local gap of the map) (+ fp32 slack)."""
    rng = np.random.default_rng(1)
    for signed in (True, False):
        mp = CM.dynamic_map(signed).astype(np.float64)
        x = rng.normal(0, 1e-3, 2048).astype(f32)
        if not signed:
            x = np.abs(x)
        q, a = CM.dyn_quantize(x, signed)
        y = x.astype(np.float64) / float(a)
        hi = np.clip(np.searchsorted(mp, y), 1, 255)
        gap = mp[hi] - mp[hi - 1]
        err = np.abs(x - CM.dyn_dequantize(q, a, signed)).astype(np.float64)
        assert np.all(err <= float(a) * (gap / 2 + 1e-6) + 1e-12)


def test_dynamic_codec_in_adam_step():
    """Step 1 from the zero state: both codecs dequantize to exact zeros, so
    the master update is identical bit for bit and equals the closed form
    p0 c_wd - lr g / (|g| + eps); the stored codes are the dynamic codes of
    the fresh moments."""
    rng = np.random.default_rng(2)
    n = 2048 + 300
    p0 = rng.normal(0, 0.02, n).astype(f32)
    g = rng.normal(0, 1e-3, n).astype(f32)
    blocks = [(0, 2048), (2048, 300)]
    cfg = OA.AdamCfg()
    lin = OA.step_8bit_adam(p0, g, np.zeros(n, np.int8), np.zeros(n, np.uint8), np.zeros(2, f32),
                            np.zeros(2, f32), blocks, cfg, 1)
    dyn = OA.step_8bit_adam(p0, g, np.full(n, CM.zero_code(True), np.uint8),
                            np.full(n, CM.zero_code(False), np.uint8), np.zeros(2, f32),
                            np.zeros(2, f32), blocks, cfg, 1, codec="dynamic")
    assert np.array_equal(lin[0], dyn[0])
    closed = p0.astype(np.float64) * (1 - 1e-5) - 1e-3 * g / (np.abs(g) + 1e-8)
    assert np.allclose(dyn[0], closed, rtol=0, atol=1e-6)
    m1 = (f32(1.0 - 0.9) * g).astype(f32)  # m = 0 + w1 (g - 0), w1 = fl(1 - beta1)
    for (off, ln), k in zip(blocks, range(2)):
        q, a = CM.dyn_quantize(m1[off:off + ln], True)
        assert np.array_equal(dyn[1][off:off + ln], q) and dyn[3][k] == a


def test_dynamic_codec_total_at_tiny_and_non_finite_absmax():
    """R27 for the dynamic map: a subnormal absmax still gives the nearest
    code of the exactly-rounded y = fl(x / A) (brute force over the map);
    A NaN / +inf gives the code of 0 everywhere and keeps A."""
    for signed in (True, False):
        mp = CM.dynamic_map(signed).astype(np.float64)
        for a in (np.float32(1e-45), np.float32(1e-41), np.float32(3e-39), np.float32(1e-37)):
            x = np.float32([a, a / 3, a / 7, 0.0, a / 1000])
            if signed:
                x = np.concatenate([x, -x])
            q, aa = CM.dyn_quantize(x, signed)
            assert aa == a
            y = (x / a).astype(np.float32).astype(np.float64)
            for yi, qi in zip(y, q):
                d = np.abs(mp - yi)
                assert d[qi] == d.min()
        for bad in (np.nan, np.inf):
            q, aa = CM.dyn_quantize(np.float32([0.5, bad, 0.0]), signed)
            assert np.all(q == CM.zero_code(signed))
            assert (np.isnan(aa) and np.isnan(bad)) or aa == bad
