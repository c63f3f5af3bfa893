"""Pins of the FP8 (E4M3) block-quantization oracle (oracle/fp8.py, SURVEY N2,
DESIGN.md R18-R20) against things other than itself: the format's landmark
values, torch's float8_e4m3fn (library routine), brute-force nearest search,
error bounds, grid round trips and per-tensor (unsharded) quantization."""
import numpy as np
import pytest
import torch

from oracle import fp8 as F
from oracle import planner as OP

f32 = np.float32


def test_landmarks():
    v = F.e4m3_value
    assert v(0x7E) == 448.0 and v(0xFE) == -448.0  # largest finite
    assert v(0x38) == 1.0 and v(0x39) == 1.125     # exponent bias 7, 3 mantissa bits
    assert v(0x08) == 2.0 ** -6                    # smallest normal
    assert v(0x01) == 2.0 ** -9                    # smallest subnormal
    assert v(0x07) == 7 * 2.0 ** -9                # largest subnormal
    assert np.isnan(v(0x7F)) and np.isnan(v(0xFF))  # the only NaNs, no infinities
    assert v(0x00) == 0.0 and np.signbit(v(0x80))
    t = F.e4m3_table()
    assert np.sum(np.isnan(t)) == 2
    pos = t[:0x7F]
    assert np.all(np.diff(pos) > 0)                # codes are monotone in value


def test_table_matches_torch():
    codes = torch.arange(256, dtype=torch.uint8)
    ref = codes.view(torch.float8_e4m3fn).float().numpy()
    t = F.e4m3_table()
    nan = np.isnan(ref)
    assert np.array_equal(nan, np.isnan(t))
    assert np.array_equal(ref[~nan].view(np.uint32), t[~nan].view(np.uint32))


def _torch_encode(x):
    return torch.from_numpy(np.asarray(x, f32)).to(torch.float8_e4m3fn).view(torch.uint8).numpy()


def test_encode_matches_torch_grid_midpoints_random():
    t = F.e4m3_table()
    fin = t[~np.isnan(t)]
    pos = np.sort(t[:0x7F].astype(np.float64))
    mids = ((pos[1:] + pos[:-1]) / 2).astype(f32)  # exact ties (fp32-representable)
    assert np.all(mids.astype(np.float64) == (pos[1:] + pos[:-1]) / 2)
    near = np.concatenate([np.nextafter(mids, f32(0)), np.nextafter(mids, f32(1e9))])
    rng = np.random.default_rng(0)
    rnd = np.concatenate([rng.normal(0, 30, 20000), rng.normal(0, 0.01, 20000),
                          rng.uniform(-448, 448, 20000)]).astype(f32)
    for x in (fin, mids, -mids, near, -near, rnd):
        x = x[np.abs(x) <= 448]
        assert np.array_equal(F.e4m3_encode(x), _torch_encode(x))


def test_encode_brute_force_nearest_and_saturation():
    t = F.e4m3_table().astype(np.float64)
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.uniform(-460, 460, 3000), rng.normal(0, 0.02, 3000)]).astype(f32)
    c = F.e4m3_encode(x)
    fin = ~np.isnan(t)
    for xi, ci in zip(x.astype(np.float64), c):
        d = np.abs(t[fin] - xi)
        assert abs(t[ci] - xi) == d.min()
        assert np.sign(t[ci]) in (0, np.sign(xi)) and (ci >= 0x80) == (xi < 0)
    big = np.array([449, 464, 480, 1e6, np.inf, -1e6, -np.inf], f32)
    assert list(F.e4m3_encode(big)) == [0x7E] * 5 + [0xFE] * 2
    assert F.e4m3_encode(np.array([np.nan], f32))[0] == 0x7F
    assert list(F.e4m3_encode(np.array([0.0, -0.0], f32))) == [0x00, 0x80]


def test_quantize_tile_properties():
    rng = np.random.default_rng(2)
    x = rng.normal(0, 0.02, (128, 128)).astype(f32)
    x[5, 7] = -0.3
    q, s = F.quantize_tile(x)
    assert q[5, 7] == 0xFE                                   # -A maps to -448
    assert s == f32(f32(0.3) / f32(448))
    inv = f32(f32(448) / f32(0.3))
    y = (x * inv).astype(f32).astype(np.float64)
    err = np.abs(y - F.e4m3_decode(q).astype(np.float64))
    assert np.all(err <= 2.0 ** -4 * np.abs(y) + 2.0 ** -10)
    z, sz = F.quantize_tile(np.zeros((128, 64), f32))
    assert sz == 0 and not z.any()


def test_grid_round_trip():
    """Values that are decode(code) * scale for a tile whose max is +-448*scale
    come back as the same codes."""
    rng = np.random.default_rng(3)
    t = F.e4m3_table()
    for scale in (f32(1e-4), f32(0.5), f32(3.0)):
        codes = rng.integers(0, 0x7F, (64, 96)).astype(np.uint8)
        codes = np.where(rng.random(codes.shape) < 0.5, codes | 0x80, codes).astype(np.uint8)
        codes[0, 0] = 0x7E
        x = (t[codes].astype(np.float64) * float(scale)).astype(f32)
        q, s = F.quantize_tile(x)
        same = (q == codes) | ((q & 0x7F) == 0) & ((codes & 0x7F) == 0)  # +-0 either sign
        assert np.all(same)


@pytest.mark.parametrize("m", [1, 2, 3])
def test_sharded_equals_unsharded(m):
    """Containment: with 128-row granularity every tile lies on
    one rank, so quantizing rank shards and gathering == quantizing each
    logical tensor's tiles directly (cut by an independent numpy reshape)."""
    shapes = [(256, 384), (512, 128), (128, 200), (130, 128), (384, 64)]
    es = [r * c for r, c in shapes]
    gs = [min(128, r) * c for r, c in shapes]
    lay = OP.plan(es, gs, m, OP.gcoll_elems(1))
    specs = F.tile_specs([c for _, c in shapes])
    rng = np.random.default_rng(4)
    logical = [rng.normal(0, 0.02, s).astype(f32) for s in shapes]
    full = np.zeros(m * lay.S, f32)
    for x, l in zip(logical, lay.starts):
        full[l:l + x.size] = x.ravel()
    codes, scales = F.quantize_all_gather(lay, full, specs)
    exp_codes = np.zeros(m * lay.S, np.uint8)
    exp_scales = []
    for x, l in zip(logical, lay.starts):
        R, C = x.shape
        qt = np.zeros(x.shape, np.uint8)
        for i in range(0, R, 128):
            for j in range(0, C, 128):
                q, s = F.quantize_tile(x[i:i + 128, j:j + 128])
                qt[i:i + 128, j:j + 128] = q
                exp_scales.append(s)
        exp_codes[l:l + x.size] = qt.ravel()
    assert np.array_equal(codes, exp_codes)
    assert np.array_equal(scales.view(np.uint32), np.array(exp_scales, f32).view(np.uint32))
    # slot bases: rank r's tiles are the contiguous run [slot_base(r), slot_base(r+1))
    bases = [F.slot_base(lay, r, specs) for r in range(m + 1)]
    assert bases[0] == 0 and bases[m] == len(exp_scales)
    assert all(bases[r] <= bases[r + 1] for r in range(m))


def test_quantize_tile_total_at_tiny_and_non_finite_absmax():
    """R28: for A < 448 / FLT_MAX, fl(448 / A) overflows; inv is clamped to
    FLT_MAX so every code is still the E4M3 code of the finite fl(x * inv)
    (no NaN code for zeros, no saturation of non-maximal values); the
    codes equal torch's float8_e4m3fn cast of x * FLT_MAX (library routine).
    A NaN / infinite weight poisons the tile (NaN codes, scale = A)."""
    fmax = np.finfo(np.float32).max
    for a in (np.float32(1e-38), np.float32(1e-40), np.float32(1.2e-36)):
        x = np.float32([a, -a, a / 3, 0.0, -a / 5]).reshape(1, 5)
        q, sc = F.quantize_tile(x)
        assert sc == np.float32(a / np.float32(448))
        y = (x * np.float32(fmax)).astype(np.float32)
        ref = torch.from_numpy(y).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
        assert np.array_equal(q, ref)
        assert not np.any((q & 0x7F) == 0x7F)
    for bad in (np.nan, np.inf, -np.inf):
        q, sc = F.quantize_tile(np.float32([[1.0, bad, 0.0]]))
        assert np.all(q == 0x7F) and not np.isfinite(sc)
