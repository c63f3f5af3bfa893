"""Pins for oracle/dbuffer.py: AllGather o shard = identity (bit exact), views
alias the buffer, ReduceScatter = per-rank sum (exact integer closed
form on dyadic inputs), fp32 error bound vs the exact sum, bf16 once-rounding
vs exact rational rounding and vs torch's bf16 cast (library routine)."""
import random
from fractions import Fraction

import numpy as np
import torch

from oracle import dbuffer as D
from oracle import planner as P
from synth import hashgen as H


def _rand_layout(rng, m=None):
    n = rng.randint(1, 8)
    es = [rng.randint(1, 400) for _ in range(n)]
    gs = [min(rng.choice([1, 16, 64]), e) for e in es]
    m = m or rng.randint(1, 8)
    return P.plan(es, gs, m, rng.choice([4, 8]))


def test_allgather_of_shards_is_identity_and_views_alias():
    rng = random.Random(0)
    for _ in range(200):
        lay = _rand_layout(rng)
        flat = H.params_np(rng.randint(0, 99), 0, lay.E)
        buf = D.place_logical(lay, flat)
        shards = [D.shard(lay, buf, k).copy() for k in range(lay.m)]
        g = D.all_gather(shards)
        assert np.array_equal(g.view(np.uint32), buf.view(np.uint32))
        vs = D.views(lay, g)
        assert np.array_equal(np.concatenate(vs), flat)
        # aliasing: a write through a view is visible in the buffer
        if vs:
            vs[0][0] = 7.0
            assert g[lay.starts[0]] == 7.0
        # padding is never covered by a view
        for a, b in lay.padding_intervals():
            assert np.all(g[a:b] == 0)


def test_grouped_cast_scale_exact_and_padding_zero():
    rng = random.Random(1)
    for _ in range(50):
        lay = _rand_layout(rng)
        flat = H.grads_np(0, 1, 0, lay.E)
        buf = D.place_logical(lay, flat, fill=np.nan)          # garbage padding
        bf = D.to_bf16_rne(buf)
        out = D.grouped_cast_scale(lay, bf, src_is_bf16=True)
        assert out.dtype == np.float32
        exp = D.place_logical(lay, flat) / lay.m               # dyadic -> exact when m | 2^k
        if lay.m in (1, 2, 4, 8):
            assert np.array_equal(out, exp.astype(np.float32))
        assert np.all(np.isfinite(out))


def test_reduce_scatter_is_rank_sum_exact_closed_form():
    """Dyadic inputs k * 2^-14 with |k| < 2^13: every partial sum of <= 8 terms
    (after * 1/m) is exact in fp32, so RS equals the integer sum exactly."""
    rng = random.Random(2)
    for _ in range(40):
        lay = _rand_layout(rng, m=rng.choice([1, 2, 4, 8]))
        grads = [D.place_logical(lay, H.grads_np(3, r, 0, lay.E)) for r in range(lay.m)]
        scaled = [D.grouped_cast_scale(lay, g, src_is_bf16=False) for g in grads]
        ys = D.reduce_scatter(lay, scaled)
        ints = [np.rint(g * 2.0 ** 14).astype(np.int64) for g in grads]
        tot = sum(ints)
        for k in range(lay.m):
            exact = tot[k * lay.S:(k + 1) * lay.S].astype(np.float64) * 2.0 ** -14 / lay.m
            assert np.array_equal(ys[k].astype(np.float64), exact)


def test_reduce_scatter_error_bound_random_normal():
    rng = np.random.default_rng(3)
    for m in (2, 3, 5, 8):
        lay = P.plan([3000, 1234], [1, 1], m, 4)
        xs = [rng.normal(0, 1e-2, m * lay.S).astype(np.float32) for _ in range(m)]
        ys = D.reduce_scatter(lay, xs)
        ref = D.reduce_scatter_f64(lay, xs)
        for k in range(m):
            absum = sum(np.abs(x[k * lay.S:(k + 1) * lay.S].astype(np.float64)) for x in xs)
            err = np.abs(ys[k] - ref[k])
            assert np.all(err <= (m - 1) * 2.0 ** -24 * absum + 1e-45)


def _exact_bf16_rne(x: Fraction) -> float:
    """Nearest bf16 to an exact rational (ties to even), by enumeration."""
    if x == 0:
        return 0.0
    s = -1 if x < 0 else 1
    a = abs(x)
    e = 0
    while a >= 2:
        a /= 2
        e += 1
    while a < 1:
        a *= 2
        e -= 1
    # a in [1, 2): 7 fraction bits
    scaled = a * 128
    lo = int(scaled)
    frac = scaled - lo
    if frac > Fraction(1, 2) or (frac == Fraction(1, 2) and lo % 2 == 1):
        lo += 1
    return s * lo / 128 * 2.0 ** e


def test_bf16_once_rounding():
    rng = np.random.default_rng(4)
    x = rng.normal(0, 1, 4000) * np.exp2(rng.integers(-20, 20, 4000))
    # add exact halfway cases and near-halfway cases in fp64
    base = rng.integers(128, 256, 200) * 2.0 ** -7
    x = np.concatenate([x, base + 2.0 ** -8, base + 2.0 ** -8 + 2.0 ** -40,
                        base + 2.0 ** -8 - 2.0 ** -40])
    got = D.bf16_to_f32(D.f64_to_bf16_rne(x)).astype(np.float64)
    exp = np.array([_exact_bf16_rne(Fraction(float(v))) for v in x])
    assert np.array_equal(got, exp)
    # fp32 -> bf16 matches torch's conversion (RNE)
    y = rng.normal(0, 1, 10000).astype(np.float32)
    t = torch.from_numpy(y).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(D.to_bf16_rne(y), t)


def test_reduce_scatter_bf16_mode_once_rounded():
    rng = np.random.default_rng(5)
    m = 4
    lay = P.plan([4096], [1], m, 8)
    gs = [D.to_bf16_rne(rng.normal(0, 1e-2, m * lay.S).astype(np.float32)) for _ in range(m)]
    ys = D.reduce_scatter_bf16(lay, gs)
    for k in range(m):
        tot = sum(D.bf16_to_f32(g[k * lay.S:(k + 1) * lay.S]).astype(np.float64) for g in gs) / m
        for i in range(0, lay.S, 97):
            assert D.bf16_to_f32(ys[k][i:i + 1])[0] == _exact_bf16_rne(Fraction(float(tot[i])))
