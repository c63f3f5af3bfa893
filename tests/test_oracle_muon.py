"""Pins of the distributed-Muon oracle (oracle/muon.py, PAPER.md
Algorithm 2; readings R21-R24): the SVD closed form of Newton-Schulz
(numpy.linalg.svd), transpose equivariance, the momentum closed form, LPT
root selection against brute force and Graham's bound, and the sharded step
against Muon applied to each logical matrix."""
import numpy as np
import pytest

from oracle import muon as MU
from oracle import planner as OP


def _phi5(s, steps=5):
    a, b, c = MU.NS_COEFFS
    for _ in range(steps):
        s = a * s + b * s ** 3 + c * s ** 5
    return s


@pytest.mark.parametrize("shape", [(48, 80), (80, 48), (64, 64), (1, 33), (130, 7)])
def test_newton_schulz_svd_closed_form(shape):
    rng = np.random.default_rng(sum(shape))
    G = rng.normal(size=shape)
    U, s, Vt = np.linalg.svd(G, full_matrices=False)
    s0 = s / (np.linalg.norm(G) + 1e-7)
    exp = (U * _phi5(s0)) @ Vt
    got = MU.newton_schulz(G)
    assert np.allclose(got, exp, rtol=0, atol=1e-10 * max(1.0, np.abs(exp).max()))
    # the iteration pushes singular values toward ~1 (0.68..1.2 band of Muon)
    sv = np.linalg.svd(got, compute_uv=False)
    assert sv.max() < 1.25


def test_newton_schulz_transpose_and_scale_invariance():
    rng = np.random.default_rng(1)
    G = rng.normal(size=(40, 96))
    assert np.array_equal(MU.newton_schulz(G.T), MU.newton_schulz(G).T)
    # scale invariance up to eps: NS(c G) ~= NS(G)
    assert np.allclose(MU.newton_schulz(1e3 * G), MU.newton_schulz(G), atol=1e-8)
    # orthogonal input: NS(Q) = phi^5(1/sqrt(n)) Q
    Q, _ = np.linalg.qr(rng.normal(size=(32, 32)))
    s0 = 1.0 / (np.sqrt(32) + 1e-7)
    assert np.allclose(MU.newton_schulz(Q), _phi5(s0) * Q, atol=1e-12)


def test_momentum_closed_form():
    mu = 0.95
    g = np.array([1.0, -2.0, 0.5])
    buf = np.zeros(3)
    for k in range(1, 8):
        buf, u = MU.momentum_update(buf, g, mu)
        assert np.allclose(buf, g * (1 - mu ** k) / (1 - mu), rtol=1e-14)
        assert np.allclose(u, g + mu * g * (1 - mu ** k) / (1 - mu), rtol=1e-14)


def test_select_roots_lpt_bound_and_rules():
    rng = np.random.default_rng(2)
    for _ in range(200):
        m = int(rng.integers(2, 4))
        n = int(rng.integers(1, 7))
        shapes = [(int(rng.integers(1, 9)) * 4, int(rng.integers(1, 9)) * 4) for _ in range(n)]
        es = [r * c for r, c in shapes]
        lay = OP.plan(es, [1] * n, m, 1)
        roots = MU.select_roots(lay, shapes)
        costs = [MU.ns_cost(*s) for s in shapes]
        load = [0] * m
        for c, r in zip(costs, roots):
            load[r] += c
        opt = MU.brute_force_makespan(costs, m)
        assert max(load) <= (4 / 3 - 1 / (3 * m)) * opt + 1e-9
        # greedy balance (SPEC S:428 invariant): spread <= the largest single cost
        assert max(load) - min(load) <= max(costs)
    # rules: biggest first; ties in load -> the rank owning most of the matrix
    shapes = [(4, 4), (8, 8), None]
    lay = OP.plan([16, 64, 3], [1, 1, 1], 2, 1)  # S = 42: (8,8) spans ranks 0 (26) and 1 (38)
    roots = MU.select_roots(lay, shapes)
    assert roots[2] == -1
    assert roots[1] == 1 and roots[0] == 0


@pytest.mark.parametrize("m", [1, 2, 3])
def test_sharded_step_equals_per_matrix_muon(m):
    shapes = [(24, 40), None, (40, 24), (16, 16), None]
    es = [24 * 40, 77, 40 * 24, 256, 5]
    lay = OP.plan(es, [1] * len(es), m, 4)  # element granularity: matrices straddle ranks
    rng = np.random.default_rng(m)
    logical = [[rng.normal(size=e) for e in es] for _ in range(3)]  # master, buf, grad
    bufs = []
    for arrs in logical:
        full = np.zeros(m * lay.S)
        for x, l in zip(arrs, lay.starts):
            full[l:l + x.size] = x
        bufs.append(full)
    cfg = MU.MuonCfg()
    master, buf, roots, o_full = MU.muon_step_sharded(lay, shapes, *bufs, cfg)
    for t, (l, e) in enumerate(zip(lay.starts, es)):
        w0, b0, g = (logical[i][t] for i in range(3))
        if shapes[t] is None:
            assert np.array_equal(master[l:l + e], w0) and np.array_equal(buf[l:l + e], b0)
            continue
        r, c = shapes[t]
        b1 = 0.95 * b0 + g
        u = g + 0.95 * b1
        o = MU.newton_schulz(u.reshape(r, c)).reshape(-1)
        assert np.allclose(buf[l:l + e], b1, rtol=0, atol=1e-15)
        assert np.allclose(master[l:l + e], w0 - 0.02 * np.sqrt(max(1, r / c)) * o, atol=1e-14)
        assert roots[t] in range(m)


@pytest.mark.parametrize("shape", [(96, 24), (24, 96), (64, 64), (200, 40)])
def test_shape_scale_makes_update_rms_about_one_over_sqrt_cols(shape):
    """R23's sqrt(max(1, rows/cols)) is Muon's scale: NS output has singular
    values in Muon's ~[0.68, 1.13] band, so its RMS is about
    1/sqrt(max(rows, cols)), and the scaled update's RMS * sqrt(cols) lands in
    that band for both orientations (a transposed ratio would put tall
    matrices at sqrt(cols/rows) < 0.68)."""
    rng = np.random.default_rng(sum(shape))
    G = rng.normal(size=shape)
    o = MU.newton_schulz(G)
    r, c = shape
    rms = np.sqrt(np.mean((MU.shape_scale(r, c) * o) ** 2)) * np.sqrt(c)
    assert 0.6 < rms < 1.2
