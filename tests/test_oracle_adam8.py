"""Pins for oracle/adam8.py: step-1 closed form (bias corrections cancel),
identity-codec variant = torch.optim.AdamW (library routine), codec round
trip / bound / zero block, and containment: the sharded
step equals the unsharded step bit for bit."""
import numpy as np
import pytest
import torch

from oracle import adam8 as A
from oracle import dbuffer as D
from oracle import planner as P
from synth import hashgen as H


def _zero_state(S, nb):
    return (np.zeros(S, np.int8), np.zeros(S, np.uint8),
            np.zeros(nb, np.float32), np.zeros(nb, np.float32))


def test_step1_closed_form():
    """From the zero state: p1 = p0 (1 - lr wd) - lr g / (|g| + eps)."""
    cfg = A.AdamCfg()
    S = 4 * 2048 + 100
    p0 = H.params_np(0, 0, S)
    g = H.grads_np(0, 0, 0, S)
    blocks = [(i * 2048, min(2048, S - i * 2048)) for i in range(-(-S // 2048))]
    mq, vq, ma, va = _zero_state(S, len(blocks))
    p1 = A.step_8bit_adam(p0, g, mq, vq, ma, va, blocks, cfg, 1)[0]
    exp = p0.astype(np.float64) * (1 - cfg.lr * cfg.weight_decay) \
        - cfg.lr * g.astype(np.float64) / (np.abs(g.astype(np.float64)) + cfg.eps)
    assert np.max(np.abs(p1 - exp)) < 1e-8


def test_identity_codec_matches_torch_adamw():
    """torch.optim.AdamW (single-tensor path) is the library routine the
    identity codec reduces to (R11).  Its moments are bit for bit the
    oracle's steps 3-4 (lerp_ and addcmul_ round once, R26), and its
    parameter is bit for bit the oracle's step 5-6 (mul_, then addcdiv_)
    wherever torch's CPU sqrt returns the correctly rounded root -- it does
    not on ~0.6 % of elements; there the two agree within 1e-6.  Each step
    starts from torch's parameter, so a sqrt difference does not propagate."""
    cfg = A.AdamCfg(lr=3e-3, weight_decay=0.05)
    n = 1 << 16
    rng = np.random.default_rng(0)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    tp = torch.nn.Parameter(torch.from_numpy(rng.normal(0, 0.02, n).astype(np.float32)))
    opt = torch.optim.AdamW([tp], lr=cfg.lr, betas=(cfg.beta1, cfg.beta2), eps=cfg.eps,
                            weight_decay=cfg.weight_decay, foreach=False, fused=False)
    exact = 0
    for step in range(1, 6):
        g = rng.normal(0, 1e-3, n).astype(np.float32)
        p_in = tp.detach().numpy().copy()
        p, m, v = A.step_adam_fp32_states(p_in, g, m, v, cfg, step)
        tp.grad = torch.from_numpy(g.copy())
        opt.step()
        ref = tp.detach().numpy()
        st = opt.state[tp]
        assert np.array_equal(m, st["exp_avg"].numpy())
        assert np.array_equal(v, st["exp_avg_sq"].numpy())
        ieee = np.sqrt(v) == torch.from_numpy(v).sqrt().numpy()
        assert np.array_equal(p[ieee], ref[ieee])
        assert np.max(np.abs(p - ref) / (np.abs(ref) + cfg.lr)) < 1e-6
        exact += int(ieee.sum())
    assert exact > 0.95 * 5 * n


def _fma_exact(a, b, c):
    from fractions import Fraction
    return _rn32(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


def _rn32(x):
    """The rational x rounded to fp32, nearest-even (subnormals included),
    by bracketing with nextafter."""
    from fractions import Fraction
    if abs(x) >= Fraction(2) ** 128 - Fraction(2) ** 103:  # past the overflow midpoint
        return np.float32(np.inf) if x > 0 else np.float32(-np.inf)
    r = np.float32(float(x))  # float(x) is RN64(x); fix the possible double rounding below
    lo = r if Fraction(float(r)) <= x else np.nextafter(r, np.float32(-np.inf))
    hi = np.nextafter(lo, np.float32(np.inf))
    dl, dh = x - Fraction(float(lo)), Fraction(float(hi)) - x
    if dl != dh:
        return lo if dl < dh else hi
    return lo if (lo.view(np.uint32) & 1) == 0 else hi


def test_fma32_is_the_exact_value_rounded_once():
    """fma32 against exact rational arithmetic: random triples over a wide
    exponent range (cancellation included), and a case where rounding the
    exact sum to fp64 first lands on an fp32 midpoint (double rounding)."""
    rng = np.random.default_rng(5)
    n = 4000
    a = (rng.normal(size=n) * np.exp2(rng.integers(-20, 20, n))).astype(np.float32)
    b = (rng.normal(size=n) * np.exp2(rng.integers(-20, 20, n))).astype(np.float32)
    c = np.where(rng.random(n) < 0.3, -(a * b).astype(np.float32),   # near-cancellation
                 (rng.normal(size=n) * np.exp2(rng.integers(-40, 40, n)))).astype(np.float32)
    got = A.fma32(a, b, c)
    exp = np.array([_fma_exact(x, y, z) for x, y, z in zip(a, b, c)], np.float32)
    assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))
    # exact = 1 + 2^-23 + 2^-24 - 2^-70: RN64 gives the midpoint 1 + 2^-23 + 2^-24,
    # whose tie-to-even is 1 + 2^-22; the correct RN32 is 1 + 2^-23
    a1 = np.float32(1 + 2.0 ** -23)
    b1 = np.float32(2.0 ** -24 * (1 - 2.0 ** -23))
    c1 = np.float32(1 + 2.0 ** -23)
    assert np.float32(float(a1) * float(b1) + float(c1)) == np.float32(1 + 2.0 ** -22)
    assert A.fma32(a1, b1, c1) == np.float32(1 + 2.0 ** -23) == _fma_exact(a1, b1, c1)
    # torch's CPU lerp is this fused form (R26)
    mt = rng.normal(0, 1e-3, 1 << 16).astype(np.float32)
    g = rng.normal(0, 1e-3, 1 << 16).astype(np.float32)
    w = np.float32(0.1)
    tl = torch.lerp(torch.from_numpy(mt), torch.from_numpy(g), 0.1).numpy()
    assert np.array_equal(tl, A.fma32(w, (g - mt).astype(np.float32), mt))


def test_codec_properties():
    # zero block -> zero codes, zero absmax, exact round trip
    q, a = A.quantize(np.zeros(2048, np.float32), signed=True)
    assert a == 0 and not q.any()
    assert not A.dequantize(q, a, True).any()
    # block = c * [-127..127] -> exact round trip
    c = np.float32(2.0 ** -9)
    x = (np.arange(-127, 128, dtype=np.float32) * c).astype(np.float32)
    q, a = A.quantize(x, signed=True)
    assert a == 127 * c and np.array_equal(A.dequantize(q, a, True), x)
    x = (np.arange(0, 256, dtype=np.float32) * c).astype(np.float32)
    q, a = A.quantize(x, signed=False)
    assert np.array_equal(A.dequantize(q, a, False), x)
    # |x - deq(q(x))| <= A/254 (signed), A/510 (unsigned), up to fp32 rounding:
    # the code is decided on fl(x / fl(A/L)) (O4 step 8), within L * 2^-23 code steps
    # of the exact x * L / A, so at a tie the error exceeds half a step by at most
    # that: the bound is (A / 2L) (1 + 2 L 2^-23) plus the dequantization rounding
    rng = np.random.default_rng(1)
    for _ in range(50):
        x = (rng.normal(0, 1, 2048) * np.exp2(rng.integers(-30, 5))).astype(np.float32)
        q, a = A.quantize(x, True)
        err = np.abs(x.astype(np.float64) - A.dequantize(q, a, True))
        assert np.all(err <= a / 254 * (1 + 2 * 127 * 2.0 ** -23 + 1e-6))
        q, a = A.quantize(np.abs(x), False)
        err = np.abs(np.abs(x).astype(np.float64) - A.dequantize(q, a, False))
        assert np.all(err <= a / 510 * (1 + 2 * 255 * 2.0 ** -23 + 1e-6))


def _code_exact(x, a, signed):
    """O4 step 8 in exact rational arithmetic: d = RN32(A / L), y = RN32(x / d),
    round half to even, clamp; a NaN quotient (0/0, x/NaN) -> 0 (R27)."""
    from fractions import Fraction
    L, lo, hi = (127, -127, 127) if signed else (255, 0, 255)
    if not np.isfinite(a):  # A = NaN: every quotient NaN; A = inf: x/inf = 0, inf/inf = NaN
        return 0
    d = _rn32(Fraction(float(a)) / L)
    if d == 0:
        return 0 if x == 0 else (hi if x > 0 else lo)
    y = _rn32(Fraction(float(x)) / Fraction(float(d)))
    if not np.isfinite(y):
        return hi if y > 0 else lo
    fy = Fraction(float(y))
    n = int(np.floor(float(y)))  # exact: |y| < 2^24 here or the clamp decides
    rem = fy - n
    k = n + 1 if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2) else n
    return max(lo, min(hi, k))


def test_code_is_the_exact_division_rounded_twice():
    """O4 step 8: the code is rint(RN32(x / RN32(A/L))),
    checked against exact rational arithmetic on inputs within a few ulps of
    every rounding tie k + 1/2 and over the whole exponent range of A,
    subnormal steps d included.  The reciprocal-multiply form
    rint(RN32(x * RN32(L/A))) disagrees on some of these inputs (asserted),
    so the pin tells the two apart."""
    rng = np.random.default_rng(7)
    n_diff_recip = 0
    cases = 0
    for signed in (True, False):
        L = 127 if signed else 255
        for e in list(range(-149, -120, 3)) + list(range(-120, 120, 7)):
            a = np.float32(np.ldexp(1.0 + rng.random(), e))
            if not np.isfinite(a) or a == 0:
                continue
            d = np.float32(a / np.float32(L))
            ks = rng.integers(0 if not signed else -L, L, 24)
            xs = []
            for k in ks:
                t = np.float32((k + 0.5) * float(d))
                for u in range(-3, 4):
                    xs.append(t)
                    t = np.nextafter(t, np.float32(np.inf))
            x = np.array([v for v in xs if abs(v) <= a], np.float32)
            x = np.concatenate([x, np.float32([a, -a if signed else 0, 0])])
            if not signed:
                x = np.abs(x)
            blk = np.concatenate([x, np.float32([a])])  # pin the block's absmax to a
            q, aa = A.quantize(blk, signed)
            assert aa == a
            exp = [_code_exact(v, a, signed) for v in blk]
            assert q.astype(int).tolist() == exp, (signed, e)
            with np.errstate(all="ignore"):
                rq = np.clip(np.rint((blk * np.float32(np.float32(L) / a)).astype(np.float32)),
                             -L if signed else 0, L)
            n_diff_recip += int(np.sum(np.isfinite(rq) & (rq != np.array(exp))))
            cases += blk.size
    assert cases > 5000 and n_diff_recip > 0


def test_codec_total_at_tiny_and_non_finite_absmax():
    """R27: the codec is defined for every block.  Tiny absmax (d = A/L
    subnormal, or underflowing to 0 -- the regime a block with a long run of
    zero gradients reaches, m decaying x0.9 per step) gives in-range codes
    equal to the exact-arithmetic decision; A = 0 gives zeros; a NaN
    or infinite element gives all-zero codes and keeps A (NaN / +inf)."""
    for a in [np.float32(v) for v in (1e-45, 3e-45, 1e-44, 1e-43, 7e-42, 1e-40, 1.2e-38,
                                      3.7e-37, 7.5e-37, 1e-30, 3e38)]:
        x = np.float32([a, -a, a / 2, a / 3, -a / 7, 0, np.float32(-0.0)])
        for signed in (True, False):
            xx = x if signed else np.abs(x)
            q, aa = A.quantize(xx, signed)
            assert aa == a
            assert q.astype(int).tolist() == [_code_exact(v, a, signed) for v in xx]
            deq = A.dequantize(q, aa, signed)
            assert np.all(np.isfinite(deq))
    for bad, exp_a in ((np.nan, np.nan), (np.inf, np.inf), (-np.inf, np.inf)):
        x = np.float32([1.0, bad, -2.0, 0.0])
        for signed in (True, False):
            q, aa = A.quantize(x if signed else np.abs(x), signed)
            assert not q.any()
            assert (np.isnan(aa) and np.isnan(exp_a)) or aa == exp_a
            assert np.all(np.isnan(A.dequantize(q, aa, signed)))  # the block is poisoned


def test_zero_gradient_run_stays_in_range():
    """A block whose gradient stays 0 decays m by beta1 per step (and v by
    beta2) until A_m underflows; 900 oracle steps keep every code in range,
    A_m non-increasing, and m's dequantized value within one step of 0.9x
    the previous one -- no overflow, no NaN."""
    rng = np.random.default_rng(3)
    n = 2048
    p = rng.normal(0, 0.02, n).astype(np.float32)
    g0 = rng.normal(0, 1e-3, n).astype(np.float32)
    mq, vq, ma, va = _zero_state(n, 1)
    cfg = A.AdamCfg()
    st = A.step_8bit_adam(p, g0, mq, vq, ma, va, [(0, n)], cfg, 1)
    zero = np.zeros(n, np.float32)
    prev = st[3][0]
    for t in range(2, 902):
        st = A.step_8bit_adam(st[0], zero, st[1], st[2], st[3], st[4], [(0, n)], cfg, t)
        assert np.isfinite(st[3][0]) and np.isfinite(st[4][0])
        assert st[3][0] <= prev
        prev = st[3][0]
        assert np.all(np.isfinite(st[0]))
    assert st[3][0] < np.float32(3.7e-37)  # reached the regime where fl(127/A) overflows


@pytest.mark.parametrize("m", [2, 3, 4, 8])
def test_sharded_step_equals_unsharded(m):
    """Containment: with 2048-element blocks kept whole by the
    planner, each rank's local step equals the single-rank step exactly."""
    es = [256 * 128, 256, 5000, 2048 * 3, 77]
    q = 2048
    gs = [min(q, e) for e in es]
    cfg = A.AdamCfg()
    E = sum(es)
    p_log = H.params_np(1, 0, E)
    g_log = H.grads_np(1, 0, 0, E)
    mq_log = H.codes_np(1, H.STREAM_MCODE, 0, E, True)
    vq_log = H.codes_np(1, H.STREAM_VCODE, 0, E, False)

    def run(mm):
        lay = P.plan(es, gs, mm, 4)
        bufs = {k: D.place_logical(lay, v) for k, v in
                dict(p=p_log, g=g_log, mq=mq_log, vq=vq_log).items()}
        out = {k: np.zeros_like(v) for k, v in bufs.items() if k != "g"}
        out["bf"] = np.zeros(mm * lay.S, np.uint16)
        for r in range(mm):
            blocks = P.rank_blocks(lay, r, q)
            sl = slice(r * lay.S, (r + 1) * lay.S)
            # absmax indexed per block: derive from a per-(tensor,block) id so
            # both layouts see the same initial state
            ids = _block_ids(lay, r, q)
            ma = H.absmax_np(1, H.STREAM_ABSM, 0, 10 ** 4, 14)[ids]
            va = H.absmax_np(1, H.STREAM_ABSV, 0, 10 ** 4, 20)[ids]
            res = A.step_8bit_adam(bufs["p"][sl], bufs["g"][sl], bufs["mq"][sl], bufs["vq"][sl],
                                   ma, va, blocks, cfg, 4)
            out["p"][sl], out["mq"][sl], out["vq"][sl] = res[0], res[1], res[2]
            out["bf"][sl] = res[5]
        return lay, out

    lay1, o1 = run(1)
    layk, ok = run(m)
    for key in o1:
        v1 = np.concatenate(D.views(lay1, o1[key]))
        vk = np.concatenate(D.views(layk, ok[key]))
        assert np.array_equal(v1.view(np.uint8), vk.view(np.uint8)), key


def _block_ids(lay, rank, q):
    ids = []
    lo = rank * lay.S
    base = 0
    for l, e in zip(lay.starts, lay.numel):
        for j in range(-(-e // q)):
            a = l + j * q
            if lo <= a < lo + lay.S:
                ids.append(base + j)
        base += -(-e // q)
    return np.array(ids, dtype=np.int64)


def test_8bit_step_composes_codec_and_torch_pinned_update():
    """The 8-bit step = dequantize (pinned by the codec tests) -> the fp32
    update (pinned to torch AdamW) -> quantize, block by block: catches wiring
    mistakes (swapped m/v absmax, wrong block index, wrong signedness)."""
    cfg = A.AdamCfg()
    S, q = 5 * 2048 + 300, 2048
    blocks = [(i * q, min(q, S - i * q)) for i in range(-(-S // q))]
    p0 = H.params_np(5, 0, S)
    g = H.grads_np(5, 0, 0, S)
    mq = H.codes_np(5, H.STREAM_MCODE, 0, S, True)
    vq = H.codes_np(5, H.STREAM_VCODE, 0, S, False)
    ma = H.absmax_np(5, H.STREAM_ABSM, 0, len(blocks), 12)
    va = H.absmax_np(5, H.STREAM_ABSV, 0, len(blocks), 22)
    out = A.step_8bit_adam(p0, g, mq, vq, ma, va, blocks, cfg, 7)
    for b, (off, n) in enumerate(blocks):
        s = slice(off, off + n)
        mt = A.dequantize(mq[s], ma[b], True)
        vt = A.dequantize(vq[s], va[b], False)
        p, m, v = A.step_adam_fp32_states(p0[s], g[s], mt, vt, cfg, 7)
        assert np.array_equal(out[0][s], p)
        qm, am = A.quantize(m, True)
        qv, av = A.quantize(v, False)
        assert np.array_equal(out[1][s], qm) and out[3][b] == am
        assert np.array_equal(out[2][s], qv) and out[4][b] == av


def test_bf16_output_is_rne_of_master():
    S = 2048
    p0 = H.params_np(2, 0, S)
    g = H.grads_np(2, 0, 0, S)
    mq, vq, ma, va = _zero_state(S, 1)
    res = A.step_8bit_adam(p0, g, mq, vq, ma, va, [(0, S)], A.AdamCfg(), 1)
    t = torch.from_numpy(res[0]).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(res[5], t)


# ----------------------------------------------------------------- N2: 2-D tiles
def _tile_layout(m, tr=32):
    # two matrices [96, 64] and [64, 40] + a vector, 32-row sharding granularity
    shapes = [(96, 64), (64, 40), (130,)]
    es = [int(np.prod(s)) for s in shapes]
    gs = [tr * 64, tr * 40, 1]
    return shapes, P.plan(es, gs, m, 4)


def test_tiles_with_one_row_are_flat_blocks():
    shapes, lay = _tile_layout(3)
    for r in range(3):
        specs = [("tile", s[-1], 1, s[-1]) if len(s) == 2 else ("flat", 130) for s in shapes]
        t = P.rank_tiles(lay, r, specs)
        fl = P.rank_tiles(lay, r, [("flat", s[-1]) if len(s) == 2 else ("flat", 130) for s in shapes])
        assert t == fl


def test_tiles_partition_every_tensor():
    for m in (1, 2, 3, 4):
        shapes, lay = _tile_layout(m)
        specs = [("tile", 64, 32, 32), ("tile", 40, 32, 32), ("flat", 130)]
        cover = np.zeros(m * lay.S, int)
        for r in range(m):
            for off, rows, cols, pitch in P.rank_tiles(lay, r, specs):
                idx = r * lay.S + off + np.arange(rows)[:, None] * pitch + np.arange(cols)[None, :]
                cover[idx.ravel()] += 1
        exp = np.zeros(m * lay.S, int)
        for l, e in zip(lay.starts, lay.numel):
            exp[l:l + e] = 1
        assert np.array_equal(cover, exp)


def test_tile_straddle_detected():
    lay = P.plan([96 * 64], [1], 5, 4)  # element granularity: S = 1232 cuts row 19
    with pytest.raises(ValueError):
        for r in range(5):
            P.rank_tiles(lay, r, [("tile", 64, 32, 32)])


def test_tiled_step_equals_flat_step_on_each_tile():
    """Independent tile derivation: reshape [R, C] -> [R/32, 32, C/32, 32]."""
    cfg = A.AdamCfg()
    R_, C_ = 96, 64
    lay = P.plan([R_ * C_], [32 * C_], 1, 4)
    S = lay.S
    p = H.params_np(9, 0, S)
    g = H.grads_np(9, 0, 0, S)
    mq = H.codes_np(9, H.STREAM_MCODE, 0, S, True)
    vq = H.codes_np(9, H.STREAM_VCODE, 0, S, False)
    tiles = P.rank_tiles(lay, 0, [("tile", C_, 32, 32)])
    nb = len(tiles)
    ma = H.absmax_np(9, H.STREAM_ABSM, 0, nb, 12)
    va = H.absmax_np(9, H.STREAM_ABSV, 0, nb, 22)
    out = A.step_8bit_adam(p, g, mq, vq, ma, va, tiles, cfg, 3)
    idx = np.arange(R_ * C_).reshape(R_ // 32, 32, C_ // 32, 32).transpose(0, 2, 1, 3).reshape(-1, 1024)
    for b in range(nb):
        e = idx[b]
        ref = A.step_8bit_adam(p[e], g[e], mq[e], vq[e], ma[b:b + 1], va[b:b + 1], [(0, 1024)], cfg, 3)
        assert np.array_equal(out[0][e], ref[0]) and np.array_equal(out[1][e], ref[1])
        assert np.array_equal(out[2][e], ref[2]) and out[3][b] == ref[3][0] and out[4][b] == ref[4][0]
