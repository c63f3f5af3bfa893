"""-m gpu parity: the CUDA path (through the C-ABI) vs the CPU oracle, element
by element on identical seeded inputs.

Tolerances (BASELINE.json north_star, made well-defined in DESIGN.md):
  * AllGather / layouts: bit exact;
  * cast/scale group op: bit exact (one fp32 multiply by fl(1/m) both sides);
  * ReduceScatter fp32: |y - y_ref| <= 1e-6 * sum_r |x_r| (bit exact on the
    dyadic synth inputs, where every fp32 partial sum is exact);
  * 8-bit Adam: codes within +-1, params |dp| <= 1e-5 (|p_ref| + lr), absmax
    relative 1e-6, bf16 shard = RNE(GPU master) exactly and, by value, within
    the param tolerance plus one bf16 ulp of the oracle's.
"""
import numpy as np
import pytest
import torch

import paper_2602_22437_b200 as R
from oracle import adam8 as OA
from oracle import codemap as CM
from oracle import dbuffer as OD
from oracle import planner as OP
from synth import hashgen as H
from synth import workloads as W

from gpu_helpers import bf16_bits, f32, logical_grads, logical_params, place_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _plans(es, gs, m, eb):
    gc = OP.gcoll_elems(eb)
    o = OP.plan(es, gs, m, gc)
    c = R.plan(es, gs, m, elem_bytes=eb)
    assert c.starts == o.starts and c.S == o.S
    return o, c


# ------------------------------------------------------------------ synth
def test_hash_generator_on_device_matches_numpy():
    a = H.values_np(7, 17, 1000, 300000, 14, True)
    b = H.values_torch(7, 17, 1000, 300000, 14, True, device="cuda", chunk=65536).cpu().numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    c = H.codes_np(7, 64, 5, 100000, True)
    d = H.codes_torch(7, 64, 5, 100000, True, device="cuda").cpu().numpy()
    assert np.array_equal(c, d)


# ------------------------------------------------------------------ a6
CAST_CASES = [
    ([256 * 128, 256] * 6, "flat", 1, 2), ([256 * 128, 256] * 6, "flat", 2, 4),
    ([5000, 77, 4109, 2048 * 3, 1], "flat", 3, 2), ([5000, 77, 4109, 2048 * 3, 1], "elem", 8, 2),
    ([123457, 99, 7], "whole", 5, 2), ([4096 * 9 + 5], "elem", 4, 4), ([1 << 20, 3], "flat", 8, 2),
]


@pytest.mark.parametrize("es,gk,m,eb", CAST_CASES)
def test_cast_scale_bit_exact(es, gk, m, eb):
    gs = [min(2048, e) if gk == "flat" else (1 if gk == "elem" else e) for e in es]
    o, c = _plans(es, gs, m, eb)
    E = sum(es)
    g_log = logical_grads(0, 1, E)
    dt = torch.bfloat16 if eb == 2 else torch.float32
    grad_full = place_gpu(c, g_log, dt, fill=float("nan"))       # garbage padding
    grad_f32 = torch.empty(m * c.S, dtype=torch.float32, device="cuda")
    param_full = torch.zeros(m * c.S, dtype=dt, device="cuda")
    for rank in sorted({0, m - 1}):
        q = {"flat": 2048, "elem": 1, "whole": max(es)}[gk]
        u = R.Unit(c, rank, param_full, grad_full, grad_f32 if eb == 2 else grad_full, qblock=q)
        out = grad_f32 if eb == 2 else grad_full
        if eb == 4:
            grad_full.copy_(place_gpu(c, g_log, dt, fill=float("nan")))
        R.unit_cast_scale(u)
        torch.cuda.synchronize()
        src = OD.place_logical(o, g_log.numpy(), fill=np.nan)
        ref = OD.grouped_cast_scale(o, OD.to_bf16_rne(src) if eb == 2 else src, eb == 2)
        assert np.array_equal(f32(out).view(np.uint32), ref.view(np.uint32))


def test_unit_rejects_misaligned_buffers():
    """Units require 16-byte aligned buffers (NCCL alignment)."""
    es, gs, m = [3000, 5], [1, 1], 2
    o, c = _plans(es, gs, m, 4)
    E = sum(es)
    g_log = logical_grads(3, 0, E)
    base = torch.zeros(m * c.S + 4, dtype=torch.float32, device="cuda")
    src = base[1:1 + m * c.S]
    src.copy_(place_gpu(c, g_log, torch.float32))
    dst = torch.zeros(m * c.S + 4, dtype=torch.float32, device="cuda")[1:1 + m * c.S]
    pf = torch.zeros(m * c.S, dtype=torch.float32, device="cuda")
    with pytest.raises(R.RsdbError):        # units require 16-B aligned buffers
        R.Unit(c, 0, pf, src, dst, qblock=1)


# ------------------------------------------------------------------ a8
def _adam_case(es, q, m, eb, rank, step, warm, seed=0, zero_grad_tensor=None, codec="linear",
               exact_codes=True, g_log=None, state=None):
    gs = [min(q, e) for e in es]
    o, c = _plans(es, gs, m, eb)
    E = sum(es)
    S = c.S
    dt = torch.bfloat16 if eb == 2 else torch.float32
    p_log = logical_params(seed, E)
    if g_log is None:
        g_log = logical_grads(seed, rank, E)
    if zero_grad_tensor is not None:
        a = sum(es[:zero_grad_tensor])
        g_log[a:a + es[zero_grad_tensor]] = 0
    # ----- GPU side (product layout) -----
    master_full = place_gpu(c, p_log, torch.float32)
    master = master_full[rank * S:(rank + 1) * S].clone()
    grad_f32 = place_gpu(c, g_log, torch.float32)
    grad_full = torch.zeros(m * S, dtype=dt, device="cuda")
    param_full = torch.zeros(m * S, dtype=dt, device="cuda")
    u = R.Unit(c, rank, param_full, grad_full if eb == 2 else grad_f32, grad_f32, qblock=q)
    nb = u.num_blocks
    blocks_c = c.rank_blocks(rank, q)
    assert len(blocks_c) == nb
    if codec == "dynamic":  # uint8 indices into the dynamic maps (R25); zero state = code of 0
        if warm:
            mq = H.codes_torch(seed, H.STREAM_MCODE, rank * S, S, False, device="cuda")
            vq = H.codes_torch(seed, H.STREAM_VCODE, rank * S, S, False, device="cuda")
            ma = H.absmax_torch(seed, H.STREAM_ABSM, rank * 100000, nb, 14, device="cuda")
            va = H.absmax_torch(seed, H.STREAM_ABSV, rank * 100000, nb, 22, device="cuda")
        else:
            mq = torch.full((S,), CM.zero_code(True), dtype=torch.uint8, device="cuda")
            vq = torch.full((S,), CM.zero_code(False), dtype=torch.uint8, device="cuda")
            ma = torch.zeros(nb, dtype=torch.float32, device="cuda")
            va = torch.zeros(nb, dtype=torch.float32, device="cuda")
    elif state is not None:  # explicit (m codes, v codes, m absmax, v absmax) numpy arrays
        mq, vq, ma, va = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in state)
    elif warm:
        mq = H.codes_torch(seed, H.STREAM_MCODE, rank * S, S, True, device="cuda")
        vq = H.codes_torch(seed, H.STREAM_VCODE, rank * S, S, False, device="cuda")
        ma = H.absmax_torch(seed, H.STREAM_ABSM, rank * 100000, nb, 14, device="cuda")
        va = H.absmax_torch(seed, H.STREAM_ABSV, rank * 100000, nb, 22, device="cuda")
    else:
        mq = torch.zeros(S, dtype=torch.int8, device="cuda")
        vq = torch.zeros(S, dtype=torch.uint8, device="cuda")
        ma = torch.zeros(nb, dtype=torch.float32, device="cuda")
        va = torch.zeros(nb, dtype=torch.float32, device="cuda")
    ins = [t.cpu().numpy().copy() for t in (master, mq, vq, ma, va)]
    cfg = R.AdamConfig()
    (R.step_8bit_adam_dynamic if codec == "dynamic" else R.step_8bit_adam)(
        u, master, mq, vq, ma, va, cfg, step)
    torch.cuda.synchronize()
    # ----- oracle side (oracle layout) -----
    blocks_o = OP.rank_blocks(o, rank, q)
    assert [tuple(b) for b in blocks_o] == blocks_c
    g_or = OD.shard(o, OD.place_logical(o, g_log.numpy()), rank)
    ref = OA.step_8bit_adam(ins[0], g_or, ins[1], ins[2], ins[3], ins[4], blocks_o,
                            OA.AdamCfg(), step, out_bf16=(eb == 2), codec=codec)
    _check_adam(o, rank, blocks_o, (master, mq, vq, ma, va, param_full), ref, ins, eb, cfg.lr,
                exact_codes=exact_codes)
    return u


def _check_adam(o, rank, blocks, gpu, ref, ins, eb, lr, exact_codes=True):
    master, mq, vq, ma, va, param_full = gpu
    S = o.S
    mask = np.zeros(S, bool)
    for blk in blocks:
        if len(blk) == 2:
            mask[blk[0]:blk[0] + blk[1]] = True
        else:
            off, rows, cols, pitch = blk
            mask[(off + np.arange(rows)[:, None] * pitch + np.arange(cols)[None, :]).ravel()] = True
    gm = f32(master)
    # params (NaN exactly where the oracle's are: non-finite gradients, R27)
    nan = np.isnan(ref[0])
    assert np.array_equal(np.isnan(gm), nan)
    fin = mask & ~nan
    err = np.abs(gm - ref[0]) / (np.abs(ref[0]) + lr)
    assert err[fin].max(initial=0) <= 1e-5, err[fin].max()
    assert np.array_equal(gm[~mask], ins[0][~mask])  # padding untouched
    # codes: +-1 is the north_star bound; the moments (R26) and the code
    # decision (O4 step 8, R9/R27) are the same IEEE operations on both
    # sides, so the codes and absmax must be exact
    dm = np.abs(mq.cpu().numpy().astype(np.int32) - ref[1].astype(np.int32))
    dv = np.abs(vq.cpu().numpy().astype(np.int32) - ref[2].astype(np.int32))
    assert dm[mask].max(initial=0) <= 1 and dv[mask].max(initial=0) <= 1
    if exact_codes:
        assert not dm[mask].any() and not dv[mask].any(), (int(dm[mask].sum()), int(dv[mask].sum()))
    # absmax: bit exact (NaN where the oracle's is NaN)
    for a, r in ((f32(ma), ref[3]), (f32(va), ref[4])):
        a, r = a[:len(r)], r
        assert np.array_equal(np.isnan(a), np.isnan(r))
        ok = np.isfinite(r)
        assert np.array_equal(a[~ok & ~np.isnan(r)], r[~ok & ~np.isnan(r)])  # +inf
        if exact_codes:
            assert np.array_equal(a[ok].view(np.uint32), r[ok].view(np.uint32))
        assert np.all(np.abs(a[ok] - r[ok]) <= 1e-6 * np.abs(r[ok]) + 1e-30)
    # parameter shard for the next AllGather
    shard = param_full[rank * S:(rank + 1) * S]
    if eb == 2:
        b = bf16_bits(shard)
        rne = OD.to_bf16_rne(gm)
        assert np.array_equal(b[mask], rne[mask])
        # by value: the fp32 param tolerance plus one bf16 ulp (bit patterns
        # of near-zero params, |p| << lr, are not comparable)
        bv = OD.bf16_to_f32(b[fin]).astype(np.float64)
        rv = OD.bf16_to_f32(ref[5][fin]).astype(np.float64)
        r0 = np.abs(ref[0][fin]).astype(np.float64)
        # one bf16 ulp is <= 2^-7 |x| (8 significant bits)
        assert np.all(np.abs(bv - rv) <= 1e-5 * (r0 + lr) + 2.0 ** -7 * r0)
        assert not b[~mask].any()
    else:
        assert np.array_equal(f32(shard)[mask].view(np.uint32), gm[mask].view(np.uint32))


ADAM_CASES = [
    # es, q, m, eb, rank, step, warm
    ([256 * 128, 256] * 6, 2048, 2, 4, 1, 1, False),          # toy config, fp32 unit
    ([256 * 128, 256] * 6, 2048, 2, 4, 0, 5, True),
    ([5000, 77, 4109, 2048 * 3, 1, 40000], 2048, 3, 2, 0, 3, True),   # ragged, misaligned
    ([5000, 77, 4109, 2048 * 3, 1, 40000], 2048, 3, 2, 2, 3, True),
    ([5000, 77, 4109, 2048 * 3, 1, 40000], 2048, 1, 2, 0, 1, False),
    ([2048 * 40, 2048 * 7 + 100, 33], 4096, 2, 2, 1, 2, True),     # q > 2048: two-pass path
    ([2048 * 40, 2048 * 7 + 100, 33], 1024, 4, 2, 3, 9, True),
    ([2048 * 64 + 1000], 2048, 8, 2, 5, 100, True),
]


@pytest.mark.parametrize("es,q,m,eb,rank,step,warm", ADAM_CASES)
def test_adam8_parity(es, q, m, eb, rank, step, warm):
    _adam_case(es, q, m, eb, rank, step, warm)


@pytest.mark.parametrize("es,q,m,eb,rank,step,warm", [ADAM_CASES[i] for i in (0, 1, 3, 4, 5, 7)])
def test_adam8_dynamic_codec_parity(es, q, m, eb, rank, step, warm):
    """N2: the dynamic (tree) code map codec (R25) against the oracle: codes
    (map indices) and absmax exact (same moments, same fp32 nearest-code
    decision), params 1e-5 (|p| + lr)."""
    _adam_case(es, q, m, eb, rank, step, warm, codec="dynamic")


# ---- the codec at its edges (R27): tiny / subnormal / zero absmax, long runs
# of zero gradients, full-mantissa gradients over many decades, non-finite
# gradients.  Codes and absmax must be exact (same IEEE operations).
EDGE_ES = [2048 * 6, 2048 + 700, 5000]


def _edge_state(S, nb, seed, am_vals, av_vals):
    rng = np.random.default_rng(seed)
    mq = rng.integers(-127, 128, S).astype(np.int8)
    vq = rng.integers(0, 256, S).astype(np.uint8)
    ma = np.resize(np.float32(am_vals), nb).astype(np.float32)
    va = np.resize(np.float32(av_vals), nb).astype(np.float32)
    return mq, vq, ma, va


@pytest.mark.parametrize("codec", ["linear", "dynamic"])
def test_adam8_tiny_absmax_states(codec):
    """Warm states whose absmax sits where fl(127/A) / fl(255/A) overflow or
    fl(A/L) is subnormal or 0 (A from 3.7e-37 down to 1e-45 and 0), with zero,
    tiny and ordinary gradients."""
    es = EDGE_ES
    o, c = _plans(es, [min(2048, e) for e in es], 1, 2)
    S, E = c.S, sum(es)
    nb = len(OP.rank_blocks(o, 0, 2048))
    am = [3.7e-37, 1e-38, 1e-40, 1e-43, 1e-45, 0.0, 2e-37, 5e-39]
    av = [7.5e-37, 1e-39, 3e-42, 1e-44, 0.0, 1e-45, 6e-37, 2e-38]
    rng = np.random.default_rng(2)
    g = np.zeros(E, np.float32)
    g[2048:4096] = rng.normal(0, 1e-30, 2048)
    g[4096:6144] = rng.normal(0, 1e-20, 2048)
    g[8192:] = rng.normal(0, 1e-3, E - 8192)
    st = _edge_state(S, nb, 3, am, av)
    if codec == "dynamic":
        st = (st[0].view(np.uint8), st[1], st[2], st[3])
    _adam_case(es, 2048, 1, 2, 0, 900, False, g_log=torch.from_numpy(g), state=st, codec=codec)


@pytest.mark.parametrize("scale", [1e-8, 1e-4, 1.0, 1e2])
def test_adam8_full_mantissa_grads(scale):
    """Random-normal fp32 gradients (every mantissa bit used) at one scale per
    case over ten decades, warm state: codes / absmax exact, params 1e-5."""
    es = EDGE_ES + [2048 * 8]
    E = sum(es)
    g = (np.random.default_rng(int(np.log10(scale)) + 20).normal(0, 1, E) * scale).astype(np.float32)
    _adam_case(es, 2048, 1, 2, 0, 4, True, seed=3, g_log=torch.from_numpy(g))


@pytest.mark.parametrize("codec", ["linear", "dynamic"])
def test_adam8_nonfinite_gradients(codec):
    """R27: a NaN gradient in block 0, +inf in block 1, -inf in block 2,
    ordinary gradients elsewhere.  The poisoned blocks keep A = NaN / +inf and
    all-zero codes (the code of 0), their non-finite elements' params become
    NaN, every other element matches the oracle; then a second step from the
    poisoned state (dequantisation 0 * NaN)."""
    es = EDGE_ES
    E = sum(es)
    g = np.random.default_rng(4).normal(0, 1e-3, E).astype(np.float32)
    g[5] = np.nan
    g[2048 + 77] = np.inf
    g[4096 + 2047] = -np.inf
    _adam_case(es, 2048, 1, 2, 0, 2, True, seed=4, g_log=torch.from_numpy(g), codec=codec)


def test_adam8_zero_gradient_run():
    """A block whose gradient stays 0 decays m by beta1 per step until A_m
    falls below 127 / FLT_MAX (~730 steps) and on into the subnormals: 850
    free-running GPU steps against 850 oracle steps; codes and absmax stay
    exact at every checkpoint, params within 1e-5 (|p| + lr)."""
    es = [2048 * 2, 700]
    o, c = _plans(es, [min(2048, e) for e in es], 1, 2)
    S, E = c.S, sum(es)
    g1 = np.random.default_rng(6).normal(0, 1e-3, E).astype(np.float32)
    g1[2048:4096] = 0  # one block never sees a gradient
    grad_f32 = place_gpu(c, torch.from_numpy(g1), torch.float32)
    param_full = torch.zeros(S, dtype=torch.bfloat16, device="cuda")
    u = R.Unit(c, 0, param_full, torch.zeros(S, dtype=torch.bfloat16, device="cuda"), grad_f32, qblock=2048)
    p_log = logical_params(6, E)
    master = place_gpu(c, p_log, torch.float32)
    nb = u.num_blocks
    st = [master, torch.zeros(S, dtype=torch.int8, device="cuda"), torch.zeros(S, dtype=torch.uint8, device="cuda"),
          torch.zeros(nb, device="cuda"), torch.zeros(nb, device="cuda")]
    blocks = OP.rank_blocks(o, 0, 2048)
    ref = (f32(master), np.zeros(S, np.int8), np.zeros(S, np.uint8), np.zeros(nb, np.float32),
           np.zeros(nb, np.float32))
    g_or = OD.shard(o, OD.place_logical(o, g1), 0)
    cfg = R.AdamConfig()
    for t in range(1, 851):
        R.step_8bit_adam(u, *st, cfg, t)
        ref = OA.step_8bit_adam(ref[0], g_or, ref[1], ref[2], ref[3], ref[4], blocks, OA.AdamCfg(), t)[:5]
        if t == 1:
            grad_f32.zero_()
            g_or = np.zeros_like(g_or)
        if t % 50 == 0 or t == 1:
            torch.cuda.synchronize()
            assert np.array_equal(st[1].cpu().numpy(), ref[1]), t
            assert np.array_equal(st[2].cpu().numpy(), ref[2]), t
            assert np.array_equal(f32(st[3]).view(np.uint32), ref[3].view(np.uint32)), t
            assert np.array_equal(f32(st[4]).view(np.uint32), ref[4].view(np.uint32)), t
            # params drift only through the approximate sqrt / rcp of the
            # update: within 1e-5 (|p| + lr) over 50 steps, then resynced
            gm = f32(master)
            assert np.all(np.abs(gm - ref[0]) <= 1e-5 * (np.abs(ref[0]) + cfg.lr)), t
            ref = (gm.copy(),) + tuple(ref[1:])
    am = f32(st[3])
    assert 0 < am.max() < 3.7e-37  # every block with a step-1 gradient reached the regime


TILE_CASES = [
    # shapes, specs (per tensor), row granularity, m, rank
    ([(96, 64), (64, 40), (130,)], [("tile", 64, 32, 32), ("tile", 40, 32, 32), ("flat", 130)], 32, 2, 1),
    ([(2048, 512), (512,), (100, 96)], [("tile", 512, 32, 32), ("flat", 512), ("tile", 96, 32, 32)], 32, 3, 2),
    ([(256, 128)], [("tile", 128, 128, 128)], 128, 2, 0),          # 128x128 tiles: two-pass path
    ([(64, 30), (40, 66)], [("tile", 30, 8, 5), ("tile", 66, 8, 6)], 8, 2, 1),  # masked strided path
    # Llama-like mix at world 1: many tile pairs, a flat block between tensors
    # (unpaired items), a 1-row tail tile
    ([(128, 2048), (2048,), (64, 512), (33, 64)],
     [("tile", 2048, 32, 32), ("flat", 2048), ("tile", 512, 32, 32), ("tile", 64, 32, 32)], 32, 1, 0),
]


@pytest.mark.parametrize("shapes,specs,rows,m,rank", TILE_CASES)
def test_adam8_tiles_parity(shapes, specs, rows, m, rank):
    """N2: the paper's 8-bit Adam setup -- 2-D quantization tiles with row
    sharding granularity -- vs the oracle, through rsdb_unit_create_q."""
    es = [int(np.prod(s)) for s in shapes]
    gs = [rows * s[-1] if len(s) == 2 else min(int(sp[1]), int(np.prod(s)))
          for s, sp in zip(shapes, specs)]
    o, c = _plans(es, gs, m, 2)
    E, S = sum(es), c.S
    tiles_o = OP.rank_tiles(o, rank, specs)
    assert c.rank_tiles(rank, specs) == [tuple(t) for t in tiles_o]
    p_log, g_log = logical_params(4, E), logical_grads(4, rank, E)
    master = place_gpu(c, p_log, torch.float32)[rank * S:(rank + 1) * S].clone()
    grad_f32 = place_gpu(c, g_log, torch.float32)
    grad_full = torch.zeros(m * S, dtype=torch.bfloat16, device="cuda")
    param_full = torch.zeros(m * S, dtype=torch.bfloat16, device="cuda")
    u = R.Unit(c, rank, param_full, grad_full, grad_f32, qspec=specs)
    nb = u.num_blocks
    assert nb == len(tiles_o)
    mq = H.codes_torch(4, H.STREAM_MCODE, rank * S, S, True, device="cuda")
    vq = H.codes_torch(4, H.STREAM_VCODE, rank * S, S, False, device="cuda")
    ma = H.absmax_torch(4, H.STREAM_ABSM, 0, nb, 14, device="cuda")
    va = H.absmax_torch(4, H.STREAM_ABSV, 0, nb, 22, device="cuda")
    ins = [t.cpu().numpy().copy() for t in (master, mq, vq, ma, va)]
    cfg = R.AdamConfig()
    R.step_8bit_adam(u, master, mq, vq, ma, va, cfg, 6)
    torch.cuda.synchronize()
    g_or = OD.shard(o, OD.place_logical(o, g_log.numpy()), rank)
    ref = OA.step_8bit_adam(ins[0], g_or, ins[1], ins[2], ins[3], ins[4], tiles_o, OA.AdamCfg(), 6)
    _check_adam(o, rank, tiles_o, (master, mq, vq, ma, va, param_full), ref, ins, 2, cfg.lr)


@pytest.mark.parametrize("es", [[5000 * 4, 2048 * 3, 256, 4096 + 16], [256 * 128, 256] * 3,
                                [77, 5000, 2048 * 2 + 3]])
def test_fused_rs_adam_world1(es):
    """a6 + a7 + a8 in one kernel at world 1 (= cast + 8-bit Adam), vs the
    oracle's group op followed by its Adam step; grad_f32 is not written."""
    q = 2048
    gs = [min(q, e) for e in es]
    o, c = _plans(es, gs, 1, 2)
    S, E = c.S, sum(es)
    comm = R.Comm(R.Comm.unique_id(), 1, 0, 0)
    p_log, g_log = logical_params(8, E), logical_grads(8, 0, E)
    grad_full = place_gpu(c, g_log, torch.bfloat16)
    grad_f32 = torch.full((S,), float("nan"), dtype=torch.float32, device="cuda")
    param_full = torch.zeros(S, dtype=torch.bfloat16, device="cuda")
    master = place_gpu(c, p_log, torch.float32).clone()
    u = R.Unit(c, 0, param_full, grad_full, grad_f32, qblock=q, comm=comm)
    nb = u.num_blocks
    mq = H.codes_torch(8, H.STREAM_MCODE, 0, S, True, device="cuda")
    vq = H.codes_torch(8, H.STREAM_VCODE, 0, S, False, device="cuda")
    ma = H.absmax_torch(8, H.STREAM_ABSM, 0, nb, 14, device="cuda")
    va = H.absmax_torch(8, H.STREAM_ABSV, 0, nb, 22, device="cuda")
    ins = [t.cpu().numpy().copy() for t in (master, mq, vq, ma, va)]
    cfg = R.AdamConfig()
    R.reduce_scatter_adam_p2p(u, None, cfg, 3, state=(master, mq, vq, ma, va))
    torch.cuda.synchronize()
    assert torch.isnan(grad_f32).all()
    g_or = OD.grouped_cast_scale(o, OD.to_bf16_rne(OD.place_logical(o, g_log.numpy())), True)
    blocks = OP.rank_blocks(o, 0, q)
    ref = OA.step_8bit_adam(ins[0], g_or, ins[1], ins[2], ins[3], ins[4], blocks, OA.AdamCfg(), 3)
    _check_adam(o, 0, blocks, (master, mq, vq, ma, va, param_full), ref, ins, 2, cfg.lr)
    del u
    comm.close()


def test_adam8_zero_gradient_block():
    """Zero state + zero gradient: m = v = 0 -> absmax 0 -> codes 0."""
    _adam_case([4096, 2048, 300], 2048, 1, 2, 0, 1, False, zero_grad_tensor=1)


# ------------------------------------------------------ unit through NCCL, world 1
def test_unit_world1_nccl_path():
    u_decl = W.llama32_1b_layer(0)
    es = [t.numel for t in u_decl.tensors][:4] + [2048, 2048]
    gs = [min(2048, e) for e in es]
    o, c = _plans(es, gs, 1, 2)
    comm = R.Comm(R.Comm.unique_id(), 1, 0, 0)
    E, S = sum(es), c.S
    p_log, g_log = logical_params(1, E), logical_grads(1, 0, E)
    param_full = place_gpu(c, p_log, torch.bfloat16)
    before = param_full.clone()
    grad_full = place_gpu(c, g_log, torch.bfloat16)
    grad_f32 = torch.empty(S, dtype=torch.float32, device="cuda")
    u = R.Unit(c, 0, param_full, grad_full, grad_f32, qblock=2048, comm=comm)
    R.all_gather(u)
    R.reduce_scatter(u)
    torch.cuda.synchronize()
    assert torch.equal(param_full.view(torch.int16), before.view(torch.int16))
    ref = OD.grouped_cast_scale(o, OD.to_bf16_rne(OD.place_logical(o, g_log.numpy())), True)
    assert np.array_equal(f32(grad_f32), ref)
    del u
    comm.close()


# ------------------------------------------------------ DBuffer one-launch Adam
def test_dbuffer_one_launch_equals_per_unit_oracle():
    decl = [([t.numel for t in W.llama32_1b_layer(0).tensors][-3:] + [70000, 33], 2)]
    decl.append(([256 * 128, 256, 256 * 128, 256], 2))
    decl.append(([2048 * 5 + 7, 19, 4096], 2))
    m, rank, q = 4, 1, 2048
    lays_o, lays_c = [], []
    for es, eb in decl:
        o, c = _plans(es, [min(q, e) for e in es], m, eb)
        lays_o.append(o)
        lays_c.append(c)
    sizes, offs = R.arena_sizes(lays_c, rank, q, 256)
    ar = [torch.zeros(max(1, s), dtype=torch.uint8, device="cuda") for s in sizes]
    db = R.DBuffer(lays_c, rank, ar, qblock=q, align=256)
    assert db.num_blocks == sum(len(l.rank_blocks(rank, q)) for l in lays_c)
    refs, ins_all, views = [], [], []
    for ui, ((es, eb), o, c) in enumerate(zip(decl, lays_o, lays_c)):
        E, S = sum(es), c.S
        off = offs[ui]
        nb = len(c.rank_blocks(rank, q))
        v = {
            "param_full": ar[0][off[0]:off[0] + m * S * 2].view(torch.bfloat16),
            "grad_f32": ar[2][off[2]:off[2] + m * S * 4].view(torch.float32),
            "master": ar[3][off[3]:off[3] + S * 4].view(torch.float32),
            "mq": ar[4][off[4]:off[4] + S].view(torch.int8),
            "vq": ar[5][off[5]:off[5] + S],
            "ma": ar[6][off[6]:off[6] + nb * 4].view(torch.float32),
            "va": ar[7][off[7]:off[7] + nb * 4].view(torch.float32),
        }
        p_log, g_log = logical_params(ui, E), logical_grads(ui, rank, E)
        v["master"].copy_(place_gpu(c, p_log, torch.float32)[rank * S:(rank + 1) * S])
        v["grad_f32"].copy_(place_gpu(c, g_log, torch.float32))
        v["mq"].copy_(H.codes_torch(ui, H.STREAM_MCODE, 0, S, True, device="cuda"))
        v["vq"].copy_(H.codes_torch(ui, H.STREAM_VCODE, 0, S, False, device="cuda"))
        v["ma"].copy_(H.absmax_torch(ui, H.STREAM_ABSM, 0, nb, 14, device="cuda"))
        v["va"].copy_(H.absmax_torch(ui, H.STREAM_ABSV, 0, nb, 22, device="cuda"))
        ins = [v[k].cpu().numpy().copy() for k in ("master", "mq", "vq", "ma", "va")]
        blocks = OP.rank_blocks(o, rank, q)
        g_or = OD.shard(o, OD.place_logical(o, g_log.numpy()), rank)
        refs.append(OA.step_8bit_adam(ins[0], g_or, ins[1], ins[2], ins[3], ins[4], blocks,
                                      OA.AdamCfg(), 4))
        ins_all.append(ins)
        views.append(v)
    cfg = R.AdamConfig()
    db.step_8bit_adam(cfg, 4)
    torch.cuda.synchronize()
    for o, v, ref, ins in zip(lays_o, views, refs, ins_all):
        _check_adam(o, rank, OP.rank_blocks(o, rank, q),
                    (v["master"], v["mq"], v["vq"], v["ma"], v["va"], v["param_full"]),
                    ref, ins, 2, cfg.lr)
    db.close()


def test_dbuffer_step_host_world1():
    """rsdb_dbuffer_step_host (the e2e entry point): host bf16 gradients in,
    per-unit fused RS + 8-bit Adam, host bf16 shards out -- two steps, each
    against the oracle's step on the same state (state resynced to the
    oracle's after step 1, as in _adam_case), host shards = RNE(GPU master)."""
    decl = [[2048 * 3 + 5, 77, 4096], [256 * 128, 256], [2048 * 7]]
    q, m, rank = 2048, 1, 0
    lays_o, lays_c = [], []
    for es in decl:
        o, c = _plans(es, [min(q, e) for e in es], m, 2)
        lays_o.append(o)
        lays_c.append(c)
    sizes, offs = R.arena_sizes(lays_c, rank, q, 256)
    ar = [torch.zeros(max(1, s), dtype=torch.uint8, device="cuda") for s in sizes]
    db = R.DBuffer(lays_c, rank, ar, qblock=q, align=256)
    views, host_g, host_p, g_logs = [], [], [], []
    for ui, (es, c) in enumerate(zip(decl, lays_c)):
        E, S, off = sum(es), c.S, offs[ui]
        nb = len(c.rank_blocks(rank, q))
        v = {"param_full": ar[0][off[0]:off[0] + S * 2].view(torch.bfloat16),
             "master": ar[3][off[3]:off[3] + S * 4].view(torch.float32),
             "mq": ar[4][off[4]:off[4] + S].view(torch.int8), "vq": ar[5][off[5]:off[5] + S],
             "ma": ar[6][off[6]:off[6] + nb * 4].view(torch.float32),
             "va": ar[7][off[7]:off[7] + nb * 4].view(torch.float32)}
        v["master"].copy_(place_gpu(c, logical_params(ui, E), torch.float32))
        views.append(v)
        g = logical_grads(ui, rank, E)
        g_logs.append(g)
        host_g.append(place_gpu(c, g, torch.bfloat16).cpu().pin_memory())
        host_p.append(torch.zeros(S, dtype=torch.bfloat16).pin_memory())
    cfg = R.AdamConfig()
    st = torch.cuda.Stream()
    for step in (1, 2):
        ins_all = [[v[k].cpu().numpy().copy() for k in ("master", "mq", "vq", "ma", "va")]
                   for v in views]
        db.step_host(cfg, step, host_g, host_p, None, st)
        st.synchronize()
        for ui, (o, v, ins) in enumerate(zip(lays_o, views, ins_all)):
            blocks = OP.rank_blocks(o, rank, q)
            g_or = OD.bf16_to_f32(OD.to_bf16_rne(OD.place_logical(o, g_logs[ui].numpy())))
            ref = OA.step_8bit_adam(ins[0], g_or, ins[1], ins[2], ins[3], ins[4], blocks,
                                    OA.AdamCfg(), step)
            _check_adam(o, rank, blocks, (v["master"], v["mq"], v["vq"], v["ma"], v["va"],
                                          v["param_full"]), ref, ins, 2, cfg.lr)
            assert np.array_equal(bf16_bits(host_p[ui]), bf16_bits(v["param_full"].cpu()))
            assert np.array_equal(bf16_bits(host_p[ui]),
                                  bf16_bits(v["master"].cpu().to(torch.bfloat16)))
    db.close()


def test_dbuffer_step_host_chunked_equals_device_step():
    """A unit larger than step_host's 16 M-element copy-out chunk (3 chunks)
    next to small ones: the chunked host-buffer step is bit-identical to the
    device-resident fused step on the same inputs (states, shard, host copy)."""
    decl = [[20_000_000, 17_000_000 + 5], [2048 * 3 + 7, 77], [4096]]
    q = 2048
    res = []
    for mode in ("host", "device"):
        lays = [R.plan(es, [min(q, e) for e in es], 1, elem_bytes=2) for es in decl]
        sizes, offs = R.arena_sizes(lays, 0, q, 256)
        ar = [torch.zeros(max(1, sz), dtype=torch.uint8, device="cuda") for sz in sizes]
        db = R.DBuffer(lays, 0, ar, qblock=q, align=256)
        host_g, host_p = [], []
        for ui, (es, c) in enumerate(zip(decl, lays)):
            E, S, off = sum(es), c.S, offs[ui]
            ar[3][off[3]:off[3] + S * 4].view(torch.float32).copy_(place_gpu(c, logical_params(ui, E), torch.float32))
            g = place_gpu(c, logical_grads(ui, 0, E), torch.bfloat16)
            if mode == "device":
                ar[1][off[1]:off[1] + S * 2].view(torch.bfloat16).copy_(g)
            host_g.append(g.cpu().pin_memory())
            host_p.append(torch.zeros(S, dtype=torch.bfloat16).pin_memory())
        cfg = R.AdamConfig()
        for t in (1, 2):
            if mode == "host":
                db.step_host(cfg, t, host_g, host_p)
            else:
                db.reduce_scatter_adam_gather(cfg, t)
        torch.cuda.synchronize()
        res.append(([a.cpu() for a in ar[3:]], ar[0].cpu(), host_p))
        db.close()
    (st_h, pf_h, hp), (st_d, pf_d, _) = res
    for a, b in zip(st_h, st_d):
        assert torch.equal(a, b)
    assert torch.equal(pf_h, pf_d)
    lays = [R.plan(es, [min(q, e) for e in es], 1, elem_bytes=2) for es in decl]
    _, offs = R.arena_sizes(lays, 0, q, 256)
    for ui, c in enumerate(lays):
        shard = pf_h[offs[ui][0]:offs[ui][0] + c.S * 2].view(torch.int16)
        assert torch.equal(hp[ui].view(torch.int16), shard), ui


def test_dbuffer_step_host_rejects_null():
    c = R.plan([4096], [2048], 1, elem_bytes=2)
    sizes, _ = R.arena_sizes([c], 0, 2048, 256)
    ar = [torch.zeros(max(1, s), dtype=torch.uint8, device="cuda") for s in sizes]
    db = R.DBuffer([c], 0, ar, qblock=2048, align=256)
    with pytest.raises(R.RsdbError):
        db.step_host(R.AdamConfig(), 1, [None], [None])
    with pytest.raises(ValueError):
        db.step_host(R.AdamConfig(), 1, [], [])
    db.close()


def test_dbuffer_tiles_one_launch_equals_oracle():
    """The DBuffer step over units planned with 32-row granularity and 32x32
    tiles (the paper's 8-bit Adam setup; dispatched to the paired-tile
    kernel) against the oracle's tiled step, unit by unit, at world 2."""
    decl = [[(256, 512), (512,), (96, 64)], [(64, 2048), (2048,)], [(40, 128), (33, 32)]]
    m, rank = 2, 1
    units = []
    for shapes in decl:
        es = [int(np.prod(s)) for s in shapes]
        gs = [32 * s[-1] if len(s) == 2 else min(2048, e) for s, e in zip(shapes, es)]
        specs = [("tile", s[-1], 32, 32) if len(s) == 2 else ("flat", min(2048, e)) for s, e in zip(shapes, es)]
        o, c = _plans(es, gs, m, 2)
        units.append((es, specs, o, c))
    lays_c = [u[3] for u in units]
    qs = [u[1] for u in units]
    sizes, offs = R.arena_sizes(lays_c, rank, qspec=qs)
    ar = [torch.zeros(max(1, sz), dtype=torch.uint8, device="cuda") for sz in sizes]
    db = R.DBuffer(lays_c, rank, ar, qspec=qs)
    refs, ins_all, views, tiles_all = [], [], [], []
    for ui, (es, specs, o, c) in enumerate(units):
        E, S, off = sum(es), c.S, offs[ui]
        tiles = OP.rank_tiles(o, rank, specs)
        nb = len(tiles)
        v = {"param_full": ar[0][off[0]:off[0] + m * S * 2].view(torch.bfloat16),
             "grad_f32": ar[2][off[2]:off[2] + m * S * 4].view(torch.float32),
             "master": ar[3][off[3]:off[3] + S * 4].view(torch.float32),
             "mq": ar[4][off[4]:off[4] + S].view(torch.int8), "vq": ar[5][off[5]:off[5] + S],
             "ma": ar[6][off[6]:off[6] + nb * 4].view(torch.float32),
             "va": ar[7][off[7]:off[7] + nb * 4].view(torch.float32)}
        p_log, g_log = logical_params(20 + ui, E), logical_grads(20 + ui, rank, E)
        v["master"].copy_(place_gpu(c, p_log, torch.float32)[rank * S:(rank + 1) * S])
        v["grad_f32"].copy_(place_gpu(c, g_log, torch.float32))
        v["mq"].copy_(H.codes_torch(ui, H.STREAM_MCODE, 0, S, True, device="cuda"))
        v["vq"].copy_(H.codes_torch(ui, H.STREAM_VCODE, 0, S, False, device="cuda"))
        v["ma"].copy_(H.absmax_torch(ui, H.STREAM_ABSM, 0, nb, 14, device="cuda"))
        v["va"].copy_(H.absmax_torch(ui, H.STREAM_ABSV, 0, nb, 22, device="cuda"))
        ins = [v[k].cpu().numpy().copy() for k in ("master", "mq", "vq", "ma", "va")]
        g_or = OD.shard(o, OD.place_logical(o, g_log.numpy()), rank)
        refs.append(OA.step_8bit_adam(ins[0], g_or, ins[1], ins[2], ins[3], ins[4], tiles, OA.AdamCfg(), 3))
        ins_all.append(ins)
        views.append(v)
        tiles_all.append(tiles)
    assert db.num_blocks == sum(len(t) for t in tiles_all)
    cfg = R.AdamConfig()
    db.step_8bit_adam(cfg, 3)
    torch.cuda.synchronize()
    for (es, specs, o, c), v, ref, ins, tiles in zip(units, views, refs, ins_all, tiles_all):
        _check_adam(o, rank, tiles, (v["master"], v["mq"], v["vq"], v["ma"], v["va"], v["param_full"]),
                    ref, ins, 2, cfg.lr)
    db.close()


# ------------------------------------------------------------------ copies
def test_copy_plan_parity():
    rng = np.random.default_rng(0)
    n_seg = 37
    lens = rng.integers(1, 20000, n_seg)
    src = torch.from_numpy(H.params_np(3, 0, int(lens.sum()) + 64)).cuda()
    dst32 = torch.zeros(int(lens.sum()) + 64 * n_seg, dtype=torch.float32, device="cuda")
    dst16 = torch.zeros_like(dst32, dtype=torch.bfloat16)
    segs32, segs16, exp = [], [], np.zeros(dst32.numel(), np.float32)
    so = do = 0
    srcn = src.cpu().numpy()
    for i, n in enumerate(lens):
        n = int(n)
        so_i = so + (i % 3)            # misaligned starts for some segments
        segs32.append((src.data_ptr() + 4 * so_i, dst32.data_ptr() + 4 * do, n))
        segs16.append((src.data_ptr() + 4 * so_i, dst16.data_ptr() + 2 * do, n))
        exp[do:do + n] = srcn[so_i:so_i + n] * np.float32(0.5)
        so += n
        do += n + (i % 5)
    R.CopyPlan(segs32, R.RSDB_F32, R.RSDB_F32, 0.5).run()
    R.CopyPlan(segs16, R.RSDB_F32, R.RSDB_BF16, 0.5).run()
    torch.cuda.synchronize()
    assert np.array_equal(f32(dst32), exp)
    assert np.array_equal(bf16_bits(dst16), OD.to_bf16_rne(exp))
