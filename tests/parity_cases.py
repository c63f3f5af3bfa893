"""Multi-rank parity cases: the CUDA path through the C-ABI on every rank vs
the oracle's simulated ranks (and the fused kernels vs the unfused sequence
of kernels), element by element.  Each case is a generator function of a rank
context (tests/rank_ctx.py), so the same code runs

  * as logical ranks on ONE device (tests/local_ranks_worker.py, driven by
    tests/test_gpu_local_ranks.py at world 2, 3, 4, 8 -- runs on the driver's
    1-GPU box), and
  * one process per GPU (tests/dist_parity_worker.py under torchrun,
    tests/test_gpu_multi.py -- multi-GPU boxes only; adds the NCCL checks).

Tolerances: layouts / AllGather / the p2p ReduceScatter
(rank-order fp32 sum, as the oracle) / 8-bit codes and absmax: bit exact;
NCCL ReduceScatter: |y - y64| <= 1e-6 sum|x| (bit exact at m a power of two
on the dyadic synth inputs); params |dp| <= 1e-5 (|p| + lr); fused kernels:
bit identical to the unfused sequence.
"""
from __future__ import annotations

import numpy as np
import torch

import paper_2602_22437_b200 as R
from oracle import adam8 as OA
from oracle import dbuffer as OD
from oracle import fp8 as F
from oracle import muon as MU
from oracle import planner as OP
from synth import hashgen as H
from synth import workloads as W

from gpu_helpers import bf16_bits, f32, logical_grads, logical_params, place_gpu


def _plans(es, gs, m, eb):
    o = OP.plan(es, gs, m, OP.gcoll_elems(eb))
    c = R.plan(es, gs, m, elem_bytes=eb)
    assert list(c.starts) == list(o.starts) and c.S == o.S
    return o, c


def _zero_state(S, nb, dev="cuda"):
    return [torch.zeros(S, dtype=torch.int8, device=dev), torch.zeros(S, dtype=torch.uint8, device=dev),
            torch.zeros(max(nb, 1), device=dev), torch.zeros(max(nb, 1), device=dev)]


def _same_bytes(a, b):
    return torch.equal(a.view(torch.uint8), b.view(torch.uint8))


def _block_mask(S, blocks):
    mask = np.zeros(S, bool)
    for blk in blocks:
        if len(blk) == 2:
            mask[blk[0]:blk[0] + blk[1]] = True
        else:
            off, rows, cols, pitch = blk
            mask[(off + np.arange(rows)[:, None] * pitch + np.arange(cols)[None, :]).ravel()] = True
    return mask


def check_adam_exact(ctx, tag, S, blocks, gpu, ref, lr):
    """GPU state (master, m_q, v_q, m_abs, v_abs) vs the oracle's: codes and
    absmax bit exact (the same IEEE operations on both sides: R26, R9), params
    |dp| <= 1e-5 (|p| + lr)."""
    master, mq, vq, ma, va = gpu
    mask = _block_mask(S, blocks)
    nb = len(blocks)
    gm = f32(master)
    err = (np.abs(gm - ref[0]) / (np.abs(ref[0]) + lr))[mask]
    if err.max(initial=0) > 1e-5:
        ctx.fail(f"{tag}: Adam params off by {err.max():.3e}")
    for name, g, r in (("m codes", mq, ref[1]), ("v codes", vq, ref[2])):
        d = g.cpu().numpy().astype(np.int32)[mask] != r.astype(np.int32)[mask]
        if d.any():
            ctx.fail(f"{tag}: {name} differ from the oracle at {int(d.sum())} elements")
    for name, g, r in (("m absmax", ma, ref[3]), ("v absmax", va, ref[4])):
        if not np.array_equal(f32(g)[:nb].view(np.uint32), r[:nb].view(np.uint32)):
            ctx.fail(f"{tag}: {name} not bit exact")


# ---------------------------------------------------------------- units
def unit_configs():
    lay = W.llama32_1b_layer(0)
    yield "toy", [t.numel for t in W.toy().units[0].tensors], 2048, 4
    yield "llama-attn", [t.numel for t in lay.tensors][:4] + [2048, 2048], 2048, 2
    yield "ragged", [5000, 77, 4109, 2048 * 3, 1, 40000, 2048 * 11 + 3], 2048, 2


def units_case(ctx):
    """a4 / a7 / a6+a7+a8 / + a4 on three units: p2p AllGather and
    ReduceScatter bit exact against the oracle, 8-bit Adam on the reduced
    shard against the oracle (codes exact), the fused kernels bit identical to
    the unfused sequence, repeated calls consistent across ranks."""
    rank, world = ctx.rank, ctx.world
    cfg = R.AdamConfig()
    for name, es, q, eb in unit_configs():
        if eb == 4 and not ctx.has_nccl:
            continue  # f32 units reduce through NCCL only (the p2p RS is bf16)
        gs = [min(q, e) for e in es]
        o, c = _plans(es, gs, world, eb)
        S, E = c.S, sum(es)
        dt = torch.bfloat16 if eb == 2 else torch.float32
        p_log = logical_params(5, E)
        full_ref = place_gpu(c, p_log, dt)
        param_full = torch.zeros_like(full_ref)
        param_full[rank * S:(rank + 1) * S] = full_ref[rank * S:(rank + 1) * S]
        grad_full = place_gpu(c, logical_grads(5, rank, E), dt, fill=float("nan"))
        grad_f32 = grad_full if eb == 4 else torch.empty(world * S, dtype=torch.float32, device="cuda")
        u = R.Unit(c, rank, param_full, grad_full, grad_f32, qblock=q, comm=ctx.comm)
        exp = OD.place_logical(o, p_log.numpy())
        exp_bits = OD.to_bf16_rne(exp) if eb == 2 else exp.view(np.uint32)

        def bits(t):
            return bf16_bits(t) if eb == 2 else f32(t).view(np.uint32)

        bufs = []
        for r in range(world):
            src = OD.place_logical(o, logical_grads(5, r, E).numpy(), fill=np.nan)
            bufs.append(OD.grouped_cast_scale(o, OD.to_bf16_rne(src) if eb == 2 else src, eb == 2))
        y_all = OD.reduce_scatter(o, bufs)  # the oracle's reduced shard of every rank
        y_ref = y_all[rank]
        if ctx.has_nccl:
            R.all_gather(u)
            yield
            if not np.array_equal(bits(param_full), exp_bits):
                ctx.fail(f"{name}: NCCL AllGather mismatch")
            R.reduce_scatter(u)
            yield
            y = f32(grad_f32[rank * S:(rank + 1) * S])
            if world & (world - 1) == 0:
                if not np.array_equal(y.view(np.uint32), y_ref.view(np.uint32)):
                    ctx.fail(f"{name}: NCCL ReduceScatter not bit exact")
            else:  # NCCL's order differs from rank order: the fp32 bound
                y64 = OD.reduce_scatter_f64(o, bufs)[rank]
                absum = sum(np.abs(x[rank * S:(rank + 1) * S].astype(np.float64)) for x in bufs)
                if np.any(np.abs(y.astype(np.float64) - y64) > 1e-6 * absum + 1e-30):
                    ctx.fail(f"{name}: NCCL ReduceScatter outside 1e-6 sum|x|")
            param_full.zero_()
            param_full[rank * S:(rank + 1) * S] = full_ref[rank * S:(rank + 1) * S]
        # ---- N1: the collectives as single kernels over peer memory
        p2p = yield from ctx.p2p([param_full, grad_full] if eb == 2 else [param_full])
        R.all_gather_p2p(u, p2p)
        yield
        if not np.array_equal(bits(param_full), exp_bits):
            ctx.fail(f"{name}: p2p AllGather mismatch")
        if eb == 2:
            grad_f32.fill_(float("nan"))
            R.reduce_scatter_p2p(u, p2p)
            yield
            y = f32(grad_f32[rank * S:(rank + 1) * S])
            if not np.array_equal(y.view(np.uint32), y_ref.view(np.uint32)):
                ctx.fail(f"{name}: p2p ReduceScatter not bit exact")
            for _ in range(3):  # repeated calls: epochs advance, barriers re-arm
                R.reduce_scatter_p2p(u, p2p)
                R.all_gather_p2p(u, p2p)
            yield
            y = f32(grad_f32[rank * S:(rank + 1) * S])
            if not np.array_equal(y.view(np.uint32), y_ref.view(np.uint32)):
                ctx.fail(f"{name}: repeated p2p ReduceScatter drifted")
        if eb == 4 and world & (world - 1):
            continue  # NCCL's fp32 order makes the reduced gradient non-unique here
        # ---- a8 on the reduced shard (grad_f32 = the oracle's y bit for bit)
        master = torch.from_numpy(OD.shard(o, exp, rank).copy()).cuda()
        nb = u.num_blocks
        st_a = [master] + _zero_state(S, nb)
        st_f = [t.clone() for t in st_a]
        st_g = [t.clone() for t in st_a]
        R.step_8bit_adam(u, *st_a, cfg, 1)
        blocks = OP.rank_blocks(o, rank, q)
        ref = OA.step_8bit_adam(OD.shard(o, exp, rank), y_ref, np.zeros(S, np.int8), np.zeros(S, np.uint8),
                                np.zeros(len(blocks), np.float32), np.zeros(len(blocks), np.float32), blocks,
                                OA.AdamCfg(), 1, out_bf16=(eb == 2))
        if eb == 2:
            # a6 + a7 + a8 in one kernel: bit identical to RS -> Adam
            R.reduce_scatter_adam_p2p(u, p2p, cfg, 1, state=st_f)
        yield
        check_adam_exact(ctx, f"{name} Adam", S, blocks, st_a, ref, cfg.lr)
        if eb == 2 and not all(_same_bytes(a, b) for a, b in zip(st_f, st_a)):
            ctx.fail(f"{name}: fused RS+Adam differs from RS then Adam")
        # the next AllGather: every rank's updated shard (oracle, within tolerance)
        if ctx.has_nccl and eb == 4:
            R.all_gather(u)
        else:
            R.all_gather_p2p(u, p2p)
        shards = yield from ctx.allgather(None)
        del shards
        refs = [OA.step_8bit_adam(OD.shard(o, exp, r), y_all[r], np.zeros(S, np.int8), np.zeros(S, np.uint8),
                                  np.zeros(len(OP.rank_blocks(o, r, q)), np.float32),
                                  np.zeros(len(OP.rank_blocks(o, r, q)), np.float32),
                                  OP.rank_blocks(o, r, q), OA.AdamCfg(), 1, out_bf16=(eb == 2))
                for r in range(world)]
        full_mask = np.zeros(world * S, bool)
        for l, e in zip(o.starts, o.numel):
            full_mask[l:l + e] = True
        if eb == 2:
            got = OD.bf16_to_f32(bf16_bits(param_full)).astype(np.float64)
            want = OD.bf16_to_f32(np.concatenate([s[5] for s in refs])).astype(np.float64)
        else:
            got = f32(param_full).astype(np.float64)
            want = np.concatenate([s[5] for s in refs]).astype(np.float64)
        p32 = np.abs(np.concatenate([s[0] for s in refs]).astype(np.float64))
        tol = 1e-5 * (p32 + 1e-3) + (2.0 ** -7 * p32 if eb == 2 else 0)
        if np.any((np.abs(got - want) > tol)[full_mask]):
            ctx.fail(f"{name}: post-Adam AllGather off by {np.abs(got - want)[full_mask].max():.3e}")
        if eb != 2:
            continue
        # a6 + a7 + a8 + a4 in one kernel: the pushed parameters equal the
        # unfused RS -> Adam -> AllGather result bit for bit
        pf_ref = param_full.clone()
        param_full.fill_(float("nan"))
        R.reduce_scatter_adam_gather_p2p(u, p2p, cfg, 1, state=st_g)
        yield
        fm = torch.from_numpy(full_mask).cuda()
        if not torch.equal(param_full.view(torch.int16)[fm], pf_ref.view(torch.int16)[fm]):
            ctx.fail(f"{name}: fused RS+Adam+AG parameters differ from RS -> Adam -> AG")
        if not all(_same_bytes(a, b) for a, b in zip(st_g, st_a)):
            ctx.fail(f"{name}: fused RS+Adam+AG state differs from RS then Adam")
        for t in range(2, 5):  # repeated steps: barriers re-arm, ranks keep agreeing
            R.reduce_scatter_adam_gather_p2p(u, p2p, cfg, t, state=st_g)
        yield
        h = int(param_full.view(torch.int16)[fm].to(torch.int64).sum().item())
        hs = yield from ctx.allgather(h)
        if len(set(hs)) != 1:
            ctx.fail(f"{name}: ranks disagree on the parameters after repeated fused steps")


def rs_random_case(ctx):
    """Random-normal bf16 gradients (non-dyadic sums): the p2p rank-order fp32
    sum equals the oracle's rank-order sum bit for bit; NCCL within the bound."""
    rank, world = ctx.rank, ctx.world
    es = [300001, 4097]
    o, c = _plans(es, [1, 1], world, 2)
    S = c.S
    g_np = [OD.to_bf16_rne(np.random.default_rng(100 + r).normal(0, 1e-2, world * S).astype(np.float32))
            for r in range(world)]
    for a, b in o.padding_intervals():
        for g in g_np:
            g[a:b] = 0
    grad_full = torch.from_numpy(g_np[rank].view(np.int16)).cuda().view(torch.bfloat16)
    grad_f32 = torch.empty(world * S, dtype=torch.float32, device="cuda")
    pf = torch.zeros(world * S, dtype=torch.bfloat16, device="cuda")
    u = R.Unit(c, rank, pf, grad_full, grad_f32, qblock=1, comm=ctx.comm)
    xs = [OD.grouped_cast_scale(o, g, True) for g in g_np]
    if ctx.has_nccl:
        R.reduce_scatter(u)
        yield
        yref = OD.reduce_scatter_f64(o, xs)[rank]
        absum = sum(np.abs(x[rank * S:(rank + 1) * S].astype(np.float64)) for x in xs)
        y = f32(grad_f32[rank * S:(rank + 1) * S]).astype(np.float64)
        if np.any(np.abs(y - yref) > 1e-6 * absum + 1e-30):
            ctx.fail("random-normal NCCL RS outside 1e-6 sum|x|")
    p2p = yield from ctx.p2p([grad_full])
    grad_f32.zero_()
    R.reduce_scatter_p2p(u, p2p)
    yield
    y32 = f32(grad_f32[rank * S:(rank + 1) * S])
    if not np.array_equal(y32.view(np.uint32), OD.reduce_scatter(o, xs)[rank].view(np.uint32)):
        ctx.fail("random-normal p2p RS differs from the rank-order oracle sum")


def channels_case(ctx):
    """rsdb_p2p_channel: AllGathers and ReduceScatters alternating over
    channels 0, 1 and 2 of one mapping (independent epochs and signal words;
    channel 2 with a 3-CTA budget) give the oracle's results: AG bit exact,
    RS = the rank-order sum bit for bit."""
    rank, world = ctx.rank, ctx.world
    es = [100003, 517, 2048 * 9]
    o, c = _plans(es, [1, 1, 1], world, 2)
    S = c.S
    pf = torch.zeros(world * S, dtype=torch.bfloat16, device="cuda")
    gf = torch.zeros(world * S, dtype=torch.bfloat16, device="cuda")
    g32 = torch.zeros(world * S, dtype=torch.float32, device="cuda")
    u = R.Unit(c, rank, pf, gf, g32, qblock=0, comm=ctx.comm)
    p2p = yield from ctx.p2p([pf, gf])
    chans = [p2p] * 3 if p2p is None else [p2p, p2p.channel(1), p2p.channel(2)]
    if p2p is not None:
        chans[2].set_max_ctas(3)  # a capped CTA budget (rsdb_p2p_set_max_ctas): same results
    ctx.keep = getattr(ctx, "keep", []) + chans
    for it in range(4):
        shards = [OD.to_bf16_rne(H.values_np(30 + it, 1 + r, 0, S, 12)) for r in range(world)]
        pf[rank * S:(rank + 1) * S].copy_(torch.from_numpy(shards[rank].view(np.int16)).view(torch.bfloat16))
        R.all_gather_p2p(u, chans[it % 3])
        yield
        if not np.array_equal(bf16_bits(pf), OD.all_gather(shards)):
            ctx.fail(f"AllGather on channel {it % 3} (iteration {it}) is not the concatenation")
        g_np = [OD.to_bf16_rne(OD.place_logical(o, H.values_np(40 + it, 16 + r, 0, o.E, 14)))
                for r in range(world)]
        gf.copy_(torch.from_numpy(g_np[rank].view(np.int16)).view(torch.bfloat16))
        R.reduce_scatter_p2p(u, chans[(it + 1) % 3])
        yield
        ref = OD.reduce_scatter(o, [OD.grouped_cast_scale(o, g, True) for g in g_np])[rank]
        y = f32(g32[rank * S:(rank + 1) * S])
        if not np.array_equal(y.view(np.uint32), ref.view(np.uint32)):
            ctx.fail(f"ReduceScatter on channel {(it + 1) % 3} (iteration {it}) != oracle")


def _fused_vs_unfused(ctx, tag, es, gs, seed, step, qblock=2048, qspec=None, oracle_check=True):
    """RS (p2p) -> 8-bit Adam -> AG (p2p) against the one fused kernel
    (bit identical, parameters and state), and the unfused result against
    the oracle (codes exact, params 1e-5)."""
    rank, world = ctx.rank, ctx.world
    o, c = _plans(es, gs, world, 2)
    S, E = c.S, sum(es)
    p_log = logical_params(seed, E)
    pf0 = place_gpu(c, p_log, torch.bfloat16)
    param_full = pf0.clone()
    grad_full = place_gpu(c, logical_grads(seed, rank, E), torch.bfloat16)
    grad_f32 = torch.zeros(world * S, dtype=torch.float32, device="cuda")
    u = R.Unit(c, rank, param_full, grad_full, grad_f32, qblock=qblock, comm=ctx.comm, qspec=qspec)
    nb = u.num_blocks
    exp = OD.place_logical(o, p_log.numpy())
    master = torch.from_numpy(OD.shard(o, exp, rank).copy()).cuda()
    st_a = [master] + _zero_state(S, nb)
    st_b = [t.clone() for t in st_a]
    st_c = [t.clone() for t in st_a]
    p2p = yield from ctx.p2p([param_full, grad_full])
    R.reduce_scatter_p2p(u, p2p)
    yield
    R.step_8bit_adam(u, *st_a, R.AdamConfig(), step)
    R.all_gather_p2p(u, p2p)
    yield
    pf_ref = param_full.clone()
    param_full.copy_(pf0)
    R.reduce_scatter_adam_p2p(u, p2p, R.AdamConfig(), step, state=st_c)  # without the AllGather
    yield
    R.reduce_scatter_adam_gather_p2p(u, p2p, R.AdamConfig(), step, state=st_b)
    yield
    mask = torch.zeros(world * S, dtype=torch.bool, device="cuda")
    for l, e in zip(c.starts, es):
        mask[l:l + e] = True
    if not torch.equal(param_full.view(torch.int16)[mask], pf_ref.view(torch.int16)[mask]):
        ctx.fail(f"{tag}: fused RS+Adam+AG parameters differ from RS -> Adam -> AG")
    for st, what in ((st_b, "RS+Adam+AG"), (st_c, "RS+Adam")):
        if not all(_same_bytes(a, b) for a, b in zip(st, st_a)):
            ctx.fail(f"{tag}: fused {what} state differs from RS then Adam")
    if oracle_check:
        if qspec is None:
            blocks = OP.rank_blocks(o, rank, qblock)
        else:
            blocks = OP.rank_tiles(o, rank, qspec)
        ys = []
        for r in range(world):
            src = OD.place_logical(o, logical_grads(seed, r, E).numpy())
            ys.append(OD.grouped_cast_scale(o, OD.to_bf16_rne(src), True))
        y = OD.reduce_scatter(o, ys)[rank]
        ref = OA.step_8bit_adam(OD.shard(o, exp, rank), y, np.zeros(S, np.int8), np.zeros(S, np.uint8),
                                np.zeros(len(blocks), np.float32), np.zeros(len(blocks), np.float32), blocks,
                                OA.AdamCfg(), step, out_bf16=True)
        check_adam_exact(ctx, tag, S, blocks, st_a, ref, R.AdamConfig().lr)


def ownerless_case(ctx):
    """One whole-tensor block on rank 0: ranks owning no block still launch the
    fused kernel (its barriers count every rank)."""
    es = [4096 * 8]
    yield from _fused_vs_unfused(ctx, "owner-less ranks", es, es, 9, 1, qblock=2048)


def tiles_case(ctx):
    """N2: 32x32 quantization tiles (the paper's 8-bit Adam setup) at
    32-row granularity through the fused kernel's strided peer-load path."""
    shapes = [(96, 64), (64, 40), (130,), (256, 96)]
    es = [int(np.prod(sh)) for sh in shapes]
    gs = [32 * sh[1] if len(sh) == 2 else e for sh, e in zip(shapes, es)]
    specs = [("tile", sh[1], 32, 32) if len(sh) == 2 else ("flat", e) for sh, e in zip(shapes, es)]
    yield from _fused_vs_unfused(ctx, "32x32 tiles", es, gs, 11, 2, qspec=specs)


def long_blocks_case(ctx):
    """Quantization blocks longer than 2048 elements through the fused kernels
    (two-pass path: the peers' gradients summed again in the second pass):
    4096-element flat blocks (with a ragged tail) and 128x128 tiles."""
    es = [4096 * 5 + 1000, 300, 4096 * 3]
    yield from _fused_vs_unfused(ctx, "4096-element blocks", es, [min(4096, e) for e in es], 13, 1,
                                 qblock=4096)
    shapes = [(256, 256), (128, 200), (384, 128)]
    es = [r * c for r, c in shapes]
    gs = [128 * c for _, c in shapes]
    specs = [("tile", c, 128, 128) for _, c in shapes]
    yield from _fused_vs_unfused(ctx, "128x128 tiles", es, gs, 15, 3, qspec=specs)


def fp8_case(ctx):
    """N2: FP8 128x128 block quantization fused with the AllGather (bit exact)."""
    rank, world = ctx.rank, ctx.world
    shapes = [(256, 384), (512, 128), (128, 200), (130, 128), (384, 64), (1024, 256)]
    es = [r * c for r, c in shapes]
    gs = [min(128, r) * c for r, c in shapes]
    o, c = _plans(es, gs, world, 1)
    specs = F.tile_specs([cc for _, cc in shapes])
    logical = np.random.default_rng(7).normal(0, 0.02, sum(es)).astype(np.float32)
    full = np.zeros(world * c.S, np.float32)
    off = 0
    for l, e in zip(c.starts, es):
        full[l:l + e] = logical[off:off + e]
        off += e
    exp_codes, exp_scales = F.quantize_all_gather(o, full, specs)
    master = torch.from_numpy(full[rank * c.S:(rank + 1) * c.S].copy()).cuda()
    codes = torch.full((world * c.S,), 0xAB, dtype=torch.uint8, device="cuda")
    scales = torch.full((len(exp_scales),), float("nan"), device="cuda")
    fu = R.Fp8Unit(c, specs, rank, master, codes, scales, comm=ctx.comm)
    p2p = yield from ctx.p2p([codes, scales])
    mask = np.zeros(world * c.S, bool)
    for l, e in zip(c.starts, es):
        mask[l:l + e] = True
    for it in range(3):  # repeated calls: epochs advance, barriers re-arm
        fu.quantize_all_gather(p2p)
        yield
        got = codes.cpu().numpy()
        if not (np.array_equal(got[mask], exp_codes[mask]) and np.all(got[~mask] == 0xAB)
                and np.array_equal(scales.cpu().numpy().view(np.uint32), exp_scales.view(np.uint32))):
            ctx.fail(f"FP8 quantize+AllGather mismatch (call {it})")
            break
    ctx.keep = getattr(ctx, "keep", []) + [fu]  # freed after the driver's last sync


# ---------------------------------------------------------------- K-slot ring
RING_UNITS = [[2048 * 20, 300, 2048 * 3], [2048 * 7 + 5, 2048 * 2], [2048 * 33]]


def ring_case(ctx, k=2):
    """Three units share K ring slots.  Forward: each unit acquires a slot, is
    rebound to it, gathers every rank's persistent shard into it (bit exact
    against the full parameters), releases it.  Backward (reverse order):
    acquire, gather again, write the gradients into the slot, fused
    ReduceScatter + 8-bit Adam writing the persistent shard, release.  Shards
    and optimizer states equal, bit for bit, the same step on dedicated
    buffers."""
    rank, world = ctx.rank, ctx.world
    q = 2048
    lays = [R.plan(es, [min(q, e) for e in es], world, elem_bytes=2) for es in RING_UNITS]
    olays = [OP.plan(es, [min(q, e) for e in es], world, OP.gcoll_elems(2)) for es in RING_UNITS]
    max_full = max(l.m * l.S for l in lays)
    dev = "cuda"
    slots = [(torch.zeros(max_full, dtype=torch.bfloat16, device=dev),
              torch.zeros(max_full, dtype=torch.bfloat16, device=dev),
              torch.zeros(max_full, dtype=torch.float32, device=dev)) for _ in range(k)]
    shard_off, acc = [], 0
    for l in lays:
        shard_off.append(acc)
        acc += (l.S + 7) // 8 * 8  # 16-B aligned shards in one arena
    shards = torch.zeros(max(acc, 8), dtype=torch.bfloat16, device=dev)
    units, refs, states, ref_states, fulls, grads = [], [], [], [], [], []
    for ui, (es, l, o) in enumerate(zip(RING_UNITS, lays, olays)):
        E, S = sum(es), l.S
        p_log = logical_params(20 + ui, E)
        full = place_gpu(l, p_log, torch.bfloat16)
        fulls.append(full)
        grads.append(place_gpu(l, logical_grads(20 + ui, rank, E), torch.bfloat16))
        shard = shards[shard_off[ui]:shard_off[ui] + S]
        shard.copy_(full[rank * S:(rank + 1) * S])
        u = R.Unit(l, rank, *slots[0], qblock=q, comm=ctx.comm)
        u.set_shard(shard)
        units.append(u)
        nb = u.num_blocks
        master = torch.from_numpy(OD.shard(o, OD.place_logical(o, p_log.numpy()), rank).copy()).to(dev)
        st = [master] + _zero_state(S, nb)
        states.append(st)
        ref_states.append([t.clone() for t in st])
        pf = full.clone()
        gf = grads[-1].clone()
        refs.append((R.Unit(l, rank, pf, gf, torch.zeros(world * S, device=dev), qblock=q, comm=ctx.comm), pf, gf))
    p2p_ring = yield from ctx.p2p([t for sl in slots for t in sl[:2]] + [shards])
    ref_p2p = []
    for ru, pf, gf in refs:
        ref_p2p.append((yield from ctx.p2p([pf, gf])))
    cfg = R.AdamConfig()
    for (ru, pf, gf), st, p in zip(refs, ref_states, ref_p2p):  # reference: dedicated buffers
        R.reduce_scatter_adam_p2p(ru, p, cfg, 1, state=st)
    yield
    ring = R.Ring(k)
    got = []
    for ui, u in enumerate(units):  # forward: gather, use, release
        s = ring.acquire()
        u.rebind(*slots[s])
        R.all_gather_shards_p2p(u, p2p_ring)
        l = lays[ui]
        got.append(slots[s][0][:l.m * l.S].clone())
        ring.release(s)
    for ui in reversed(range(len(units))):  # backward: gather, grads, RS+Adam into the shard
        u, l = units[ui], lays[ui]
        s = ring.acquire()
        u.rebind(*slots[s])
        R.all_gather_shards_p2p(u, p2p_ring)
        slots[s][1][:l.m * l.S].copy_(grads[ui])
        R.reduce_scatter_adam_p2p(u, p2p_ring, cfg, 1, state=states[ui])
        ring.release(s)
    yield
    for ui, g in enumerate(got):
        if not torch.equal(g.view(torch.int16), fulls[ui].view(torch.int16)):
            ctx.fail(f"ring unit {ui}: gathered shards differ from the full parameters")
    for ui, l in enumerate(lays):
        S = l.S
        shard = shards[shard_off[ui]:shard_off[ui] + S]
        if not torch.equal(shard.view(torch.int16), refs[ui][1][rank * S:(rank + 1) * S].view(torch.int16)):
            ctx.fail(f"ring unit {ui}: shard differs from the dedicated-buffer step")
        if not all(_same_bytes(a, b) for a, b in zip(states[ui], ref_states[ui])):
            ctx.fail(f"ring unit {ui}: optimizer state differs")
    ctx.keep = getattr(ctx, "keep", []) + [ring, units, refs]


# ---------------------------------------------------------------- N3 distributed Muon
MUON_SHAPES = [(24, 40), None, (40, 24), (16, 16), None, (96, 160), (160, 96), (1, 64)]
MUON_TOL = {"f32": 1e-4, "bf16": 3e-2}


def muon_case(ctx, shapes=MUON_SHAPES, seed=5, steps=2, precision="f32"):
    """`steps` Muon steps (Algorithm 2) vs oracle/muon.py (fp64): momentum
    rtol 1e-6, the orthogonalised update per piece within relative Frobenius
    1e-4 (fp32) / 3e-2 (bf16 tensor cores), skipped tensors and padding
    untouched, bf16 shard = RNE(master)."""
    rank, m = ctx.rank, ctx.world
    es = [s[0] * s[1] if s else 37 + i for i, s in enumerate(shapes)]
    lay = R.plan(es, [1] * len(es), m, elem_bytes=2)
    o = OP.plan(es, [1] * len(es), m, 8)
    assert list(lay.starts) == list(o.starts) and lay.S == o.S
    S = lay.S
    rng = np.random.default_rng(seed)
    full = []
    for scale in (0.02, 0.01, 0.01):  # master, momentum buffer, gradient
        f = np.zeros(m * S)
        for l, e in zip(lay.starts, es):
            f[l:l + e] = rng.normal(0, scale, e).astype(np.float32)
        full.append(f)
    sh = slice(rank * S, (rank + 1) * S)
    dev = lambda a: torch.from_numpy(a[sh].astype(np.float32)).cuda()  # noqa: E731
    master, buf, grad = dev(full[0]), dev(full[1]), dev(full[2])
    u = torch.zeros(S, device="cuda")
    param = torch.zeros(S, dtype=torch.bfloat16, device="cuda")
    mu = R.Muon(lay, shapes, rank, comm=ctx.comm, precision=precision)
    ws = torch.zeros(mu.workspace_bytes, dtype=torch.uint8, device="cuda")
    mu.bind(master, buf, grad, u, ws, param_bf16=param)
    p2p = yield from ctx.p2p([u, ws])
    if [mu.root(t) for t in range(len(shapes))] != MU.select_roots(o, shapes):
        ctx.fail("Muon: roots differ from the oracle's SelectRoot")
    ref_m, ref_b, ref_g = full
    prev_gpu = master.cpu().numpy().astype(np.float64)
    for step in range(steps):
        ref_m, ref_b, _, o_full = MU.muon_step_sharded(o, shapes, ref_m, ref_b, ref_g)
        mu.step(R.MuonConfig(), p2p)
        yield
        gm = master.cpu().numpy().astype(np.float64)
        gb = buf.cpu().numpy().astype(np.float64)
        if not np.allclose(gb, ref_b[sh], rtol=1e-6, atol=1e-9):
            ctx.fail(f"Muon step {step}: momentum buffer off by {np.abs(gb - ref_b[sh]).max():.3e}")
        for t, s in enumerate(shapes):
            a, b = max(lay.starts[t], rank * S), min(lay.starts[t] + es[t], (rank + 1) * S)
            if a >= b:
                continue
            loc = slice(a - rank * S, b - rank * S)
            if s is None:
                if not np.array_equal(gm[loc], prev_gpu[loc]):
                    ctx.fail(f"Muon tensor {t} (not a matrix) changed")
                continue
            coef = 0.02 * MU.shape_scale(*s)
            o_gpu = (prev_gpu[loc] - gm[loc]) / coef
            o_ref = o_full[a:b]
            err = np.linalg.norm(o_gpu - o_ref) / max(np.linalg.norm(o_ref), 1e-30)
            if err > MUON_TOL[precision]:
                ctx.fail(f"Muon {precision} step {step} tensor {t} {s}: o rel err {err:.3e}")
        pad = np.ones(S, bool)
        for l, e in zip(lay.starts, es):
            a, b = max(l, rank * S), min(l + e, (rank + 1) * S)
            if a < b:
                pad[a - rank * S:b - rank * S] = False
        if np.any(gm[pad] != 0):
            ctx.fail("Muon: padding written")
        # resync the oracle to the GPU state (multi-step: errors must not compound)
        ref_m = ref_m.copy()
        ref_m[sh] = gm
        full_gm = yield from ctx.allgather(gm)
        for r, g in enumerate(full_gm):
            ref_m[r * S:(r + 1) * S] = g
        prev_gpu = gm
    pb = param.view(torch.int16).cpu().numpy()
    rne = master.to(torch.bfloat16).view(torch.int16).cpu().numpy()
    touched = np.zeros(S, bool)
    for t, s in enumerate(shapes):
        a, b = max(lay.starts[t], rank * S), min(lay.starts[t] + es[t], (rank + 1) * S)
        if s is not None and a < b:
            touched[a - rank * S:b - rank * S] = True
    if not np.array_equal(pb[touched], rne[touched]):
        ctx.fail("Muon: bf16 shard != RNE(master)")
    ctx.keep = getattr(ctx, "keep", []) + [mu]


def all_cases():
    """(name, generator function, kwargs) in the order the workers run them."""
    return [
        ("units", units_case, {}),
        ("rs_random", rs_random_case, {}),
        ("channels", channels_case, {}),
        ("ownerless", ownerless_case, {}),
        ("tiles", tiles_case, {}),
        ("long_blocks", long_blocks_case, {}),
        ("fp8", fp8_case, {}),
        ("ring", ring_case, {}),
        ("muon_f32", muon_case, {"precision": "f32"}),
        ("muon_bf16", muon_case, {"precision": "bf16"}),
    ]
