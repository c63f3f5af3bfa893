"""Extra measurements of the default `bench.py` run (its `extras` key), so the
round-end driver run carries every BASELINE config and every SURVEY §8(f) row
that has a kernel, not only the headline step:

  per_unit        (N>1) AllGather / ReduceScatter bus GB/s per FSDP unit of
                  config 2 (layer unit, root unit): BJ's metric as named
  kernels         the §8(a) kernels outside the fused step, on the bench's own
                  DBuffer: a6 cast/scale per unit, a8 unfused 8-bit Adam (one
                  launch), N2 dynamic-code-map Adam (one launch)
  tiles_32x32     N2: the paper's own 8-bit Adam setup (32x32 blocks,
                  32-row granularity) on the whole Llama-3.2-1B DBuffer
  muon_8b_layer   config 3 / N3: one distributed-Muon step (Alg. 2) over the
                  Llama-3-8B decoder layer, Newton-Schulz TFLOP/s
  fp8_allgather   N2 / config 4: the fused FP8 128x128 quantize + AllGather of
                  the DSV3 FFN unit (and the bf16 AllGather it replaces, N>1)
  dsv3_ragged_vs_rowwise  config 4: zero-copy RaggedShard AG/RS against the
                  FSDP2 row-wise layout's Copy-Out / Copy-In + collective
  bucket_sweep    config 5: padding and rank-chunk alignment of aligned ragged
                  vs even split (host), and (N>1) AllGather bus GB/s of both
  zero3_overlap   (N>1) N4: FSDP's reshard schedule (K=2 gathered slots, AG
                  before forward and before backward, prefetched on a copy
                  stream) under a synthetic compute stream: exposed comm time

Every timing is CUDA events on the launching stream, median of `reps`, max
over ranks.  Measurement only: parity lives in tests/ (only tests/ run the
oracle).  Each item is independent; an exception is recorded in the item
(`{"error": ...}`) and the next item runs.
"""
from __future__ import annotations

import json
import os
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HBM_SPEC_GBS = 8000.0
NVLINK_SPEC_GBS = 900.0


def _max(x, world):
    if world == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def _barrier(world):
    if world > 1:
        dist.barrier()


def timed(fn, reps, stream, world, warm=2):
    """Median ms per call of fn (launching on `stream`), max over ranks."""
    with torch.cuda.stream(stream):
        for _ in range(warm):
            fn()
    stream.synchronize()
    _barrier(world)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(reps)]
    with torch.cuda.stream(stream):
        for a, b in evs:
            a.record(stream)
            fn()
            b.record(stream)
    stream.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in evs)
    return _max(ms[len(ms) // 2], world)


def _peaks():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1590.0))
    except Exception:
        return 6650.0, 1590.0


def _run(name, fn, out):
    t0 = time.perf_counter()
    try:
        out[name] = fn()
    except Exception as e:  # recorded, not hidden: the item shows the error
        out[name] = {"error": f"{type(e).__name__}: {e}"}
    if isinstance(out[name], dict):
        out[name]["wall_s"] = round(time.perf_counter() - t0, 2)


# ---------------------------------------------------------------- per-unit collectives
def per_unit(R, ctx):
    """BJ metric as named: AG and RS bus GB/s per FSDP unit (nccl-tests
    convention, bus bytes = (m-1) S b per rank), p2p kernels over NVLink,
    on the bench DBuffer's first layer unit and its root unit."""
    db, p2p, st, world = ctx["db"], ctx["p2p"], ctx["stream"], ctx["world"]
    # the fixed cost inside every p2p collective: its start + done barriers
    res = {"barrier_pair_us": 1e3 * timed(lambda: p2p.barrier(st), ctx["reps"], st, world)}
    for name, idx in (("layer", 1), ("root", 0)):
        u = db.units[idx]
        lay = u.layout
        S, m = lay.S, lay.m
        t_ag = timed(lambda: R.all_gather_p2p(u, p2p, st), ctx["reps"], st, world)
        t_rs = timed(lambda: R.reduce_scatter_p2p(u, p2p, st), ctx["reps"], st, world)
        bus = (m - 1) * S * 2
        res[name] = {"S": S, "params": lay.E, "pad_ratio": lay.padding / max(1, lay.E),
                     "ag_goodput_gbs": lay.E * 2 / t_ag / 1e6, "rs_goodput_gbs": lay.E * 2 / t_rs / 1e6,
                     "ag_ms": t_ag, "rs_ms": t_rs,
                     "ag_bus_gbs": bus / t_ag / 1e6, "rs_bus_gbs": bus / t_rs / 1e6,
                     "ag_frac_of_900": bus / t_ag / 1e6 / NVLINK_SPEC_GBS,
                     "rs_frac_of_900": bus / t_rs / 1e6 / NVLINK_SPEC_GBS,
                     "rs_wire": "bf16 (cast + 1/m fused into the reduction)"}
    return res


# ---------------------------------------------------------------- standalone kernels on the bench DBuffer
def kernels(R, ctx):
    db, st, world, lays, cfg = ctx["db"], ctx["stream"], ctx["world"], ctx["lays"], ctx["cfg"]
    hbm, _ = _peaks()
    rank = ctx["rank"]
    n_el = n_blk = 0
    for lay in lays:
        b = lay.rank_blocks(rank, 2048)
        n_el += sum(n for _, n in b)
        n_blk += len(b)
    adam_bytes = 18 * n_el + 16 * n_blk
    t = [ctx["t"]]

    def adam():
        db.step_8bit_adam(cfg, t[0], st)
        t[0] += 1

    def adam_dyn():
        db.step_8bit_adam_dynamic(cfg, t[0], st)
        t[0] += 1

    out = {}
    ms = timed(adam, ctx["reps"], st, world)
    out["adam8_unfused"] = {"kernel": "adam8_tma_kernel", "ms": ms, "gbs": adam_bytes / ms / 1e6,
                            "frac": adam_bytes / ms / 1e6 / hbm, "bytes": "18 B/elem + 16 B/block"}
    ms = timed(adam_dyn, ctx["reps"], st, world)
    out["adam8_dynamic"] = {"kernel": "adam8_dyn_kernel", "ms": ms, "gbs": adam_bytes / ms / 1e6,
                            "frac": adam_bytes / ms / 1e6 / hbm, "bytes": "18 B/elem + 16 B/block"}
    cast_bytes = sum(l.m * l.S * 6 for l in lays)
    ms = timed(lambda: [R.unit_cast_scale(u, st) for u in db.units], ctx["reps"], st, world)
    out["cast_scale"] = {"kernel": "cast_scale_kernel", "launches": len(db.units), "ms": ms,
                         "gbs": cast_bytes / ms / 1e6, "frac": cast_bytes / ms / 1e6 / hbm,
                         "bytes": "6 B per element of m*S (bf16 in, fp32 out)"}
    return out


# ---------------------------------------------------------------- N2: 32x32 tiles
def tiles(R, ctx):
    from synth import workloads as W
    world, rank, comm, st, cfg = ctx["world"], ctx["rank"], ctx["comm"], ctx["stream"], ctx["cfg"]
    hbm, _ = _peaks()
    lays, qs = [], []
    for u in W.llama32_1b().units:
        es = [t.numel for t in u.tensors]
        gs = [R.block_elems(t.shape, ("rows", 32)) if len(t.shape) == 2
              else R.block_elems(t.shape, ("flat", 2048)) for t in u.tensors]
        sp = [("tile", t.shape[-1], 32, 32) if len(t.shape) == 2 else ("flat", min(2048, g))
              for t, g in zip(u.tensors, gs)]
        lays.append(R.plan(es, gs, world, elem_bytes=2))
        qs.append(sp)
    sizes, _ = R.arena_sizes(lays, rank, qspec=qs)
    arenas = [torch.zeros(max(1, n), dtype=torch.uint8, device="cuda") for n in sizes]
    g = torch.Generator(device="cuda").manual_seed(rank)
    arenas[R._c.RSDB_KIND_GRAD_F32].view(torch.float32).normal_(0.0, 1e-3, generator=g)
    arenas[R._c.RSDB_KIND_MASTER].view(torch.float32).normal_(0.0, 2e-2, generator=g)
    db = R.DBuffer(lays, rank, arenas, comm=comm, qspec=qs)
    n_el = sum(l.S for l in lays)  # upper bound: the owned elements (zero padding here)
    own = 0
    for l, q in zip(lays, qs):
        own += sum(r * c for _, r, c, _ in l.rank_tiles(rank, q))
    t = [1]

    def step():
        db.step_8bit_adam(cfg, t[0], st)
        t[0] += 1

    ms = timed(step, ctx["reps"], st, world, warm=3)
    nb = db.num_blocks
    byts = 18 * own + 16 * nb
    res = {"kernel": "adam8_pair_kernel (two 32x32 tiles per stage)", "tiles": nb, "elems": own, "shard_elems": n_el,
           "padding": sum(l.padding for l in lays), "ms": ms, "gbs": byts / ms / 1e6,
           "frac": byts / ms / 1e6 / hbm, "bytes": "18 B/elem + 16 B/tile"}
    db.close()
    del arenas
    torch.cuda.empty_cache()
    return res


# ---------------------------------------------------------------- config 3 / N3: distributed Muon
def muon(R, ctx):
    from synth import hashgen as H
    from synth import workloads as W
    world, rank, comm, st = ctx["world"], ctx["rank"], ctx["comm"], ctx["stream"]
    _, tc_peak = _peaks()
    unit = W.llama3_8b_layer(0)
    shapes = [t.shape if len(t.shape) == 2 else None for t in unit.tensors]
    es = [t.numel for t in unit.tensors]
    lay = R.plan(es, [1] * len(es), world, elem_bytes=2)
    S = lay.S
    mk = lambda s: H.values_torch(7, s, rank * S, S, 14, device="cuda")  # noqa: E731
    master, buf, grad = mk(1), mk(2), mk(3)
    u = torch.zeros(S, device="cuda")
    param = torch.zeros(S, dtype=torch.bfloat16, device="cuda")
    mu = R.Muon(lay, shapes, rank, comm=comm, precision="bf16")
    ws = torch.zeros(mu.workspace_bytes, dtype=torch.uint8, device="cuda")
    mu.bind(master, buf, grad, u, ws, param_bf16=param)
    p2p = R.P2P(comm, [u, ws]) if world > 1 else None
    reps = max(3, ctx["reps"] // 2)
    t_full = timed(lambda: mu.step(R.MuonConfig(), p2p, st), reps, st, world)
    t_zero = timed(lambda: mu.step(R.MuonConfig(ns_steps=0), p2p, st), reps, st, world)
    roots = [mu.root(i) for i in range(len(shapes))]
    load = [0] * world
    for i, s in enumerate(shapes):
        if s is not None:
            k, L = min(s), max(s)
            load[roots[i]] += 5 * (4 * k * k * L + 2 * k ** 3)
    t_ns = max(t_full - t_zero, 1e-6)
    tf = max(load) / (t_ns * 1e-3) / 1e12
    if p2p is not None:
        torch.cuda.synchronize()
        p2p.close()
    mu.close()
    # the tcgen05 GEMM alone on the layer's two big Newton-Schulz shapes
    gemm = {}
    for name, (M_, N_, K_) in (("W_Wt_4096x4096x14336", (4096, 4096, 14336)),
                               ("B_W_4096x14336x4096", (4096, 14336, 4096))):
        a_ = torch.randn(M_, K_, device="cuda").to(torch.bfloat16)
        b_ = torch.randn(N_, K_, device="cuda").to(torch.bfloat16)
        c_ = torch.empty(M_, N_, device="cuda", dtype=torch.bfloat16)
        ms = timed(lambda: R.ns_gemm_bf16(a_, b_, c_, stream=st), reps, st, 1)
        tg = 2 * M_ * N_ * K_ / (ms * 1e-3) / 1e12
        gemm[name] = {"ms": ms, "tflops": tg, "frac_of_measured_bf16": tg / tc_peak}
        del a_, b_, c_
    a_ = torch.randn(4096, 14336, device="cuda").to(torch.bfloat16)
    c_ = torch.empty(4096, 4096, device="cuda", dtype=torch.bfloat16)
    ms = timed(lambda: R.ns_gemm_bf16_sym(a_, a_, c_, stream=st), reps, st, 1)
    gemm["W_Wt_sym_4096x4096x14336"] = {
        "ms": ms, "effective_tflops": 2 * 4096 * 4096 * 14336 / (ms * 1e-3) / 1e12,
        "note": "symmetric product: upper-triangle tiles only (272 of 512), effective = full-product flop / time"}
    del a_, c_
    return {"workload": "llama-3-8b decoder layer, element-granularity RaggedShard, bf16 NS",
            "ns_gemm": gemm, "ns_kernel": "umma_gemm_kernel (tcgen05.mma + TMA + TMEM)",
            "matrices": sum(s is not None for s in shapes), "roots": roots,
            "step_ms": t_full, "step_without_ns_ms": t_zero, "ns_ms": t_ns,
            "ns_tflops_busiest_root": tf, "ns_frac_of_measured_bf16": tf / tc_peak,
            "peak_bf16_tflops": tc_peak}


# ---------------------------------------------------------------- N2: FP8 128x128 quantize + AllGather
def fp8(R, ctx):
    """DeepSeek-V3 FFN unit (27 matrices, 128-row granularity, 1-byte
    elements): the fused FP8 quantize + AllGather kernel against
    the bf16 AllGather of the same weights."""
    from synth import hashgen as H
    from synth import workloads as W
    world, rank, comm, st = ctx["world"], ctx["rank"], ctx["comm"], ctx["stream"]
    hbm, _ = _peaks()
    unit = W.dsv3_ffn_fp8_unit()
    shapes = [t.shape for t in unit.tensors]
    es = [t.numel for t in unit.tensors]
    gs = [128 * c for _, c in shapes]
    specs = [("tile", c, 128, 128) for _, c in shapes]
    lay = R.plan(es, gs, world, elem_bytes=1)
    S = lay.S
    master = H.values_torch(3, H.STREAM_PARAM, rank * S, S, 12, device="cuda")
    codes = torch.zeros(world * S, dtype=torch.uint8, device="cuda")
    u0 = R.Fp8Unit(lay, specs, rank, master, codes, torch.empty(1, device="cuda"), comm=comm)
    ntiles = u0.num_tiles
    u0.close()
    scales = torch.zeros(max(1, ntiles), dtype=torch.float32, device="cuda")
    p2p = R.P2P(comm, [codes, scales]) if world > 1 else None
    fu = R.Fp8Unit(lay, specs, rank, master, codes, scales, comm=comm)
    t_fp8 = timed(lambda: fu.quantize_all_gather(p2p, st), ctx["reps"], st, world)
    out = {"params": sum(es), "tiles": ntiles, "S": S, "fp8_quant_ag_ms": t_fp8,
           "kernel": "fp8_quant_ag_kernel", "hbm_gbs": 5 * S / t_fp8 / 1e6,
           "hbm_frac": 5 * S / t_fp8 / 1e6 / hbm, "hbm_bytes": "4 B read + 1 B written per owned element"}
    fu.close()
    if p2p is not None:
        torch.cuda.synchronize()
        p2p.close()
        wire = (world - 1) * S
        out["fp8_wire_gbs"] = wire / t_fp8 / 1e6
        lay16 = R.plan(es, gs, world, elem_bytes=2)
        pf = torch.zeros(world * lay16.S, dtype=torch.bfloat16, device="cuda")
        gf = torch.zeros(world * lay16.S, dtype=torch.bfloat16, device="cuda")
        g32 = torch.zeros(8, dtype=torch.float32, device="cuda")
        u16 = R.Unit(lay16, rank, pf, gf, g32.repeat(1), qblock=0, comm=comm)
        p16 = R.P2P(comm, [pf])
        t16 = timed(lambda: R.all_gather_p2p(u16, p16, st), ctx["reps"], st, world)
        torch.cuda.synchronize()
        p16.close()
        out.update({"bf16_ag_ms": t16, "speedup_vs_bf16_ag": t16 / t_fp8,
                    "bf16_ag_wire_gbs": (world - 1) * lay16.S * 2 / t16 / 1e6})
    return out


# ---------------------------------------------------------------- config 4: DSV3 ragged vs row-wise
def dsv3(R, ctx):
    from synth import workloads as W
    world, rank, comm, st, p2p_main = ctx["world"], ctx["rank"], ctx["comm"], ctx["stream"], ctx["p2p"]
    m = world
    unit = W.dsv3_moe_unit()
    es = [t.numel for t in unit.tensors]
    E = sum(es)
    reps = max(3, ctx["reps"] // 2)
    out = {"params": E, "tensors": len(es)}
    # ragged: planner layout, 128-row blocks, zero-copy views; AG in place, RS
    # = the fused cast + scale + reduction (p2p kernels; at m = 1 the group op)
    gs = [R.block_elems(t.shape, t.gran) for t in unit.tensors]
    lay = R.plan(es, gs, m)
    S = lay.S
    pf = torch.zeros(m * S, dtype=torch.bfloat16, device="cuda")
    gf = torch.randn(m * S, device="cuda").to(torch.bfloat16)
    g32 = torch.zeros(m * S, dtype=torch.float32, device="cuda")
    u = R.Unit(lay, rank, pf, gf, g32, qblock=0, comm=comm)
    p2p = R.P2P(comm, [pf, gf]) if m > 1 else None
    t_ag = timed(lambda: R.all_gather_p2p(u, p2p, st), reps, st, world)
    t_rs = timed(lambda: R.reduce_scatter_p2p(u, p2p, st), reps, st, world)
    out["ragged"] = {"S": S, "pad_ratio": lay.padding / E, "ag_ms": t_ag, "rs_ms": t_rs,
                     "copy_ms": 0.0, "path": "p2p kernels, zero-copy views"}
    if p2p is not None:
        torch.cuda.synchronize()
        p2p.close()
    del u, pf, gf, g32
    # row-wise (FSDP2 Shard(0)): NCCL AllGather + Copy-Out; Copy-In (cast, 1/m) + NCCL RS
    shard_rows, cols, off = [], [], []
    P = 0
    for t in unit.tensors:
        rows = t.shape[0]
        c = t.numel // rows
        sr = -(-rows // m)
        shard_rows.append(sr)
        cols.append(c)
        off.append(P)
        P += sr * c
    P = -(-P // 8) * 8
    flat = torch.zeros(m * P, dtype=torch.bfloat16, device="cuda")
    params = [torch.zeros(t.numel, dtype=torch.bfloat16, device="cuda") for t in unit.tensors]
    grads = [torch.randn(t.numel, device="cuda").to(torch.bfloat16) for t in unit.tensors]
    rsbuf = torch.zeros(m * P, dtype=torch.float32, device="cuda")
    seg_out, seg_in = [], []
    for ti, t in enumerate(unit.tensors):
        rows = t.shape[0]
        for r in range(m):
            r0 = r * shard_rows[ti]
            n_rows = max(0, min(shard_rows[ti], rows - r0))
            if n_rows == 0:
                continue
            n = n_rows * cols[ti]
            seg_out.append((flat.data_ptr() + 2 * (r * P + off[ti]),
                            params[ti].data_ptr() + 2 * r0 * cols[ti], n))
            seg_in.append((grads[ti].data_ptr() + 2 * r0 * cols[ti],
                           rsbuf.data_ptr() + 4 * (r * P + off[ti]), n))
    copy_out = R.CopyPlan(seg_out, R.RSDB_BF16, R.RSDB_BF16, 1.0)
    copy_in = R.CopyPlan(seg_in, R.RSDB_BF16, R.RSDB_F32, 1.0 / m)
    lay_rw = R.layout_from_starts([m * P], [1], m, P, [0])
    u_rw = R.Unit(lay_rw, rank, flat, torch.zeros(m * P, dtype=torch.bfloat16, device="cuda"),
                  rsbuf, qblock=0, comm=comm)
    t_co = timed(lambda: copy_out.run(st), reps, st, world)
    t_ci = timed(lambda: copy_in.run(st), reps, st, world)
    row = {"S": P, "pad_ratio": (m * P - E) / E, "copy_out_ms": t_co, "copy_in_ms": t_ci,
           "copy_segments": len(seg_out), "copy_kernel": "copy_seg_kernel",
           "copy_gbs": (2 + 2) * E / t_co / 1e6}
    if m > 1:
        t_agn = timed(lambda: R.all_gather(u_rw, st), reps, st, world)
        t_rsn = timed(lambda: R.unit_reduce_scatter_f32(u_rw, st), reps, st, world)
        row.update({"nccl_ag_ms": t_agn, "nccl_rs_ms": t_rsn, "ag_ms": t_agn + t_co,
                    "rs_ms": t_ci + t_rsn,
                    "copy_share_ag": t_co / (t_agn + t_co), "copy_share_rs": t_ci / (t_ci + t_rsn)})
    else:
        row.update({"ag_ms": t_co, "rs_ms": t_ci,
                    "note": "m = 1: the collectives are the identity; what remains is the "
                            "interleaved Copy-Out / Copy-In the row-wise layout needs"})
    out["rowwise"] = row
    out["ragged_over_rowwise_ag+rs"] = ((out["ragged"]["ag_ms"] + out["ragged"]["rs_ms"]) /
                                         (row["ag_ms"] + row["rs_ms"]))
    del u_rw, copy_in, copy_out
    return out


# ---------------------------------------------------------------- config 5: bucket sweep
def bucket_sweep(R, ctx):
    from synth import workloads as W
    world, rank, comm, st = ctx["world"], ctx["rank"], ctx["comm"], ctx["stream"]
    rows = []
    for mb in (1, 4, 16, 64, 256, 1024):
        u = W.bucket(mb)
        es = [t.numel for t in u.tensors]
        E = sum(es)
        for m in (2, 4, 8):
            lay = R.plan(es, [1] * len(es), m, elem_bytes=2)
            s_even = -(-E // m)
            rows.append({"mb": mb, "m": m, "E": E, "S_ragged": lay.S, "S_even": s_even,
                         "pad_ragged": lay.padding / E, "pad_even": (m * s_even - E) / E,
                         "ragged_chunk_align_bytes": 16 if (lay.S * 2) % 16 == 0 else 2,
                         "even_chunk_align_bytes": 2 if s_even % 2 else (4 if s_even % 4 else 8)})
    res = {"host": rows}
    if world > 1:
        timed_rows = []
        for mb in (16, 256, 1024):
            u = W.bucket(mb)
            es = [t.numel for t in u.tensors]
            E = sum(es)
            for name in ("ragged", "even"):
                if name == "ragged":
                    lay = R.plan(es, [1] * len(es), world, elem_bytes=2)
                else:  # FSDP1 flat even split: tensors back to back, S = ceil(E/m) (2-B aligned chunks)
                    S = -(-E // world)
                    starts, acc = [], 0
                    for e in es:
                        starts.append(acc)
                        acc += e
                    lay = R.layout_from_starts(es, [1] * len(es), world, S, starts, require_gcoll=False)
                S = lay.S
                pf = torch.zeros(world * S + 64, dtype=torch.bfloat16, device="cuda")
                gf = torch.zeros(world * S + 64, dtype=torch.bfloat16, device="cuda")
                g32 = torch.zeros(world * S + 64, dtype=torch.float32, device="cuda")
                un = R.Unit(lay, rank, pf, gf, g32, qblock=0, comm=comm)
                t = timed(lambda: R.all_gather(un, st), 5, st, world)
                timed_rows.append({"mb": mb, "layout": name, "S": S, "nccl_ag_ms": t,
                                   "ag_bus_gbs": (world - 1) * S * 2 / t / 1e6})
                del un, pf, gf, g32
        res["nccl_allgather"] = timed_rows
    return res


# ---------------------------------------------------------------- N4: ZeRO-3 reshard schedule + overlap
def zero3(R, ctx, tokens=4096):
    """FSDP's reshard schedule on the bench workload with K = 2 gathered slots:
    forward: AG(u+1) on a copy-engine stream while a synthetic forward GEMM of
    unit u runs on the compute stream; backward (reverse): AG(u-1) prefetched
    the same way, the synthetic backward GEMMs (2x forward) of unit u, then
    the fused RS + 8-bit Adam of unit u.  The synthetic compute is a bf16
    GEMM of tokens x 2048 x (params/2048) per unit (2 * params * tokens flop
    forward) -- plumbing standing in for the model (out of scope).  Reports
    the step time with and without the collectives and the exposed fraction."""
    from synth import hashgen as H
    import bench
    world, rank, comm = ctx["world"], ctx["rank"], ctx["comm"]
    units = bench.build_units(16)
    lays = []
    for u in units:
        es = [t.numel for t in u.tensors]
        gs = [R.block_elems(t.shape, t.gran) for t in u.tensors]
        lays.append(R.plan(es, gs, world, elem_bytes=2))
    K = 2
    max_full = max(l.m * l.S for l in lays)
    slots = [(torch.zeros(max_full, dtype=torch.bfloat16, device="cuda"),
              torch.zeros(max_full, dtype=torch.bfloat16, device="cuda"),
              torch.zeros(8, dtype=torch.float32, device="cuda")) for _ in range(K)]
    offs, acc = [], 0
    for l in lays:
        offs.append(acc)
        acc += (l.S + 7) // 8 * 8
    shards = torch.zeros(acc, dtype=torch.bfloat16, device="cuda")
    rus, states = [], []
    for ui, l in enumerate(lays):
        S = l.S
        shard = shards[offs[ui]:offs[ui] + S]
        shard.copy_(H.values_torch(ui, H.STREAM_PARAM, rank * S, S, 12, device="cuda").to(torch.bfloat16))
        ru = R.Unit(l, rank, slots[0][0], slots[0][1], slots[0][2].repeat(1), qblock=2048, comm=comm)
        ru.set_shard(shard)
        nb = ru.num_blocks
        states.append([H.values_torch(ui, H.STREAM_PARAM, rank * S, S, 12, device="cuda"),
                       H.codes_torch(ui, H.STREAM_MCODE, rank * S, S, True, device="cuda"),
                       H.codes_torch(ui, H.STREAM_VCODE, rank * S, S, False, device="cuda"),
                       H.absmax_torch(ui, H.STREAM_ABSM, rank * 10 ** 7, max(nb, 1), 14, device="cuda"),
                       H.absmax_torch(ui, H.STREAM_ABSV, rank * 10 ** 7, max(nb, 1), 22, device="cuda")])
        rus.append(ru)
    for sl in slots:
        sl[1].copy_(H.values_torch(0, H.STREAM_GRAD0 + rank, 0, max_full, 14, device="cuda").to(torch.bfloat16))
    p2p = R.P2P(comm, [t for sl in slots for t in sl[:2]] + [shards])
    p_ag = p2p.channel(1)  # the prefetched AllGathers overlap the RS+Adam kernels: own channel
    cfg = R.AdamConfig()
    comp, cstream, rstream = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    x = torch.randn(tokens, 2048, device="cuda", dtype=torch.bfloat16)
    wts = [torch.randn(2048, max(1, l.E // 2048), device="cuda", dtype=torch.bfloat16) * 0.01
           for l in lays]
    n = len(rus)
    ev_g = [torch.cuda.Event() for _ in range(n)]    # unit gathered (forward / backward)
    ev_free = [torch.cuda.Event() for _ in range(K)]  # slot no longer read by compute
    used = [False] * K
    t = [1]

    def gather(i, s, with_comm):
        cstream.wait_event(ev_free[s]) if used[s] else None
        with torch.cuda.stream(cstream):
            if with_comm:
                rus[i].rebind(*slots[s])
                R.all_gather_shards_p2p(rus[i], p_ag, cstream)
            ev_g[i].record(cstream)

    overlap_rs = [False]

    def step(with_comm=True, with_compute=True):
        seq = list(range(n)) + list(reversed(range(n)))
        slot = {}
        # prefetch the first unit
        slot[(0, 0)] = 0
        gather(seq[0], 0, with_comm)
        for j, i in enumerate(seq):
            s = j % K
            if j + 1 < len(seq):  # prefetch the next unit's gather into the other slot
                gather(seq[j + 1], (j + 1) % K, with_comm)
            comp.wait_event(ev_g[i])
            with torch.cuda.stream(comp):
                if with_compute:
                    y = x @ wts[i]
                    if j >= n:  # backward: 2x the forward flop
                        y = x @ wts[i]
                        y = x @ wts[i]
                if j >= n and with_comm and not overlap_rs[0]:  # serial: RS + Adam on the compute stream
                    rus[i].rebind(*slots[s])
                    R.reduce_scatter_adam_p2p(rus[i], p2p, cfg, t[0], state=states[i], stream=comp)
                if not (j >= n and with_comm and overlap_rs[0]):
                    ev_free[s].record(comp)
            if j >= n and with_comm and overlap_rs[0]:  # RS + Adam overlapping the next unit's backward
                rstream.wait_stream(comp)
                with torch.cuda.stream(rstream):
                    rus[i].rebind(*slots[s])
                    R.reduce_scatter_adam_p2p(rus[i], p2p, cfg, t[0], state=states[i], stream=rstream)
                    ev_free[s].record(rstream)
            used[s] = True
        t[0] += 1

    def run(reps, **kw):
        for _ in range(2):
            step(**kw)
        torch.cuda.synchronize()
        _barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        for _ in range(reps):
            step(**kw)
        comp.wait_stream(cstream)
        comp.wait_stream(rstream)
        e1.record(comp)
        torch.cuda.synchronize()
        return _max(e0.elapsed_time(e1) / reps, world)

    reps = 5
    t_full = run(reps)
    overlap_rs[0] = True
    t_full_ov = run(reps)
    p2p.set_max_ctas(32)  # the overlapped RS + Adam on a 32-CTA budget, the rest of the SMs to compute
    t_full_cap = run(reps)
    p2p.set_max_ctas(0)
    overlap_rs[0] = False
    t_comp = run(reps, with_comm=False)
    t_comm = run(reps, with_compute=False)
    torch.cuda.synchronize()
    p_ag.close()
    p2p.close()
    exposed = max(0.0, t_full - t_comp)
    flop = sum(2 * tokens * 2048 * max(1, l.E // 2048) for l in lays) * 4  # fwd 1x + bwd 3x GEMMs
    return {"schedule": "reshard (ZeRO-3): K=2 slots, AG before forward and before backward, "
                        "prefetched on a copy-engine stream (p2p channel 1); fused RS+Adam per unit after the "
                        "unit's backward on the compute stream (step_ms) or on its own stream overlapping the "
                        "next unit's backward (step_ms_rs_overlapped)",
            "step_ms_rs_overlapped": t_full_ov,
            "step_ms_rs_overlapped_32cta": t_full_cap,
            "exposed_frac_rs_overlapped_32cta": max(0.0, t_full_cap - t_comp) / max(t_comm, 1e-9),
            "exposed_frac_rs_overlapped": max(0.0, t_full_ov - t_comp) / max(t_comm, 1e-9),
            "tokens_per_rank": tokens, "synthetic_gemm_tflop": flop / 1e12,
            "synthetic_gemm_tflops": flop / (t_comp * 1e-3) / 1e12,
            "step_ms": t_full, "compute_only_ms": t_comp, "comm_only_ms": t_comm,
            "exposed_comm_ms": exposed, "exposed_frac_of_comm": exposed / max(t_comm, 1e-9),
            "gathered_bytes_per_rank": K * max_full * 2 * 2,
            "resident_gathered_bytes_per_rank": sum(l.m * l.S for l in lays) * 2 * 2}


# ---------------------------------------------------------------- N4: allocation dynamics
def memory_replay(R, ctx, m=8, steps=3, lag_us=200):
    """Replays the buffer allocations of training steps of the bench workload
    (Llama-3.2-1B, 17 units, planned for an FSDP group of m = 8; one GPU holds
    one rank's buffers) through PyTorch's caching allocator under four
    policies and reports peak RESERVED memory:

      dbuffer       DBuffer batched allocation: per unit and pass ONE
                    allocation holding the unit's gathered parameters (m S
                    bf16), gradients (m S bf16) and fp32 reduce buffer (m S),
                    freed deterministically -- the comm stream waits for the
                    compute stream before its next allocation (no record_stream);
      ring_k2       this library's K-slot ring: K = 2 such batched slots sized
                    for the largest unit, allocated once;
      per_param     FSDP2-style eager per-parameter allocation: the AllGather
                    output (m S bf16) on the comm stream, the unsharded
                    parameters one tensor each (Copy-Out), in backward one
                    gradient tensor each, the fp32 ReduceScatter input (m S,
                    Copy-In) and output (S); stream order kept with events;
      record_stream FSDP1 / DeepSpeed-style flat buffers allocated on the
                    comm stream and released through Tensor.record_stream.

    Compute is a `lag_us` sleep kernel per unit and pass, so the CPU runs
    ahead of the GPU as in training.  Only the FSDP buffers are replayed (no
    activations): the paper's 16-30 % is on whole training steps."""
    import gc
    world = ctx["world"]
    if world > 1:
        return {"skipped": "single-GPU replay (run at N = 1)"}
    units = __import__("bench").build_units(16)
    sizes = []
    for u in units:
        es = [t.numel for t in u.tensors]
        gs = [R.block_elems(t.shape, t.gran) for t in u.tensors]
        lay = R.plan(es, gs, m, elem_bytes=2)
        sizes.append((lay.S, es))
    dev = torch.device("cuda")
    comp, comm_st = torch.cuda.Stream(), torch.cuda.Stream()
    cycles = int(lag_us * 1.9e3)

    def run(policy):
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_reserved()
        base_alloc = torch.cuda.memory_allocated()
        keep = []
        if policy == "ring_k2":
            mx = max(m * S for S, _ in sizes)
            keep = [torch.empty(8 * mx, dtype=torch.uint8, device=dev) for _ in range(2)]
        for _ in range(steps):
            for phase in ("fwd", "bwd"):
                order = range(len(sizes)) if phase == "fwd" else reversed(range(len(sizes)))
                for ui in order:
                    S, es = sizes[ui]
                    if policy == "ring_k2":
                        with torch.cuda.stream(comp):
                            torch.cuda._sleep(cycles)
                        continue
                    with torch.cuda.stream(comm_st):
                        comm_st.wait_stream(comp)  # explicit order: reuse only after compute is done
                        if policy == "dbuffer":
                            buf = torch.empty(8 * m * S, dtype=torch.uint8, device=dev)  # one batched block
                            buf[:2 * m * S].zero_()
                        else:
                            ag = torch.empty(m * S, dtype=torch.bfloat16, device=dev)
                            ag.zero_()
                    ev = torch.cuda.Event()
                    ev.record(comm_st)
                    comp.wait_event(ev)
                    with torch.cuda.stream(comp):
                        if policy == "per_param":
                            params = [torch.empty(e, dtype=torch.bfloat16, device=dev) for e in es]
                            params[0].zero_()
                        elif policy == "record_stream":
                            ag.record_stream(comp)
                        torch.cuda._sleep(cycles)
                        if phase == "bwd":
                            if policy == "per_param":
                                grads = [torch.empty(e, dtype=torch.bfloat16, device=dev) for e in es]
                                rs_in = torch.empty(m * S, dtype=torch.float32, device=dev)
                                rs_in.zero_()
                            elif policy == "record_stream":
                                grads = [torch.empty(m * S, dtype=torch.bfloat16, device=dev)]
                            ev2 = torch.cuda.Event()
                            ev2.record(comp)
                    if phase == "bwd":
                        with torch.cuda.stream(comm_st):
                            comm_st.wait_event(ev2)
                            if policy == "per_param":
                                rs_out = torch.empty(S, dtype=torch.float32, device=dev)
                                rs_out.zero_()
                                ev3 = torch.cuda.Event()
                                ev3.record(comm_st)
                                comp.wait_event(ev3)
                                del rs_out, rs_in, grads
                            elif policy == "record_stream":
                                rs = torch.empty(m * S, dtype=torch.float32, device=dev)
                                rs.zero_()
                                grads[0].record_stream(comm_st)
                                del rs, grads
                            else:
                                buf[2 * m * S:].zero_()  # the gradient + fp32 reduce parts
                    if policy == "per_param":
                        del params
                    if policy == "dbuffer":
                        del buf
                    else:
                        del ag
        torch.cuda.synchronize()
        out = {"peak_reserved_bytes": torch.cuda.max_memory_reserved() - base,
               "peak_allocated_bytes": torch.cuda.max_memory_allocated() - base_alloc}
        del keep
        return out

    res = {p: run(p) for p in ("dbuffer", "ring_k2", "per_param", "record_stream")}
    d = res["dbuffer"]["peak_reserved_bytes"]
    for p in ("ring_k2", "per_param", "record_stream"):
        res[p]["reserved_vs_dbuffer"] = res[p]["peak_reserved_bytes"] / max(1, d)
    res["workload"] = f"llama-3.2-1b FSDP buffers, m = {m} (one rank), {steps} steps, {lag_us} us compute per unit-pass"
    torch.cuda.empty_cache()
    return res


# ---------------------------------------------------------------- the e2e path's roofline: PCIe
def pcie(R, ctx, mb=512, reps=5):
    """Host <-> device copy rates from pinned memory (the bound of `e2e`,
    which moves every rank's bf16 gradients in and its shard out per step):
    H2D alone, D2H alone, both at once on two streams, and with the copies
    split over two streams per direction."""
    st = ctx["stream"]
    n = mb << 20
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
    s2 = torch.cuda.Stream()

    def rate(fn):
        fn()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(st)
        st.wait_event(t0)
        for _ in range(reps):
            fn()
        s2.wait_stream(st)
        st.wait_stream(s2)
        t1.record(st)
        torch.cuda.synchronize()
        return t0.elapsed_time(t1) / reps

    def h2d():
        with torch.cuda.stream(st):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(st):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        s2.wait_stream(st)
        with torch.cuda.stream(st):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        st.wait_stream(s2)

    t_in, t_out, t_both = rate(h2d), rate(d2h), rate(both)
    return {"bytes_each_way": n, "h2d_gbs": n / t_in / 1e6, "d2h_gbs": n / t_out / 1e6,
            "bidirectional_gbs_each_way": n / t_both / 1e6,
            "note": "pinned host memory, cudaMemcpyAsync; the e2e step is bound by the bidirectional rate"}


def run_all(R, ctx, which=None):
    """ctx: rank, world, comm, stream, db, lays, cfg, t, p2p, reps."""
    out = {}
    items = [("kernels", kernels), ("tiles_32x32", tiles), ("muon_8b_layer", muon),
             ("fp8_allgather", fp8), ("dsv3_ragged_vs_rowwise", dsv3), ("bucket_sweep", bucket_sweep),
             ("memory_replay", memory_replay), ("pcie", pcie)]
    if ctx["world"] > 1:
        items = [("per_unit", per_unit)] + items + [("zero3_overlap", zero3)]
    for name, fn in items:
        if which is None or name in which:
            _run(name, lambda fn=fn: fn(R, ctx), out)
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
    return out
