#!/usr/bin/env python
"""N2 measurement: the paper's own 8-bit Adam setup -- 32x32 quantization
tiles with 32-row sharding granularity -- against the default
2048-element flat blocks, on the whole Llama-3.2-1B DBuffer (1 GPU, world 1).

Both DBuffers are built in one process and timed alternately with CUDA
events on one stream (db.step_8bit_adam = one optimizer launch over all 17
units).  Algorithmic bytes: 18 B per element + 16 B per block (absmax m, v
read and written), so the tile run is charged its 2x more absmax traffic
(1,024-element tiles vs 2,048-element blocks).  One JSON line.

  python scripts/bench_tiles.py [--reps 20] [--dry]     (--dry: host planning only)
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2602_22437_b200 as R  # noqa: E402
from synth import workloads as W  # noqa: E402

TILE = 32


def plans(mode):
    """(layouts, qspec per unit) for mode 'flat' (2048-element blocks, the
    bench default) or 'tile' (32-row granularity, 32x32 tiles on 2-D
    tensors, flat blocks on 1-D tensors)."""
    lays, qspec = [], []
    for u in W.llama32_1b().units:
        es = [t.numel for t in u.tensors]
        if mode == "flat":
            gs = [R.block_elems(t.shape, ("flat", 2048)) for t in u.tensors]
            sp = [("flat", min(2048, g)) for g in gs]
        else:
            gs = [R.block_elems(t.shape, ("rows", TILE)) if len(t.shape) == 2
                  else R.block_elems(t.shape, ("flat", 2048)) for t in u.tensors]
            sp = [("tile", t.shape[-1], TILE, TILE) if len(t.shape) == 2 else ("flat", min(2048, g))
                  for t, g in zip(u.tensors, gs)]
        lays.append(R.plan(es, gs, 1, elem_bytes=2))
        qspec.append(sp)
    return lays, qspec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--dry", action="store_true")
    args = ap.parse_args()
    modes = {m: plans(m) for m in ("flat", "tile")}
    info = {}
    for mode, (lays, qs) in modes.items():
        sizes, _ = R.arena_sizes(lays, 0, qspec=qs)
        nblk = sizes[R._c.RSDB_KIND_MABS] // 4
        info[mode] = {"elems": sum(l.E for l in lays), "padding": sum(l.padding for l in lays),
                      "arena_bytes": sum(sizes), "blocks_upper_bound": nblk}
    if args.dry:
        print(json.dumps({"dry": True, **info}))
        return

    import torch
    torch.cuda.set_device(0)
    comm = R.init_comm(0, 1, 0)
    st = torch.cuda.Stream()
    cfg = R.AdamConfig()
    dbs = {}
    for mode, (lays, qs) in modes.items():
        sizes, offs = R.arena_sizes(lays, 0, qspec=qs)
        arenas = [torch.zeros(max(1, n), dtype=torch.uint8, device="cuda") for n in sizes]
        g = torch.Generator(device="cuda").manual_seed(0)
        grad = arenas[R._c.RSDB_KIND_GRAD_F32].view(torch.float32)
        grad.normal_(0.0, 1e-3, generator=g)
        master = arenas[R._c.RSDB_KIND_MASTER].view(torch.float32)
        master.normal_(0.0, 2e-2, generator=g)
        db = R.DBuffer(lays, 0, arenas, comm=comm, qspec=qs)
        dbs[mode] = (db, arenas)
        info[mode]["blocks"] = db.num_blocks
    for mode, (db, _) in dbs.items():  # warm up (also fills the 8-bit states)
        for t in range(1, 4):
            db.step_8bit_adam(cfg, t, st)
    st.synchronize()
    ms = {m: [] for m in dbs}
    for r in range(args.reps):
        for mode, (db, _) in dbs.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            db.step_8bit_adam(cfg, 4 + r, st)
            e1.record(st)
            st.synchronize()
            ms[mode].append(e0.elapsed_time(e1))
    peak, src = __import__("bench").load_peaks()
    out = {"workload": "llama-3.2-1b DBuffer (17 units), world 1", "reps": args.reps, "peak_gbs": peak,
           "peak_source": src}
    for mode in dbs:
        t = sorted(ms[mode])[len(ms[mode]) // 2]
        byts = 18 * info[mode]["elems"] + 16 * info[mode]["blocks"]
        out[mode] = {**info[mode], "ms_p50": t, "gbs": byts / t / 1e6, "frac": byts / t / 1e6 / peak}
    out["tile_over_flat_time"] = out["tile"]["ms_p50"] / out["flat"]["ms_p50"]
    print(json.dumps(out), flush=True)
    comm.close()


if __name__ == "__main__":
    main()
