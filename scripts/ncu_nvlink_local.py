#!/usr/bin/env python
"""NVLink counter evidence for the N > 1 fused step ("NVLink
GB/s backed by captures").  ONE process drives N GPUs as N logical ranks
(rsdb_comm_create_local / rsdb_p2p_create_local, one rank per device, peer
access over NVLink) running the bench's default step -- the fused
ReduceScatter + 8-bit Adam + AllGather kernel over the Llama-3.2-1B DBuffer.
Every step launches the ranks' kernels from rank N-1 down to rank 0, so under

  ncu --devices 0 -k regex:rs_adam --metrics nvlrx__bytes.sum,nvltx__bytes.sum,...

the profiled launch (rank 0, synchronous under ncu) starts after its peers'
kernels are already running and its barriers complete.  Without ncu it
prints per-step CUDA-event times of rank 0's stream and the algorithmic wire
bytes per rank, so the counters can be compared with them.

  CUDA_MODULE_LOADING=EAGER python scripts/ncu_nvlink_local.py [--gpus 2] [--steps 5]

(EAGER: a lazily loaded kernel's module load can wait for a context that a
peer's barrier kernel keeps busy.)
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_22437_b200 as R  # noqa: E402


def log(msg):
    print(f"[ncu_nvlink_local] {msg}", file=sys.stderr, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--mode", choices=["fused", "noag", "rs"], default="fused",
                    help="fused: RS + Adam + AG pushes (the bench step); noag: RS + Adam (peer "
                         "loads only); rs: the standalone p2p ReduceScatter kernel per unit")
    args = ap.parse_args()
    n = args.gpus
    units = bench.build_units(16)
    comms, ctx = [], []
    for r in range(n):
        with torch.cuda.device(r):
            c = R.Comm.local(n, r)
            comms.append(c)
            lays, db, arenas, views, _, _ = bench.setup(r, n, r, units, c)
            ctx.append((lays, db, arenas, torch.cuda.Stream(device=r)))
        log(f"rank {r} set up on cuda:{r}")
    p2ps = R.P2P.local_group(comms, [[a[0], a[1]] for _, _, a, _ in ctx])
    for p in p2ps:
        p.set_timeout(20.0)
    log("p2p mapped")
    cfg = R.AdamConfig()
    order = list(reversed(range(n)))  # rank 0 last: its (profiled) launch finds the peers running
    for r in order:
        lays, db, _, st = ctx[r]
        with torch.cuda.device(r):
            for u in db.units:
                R.all_gather_p2p(u, p2ps[r], st)
    for r in range(n):
        torch.cuda.synchronize(r)
    for p in p2ps:
        p.check()
    log("first AllGather done")
    ev = []
    for t in range(1, args.steps + 1):
        for r in order:
            lays, db, _, st = ctx[r]
            with torch.cuda.device(r):
                if r == 0:
                    a = torch.cuda.Event(enable_timing=True)
                    a.record(st)
                if args.mode == "fused":
                    db.reduce_scatter_adam_gather(cfg, t, p2ps[r], st)
                elif args.mode == "noag":
                    db.reduce_scatter_adam(cfg, t, p2ps[r], st)
                else:
                    for u in reversed(db.units):
                        R.reduce_scatter_p2p(u, p2ps[r], st)
                if r == 0:
                    b = torch.cuda.Event(enable_timing=True)
                    b.record(st)
                    ev.append((a, b))
    for r in range(n):
        torch.cuda.synchronize(r)
    for p in p2ps:
        p.check()
    lays = ctx[0][0]
    per = 2 if args.mode == "fused" else 1  # RS reads (+ AG pushes) into each rank
    wire = sum(per * (l.m - 1) * l.S * 2 for l in lays)
    ms = [a.elapsed_time(b) for a, b in ev]
    print(json.dumps({"n_gpus": n, "mode": args.mode, "setup": "one process, one logical rank per GPU",
                      "ms_per_step_rank0": ms, "wire_in_bytes_per_rank_per_step": wire,
                      "wire_out_bytes_per_rank_per_step": wire,
                      "wire_in_gbs_best": wire / min(ms) / 1e6}), flush=True)
    for p in p2ps:
        p.close()


if __name__ == "__main__":
    main()
