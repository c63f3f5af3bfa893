#!/usr/bin/env python
"""BASELINE config 5: bucket-size sweep (1 MB .. 1 GB, bf16) of AllGather and
ReduceScatter through the C-ABI at N ranks (torchrun), three layouts:

  ragged  planner layout, element granularity: S = round_up(ceil(E/m), 8)
  even    FSDP1 flat even split S = ceil(E/m) (odd by construction: E = 1 mod 16),
          rank shards only 2-byte aligned
  ideal   same bytes, S rounded to 128 elements (256-B aligned)

busbw = (m S b / t) (m-1)/m (nccl-tests convention), t = max over ranks of the
CUDA-event time per call.  One JSON line per (size, layout, op) on rank 0.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      scripts/sweep_collectives.py [--sizes 1,4,16,64,256,1024] [--path nccl|fused]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2602_22437_b200 as R  # noqa: E402
from synth import workloads as W  # noqa: E402


def timeit(fn, iters, stream, world, gate=False):
    for _ in range(3):
        fn()
    stream.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if gate:  # hold the stream so the host enqueues every call before the first runs:
        # the events then time the device alone, not the launch rate (small sizes)
        with torch.cuda.stream(stream):
            torch.cuda._sleep(20_000_000)
        fn()  # absorbs the ranks' skew at the end of the sleep
    e0.record(stream)
    for _ in range(iters):
        fn()
    e1.record(stream)
    stream.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1,2,4,8,16,32,64,128,256,512,1024")
    ap.add_argument("--layouts", default="ragged,even,ideal")
    ap.add_argument("--ops", default="ag,rs")
    ap.add_argument("--path", choices=["nccl", "p2p"], default="nccl")
    ap.add_argument("--gate", action="store_true",
                    help="device-only timing: a sleep kernel holds the stream while the host enqueues")
    ap.add_argument("--workload", default="bucket",
                    help="bucket (config 5) | llama8b-layer | llama8b-root (config 3) | "
                         "dsv3 (config 4) | llama1b-layer | llama1b-root (config 2): whole units "
                         "with their declared granularity, layout 'ragged' only")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    comm = R.init_comm(rank, world, local)
    st = torch.cuda.Stream()
    named = {"llama8b-layer": W.llama3_8b_layer(0), "llama8b-root": W.llama3_8b_root(),
             "dsv3": W.dsv3_moe_unit(), "llama1b-layer": W.llama32_1b_layer(0),
             "llama1b-root": W.llama32_1b_root()}
    sizes = [int(x) for x in args.sizes.split(",")] if args.workload == "bucket" else [0]
    for mb in sizes:
        u = W.bucket(mb) if args.workload == "bucket" else named[args.workload]
        es = [t.numel for t in u.tensors]
        gs = [R.block_elems(t.shape, t.gran) for t in u.tensors]
        E = sum(es)
        for kind in (args.layouts.split(",") if args.workload == "bucket" else ["ragged"]):
            if kind == "ragged":
                lay = R.plan(es, gs, world)
            else:
                S = -(-E // world)
                if kind == "ideal":
                    S = -(-S // 128) * 128
                starts, acc = [], 0
                for e in es:
                    starts.append(acc)
                    acc += e
                lay = R.layout_from_starts(es, [1] * len(es), world, S, starts,
                                           require_gcoll=(kind == "ideal"))
            S = lay.S
            pf = torch.zeros(world * S, dtype=torch.bfloat16, device="cuda")
            gf = torch.zeros(world * S, dtype=torch.bfloat16, device="cuda")
            g32 = torch.zeros(world * S, dtype=torch.float32, device="cuda")
            unit = R.Unit(lay, rank, pf, gf, g32, qblock=0, comm=comm)
            p2p = None
            if args.path == "p2p":
                if (S * 2) % 16:
                    del unit, pf, gf, g32
                    continue  # p2p collectives need 16-B aligned shards
                p2p = R.P2P(comm, [pf, gf])
            iters = max(5, min(50, int(4e9 / (world * S * 4))))
            for op in args.ops.split(","):
                if op == "barrier":  # the start + done barrier pair alone (p2p path)
                    if p2p is None:
                        continue
                    fn = lambda: p2p.barrier(st)  # noqa: E731
                    nbytes = 0
                elif op == "ag":
                    fn = ((lambda: R.all_gather(unit, st)) if p2p is None
                          else (lambda: R.all_gather_p2p(unit, p2p, st)))  # noqa: E731
                    nbytes = world * S * 2
                elif op == "rs" and p2p is None:
                    fn = lambda: R.unit_reduce_scatter_f32(unit, st)  # noqa: E731
                    nbytes = world * S * 4
                elif op == "rs":  # fused cast + RS over NVLink, bf16 on the wire
                    fn = lambda: R.reduce_scatter_p2p(unit, p2p, st)  # noqa: E731
                    nbytes = world * S * 2
                else:
                    fn = lambda: R.reduce_scatter(unit, st)  # noqa: E731
                    nbytes = world * S * 4
                ms = timeit(fn, iters, st, world, args.gate)
                bus = nbytes / (ms * 1e-3) * (world - 1) / world / 1e9
                good = E * (2 if op == "ag" else 4) / (ms * 1e-3) * (world - 1) / world / 1e9
                if rank == 0:
                    print(json.dumps({"workload": args.workload,
                                      "mb": mb, "layout": kind, "op": op, "path": args.path, "gated": args.gate,
                                      "m": world, "S": S,
                                      "E": E, "ms": ms, "busbw_gbs": bus, "goodput_gbs": good,
                                      "pad": lay.padding, "nccl_env": {k: v for k, v in os.environ.items()
                                                                      if k.startswith("NCCL_")}}),
                          flush=True)
            if p2p is not None:
                st.synchronize()
                p2p.close()
            del unit, pf, gf, g32
            torch.cuda.empty_cache()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
