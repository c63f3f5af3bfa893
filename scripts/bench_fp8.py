#!/usr/bin/env python
"""SURVEY N2 measurement: FP8 (E4M3) 128x128 block quantization fused with the
AllGather (rsdb_fp8_quantize_all_gather, 1 B/element on the wire) against the
bf16 AllGather (rsdb_all_gather_p2p, 2 B/element) of the same weights: the
FFN matrices of the BJ config-4 DeepSeek-V3-style MoE unit (27 matrices,
396,361,728 params, 128-row granularity).  Measurement only: parity of this
path is in tests/ (test_gpu_fp8.py, the parity worker at N = 2 / 4, and
test_gpu_fullsize_ext.py at this size) -- only tests/ execute the oracle.
Works at world 1 (quantization only) and under torchrun.  One JSON line on
rank 0.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      scripts/bench_fp8.py [--iters 20] [--samples 24]
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
from synth import hashgen as H  # noqa: E402
from synth import workloads as W  # noqa: E402


def timeit(fn, iters, stream, world):
    for _ in range(3):
        fn()
    stream.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(iters):
        fn()
    e1.record(stream)
    stream.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--samples", type=int, default=24)
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    comm = R.init_comm(rank, world, local)
    unit = W.dsv3_ffn_fp8_unit()
    shapes = [t.shape for t in unit.tensors]
    es = [t.numel for t in unit.tensors]
    gs = [128 * c for _, c in shapes]
    specs = [("tile", c, 128, 128) for _, c in shapes]
    lay = R.plan(es, gs, world, elem_bytes=1)
    S, E = lay.S, sum(es)
    # fp32 master shard (logical index = position in the unit's concatenated tensors)
    master = torch.zeros(S, dtype=torch.float32, device="cuda")
    lo, hi = rank * S, (rank + 1) * S
    off = 0
    for l, e in zip(lay.starts, es):
        a, b = max(l, lo), min(l + e, hi)
        if a < b:
            master[a - lo:b - lo] = H.values_torch(3, H.STREAM_PARAM, off + a - l, b - a, 12,
                                                   outliers=True, device="cuda")
        off += e
    codes = torch.zeros(world * S, dtype=torch.uint8, device="cuda")
    u0 = R.Fp8Unit(lay, specs, rank, master, codes, torch.empty(1, device="cuda"), comm=comm)
    ntiles = u0.num_tiles
    u0.close()
    scales = torch.zeros(ntiles, dtype=torch.float32, device="cuda")
    p2p = R.P2P(comm, [codes, scales]) if world > 1 else None
    fu = R.Fp8Unit(lay, specs, rank, master, codes, scales, comm=comm)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        t_fp8 = timeit(lambda: fu.quantize_all_gather(p2p, st), args.iters, st, world)
    # bf16 AllGather of the same weights (the step it replaces)
    lay16 = R.plan(es, gs, world, elem_bytes=2)
    pf = torch.zeros(world * lay16.S, dtype=torch.bfloat16, device="cuda")
    t_bf16 = None
    if world > 1:
        gf = torch.zeros(world * lay16.S, dtype=torch.bfloat16, device="cuda")
        g32 = torch.zeros(world * lay16.S, dtype=torch.float32, device="cuda")
        u16 = R.Unit(lay16, rank, pf, gf, g32, qblock=2048, comm=comm)
        p16 = R.P2P(comm, [pf])
        with torch.cuda.stream(st):
            t_bf16 = timeit(lambda: R.all_gather_p2p(u16, p16, st), args.iters, st, world)
        torch.cuda.synchronize()
        p16.close()
        del u16, gf, g32
    if rank == 0:
        wire = (world - 1) * S  # code bytes into each rank
        line = {"workload": "dsv3 FFN fp8 unit (27 matrices, 128x128 tiles)", "params": E,
                "n_gpus": world, "S": S, "tiles": ntiles, "fp8_quant_ag_ms": t_fp8,
                "bf16_ag_ms": t_bf16,
                "fp8_wire_gbs": wire / (t_fp8 * 1e-3) / 1e9 if world > 1 else None,
                "fp8_hbm_gbs": 5 * S / (t_fp8 * 1e-3) / 1e9,
                "bf16_ag_wire_gbs": (world - 1) * lay16.S * 2 / (t_bf16 * 1e-3) / 1e9 if t_bf16 else None,
                "speedup_vs_bf16_ag": t_bf16 / t_fp8 if t_bf16 else None,
                "parity": "tests/test_gpu_fullsize_ext.py, tests/dist_parity_worker.py"}
        print(json.dumps(line), flush=True)
    fu.close()
    if p2p is not None:
        torch.cuda.synchronize()
        p2p.close()
    comm.close()
    if world > 1:
        dist.destroy_process_group()
    sys.exit(0)


if __name__ == "__main__":
    main()
