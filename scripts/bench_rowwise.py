#!/usr/bin/env python
"""BASELINE config 4: DeepSeek-V3-style MoE unit (38 tensors, 585,318,656
params, bf16), RaggedShard (128-row blocks, planner layout, zero-copy views)
vs FSDP2-style row-wise Shard(0) (Table 1).

Row-wise (FSDP2): every parameter is split evenly along dim 0 (rows padded to
a multiple of m; `--rowwise-rows 128` pads rows per rank to a multiple of 128
instead); the AllGather buffer is rank-major [rank][param shard]; so a step
needs
  AG:  ncclAllGather -> Copy-Out (m strided chunks per parameter into the
       parameter's full tensor)
  RS:  Copy-In with cast+scale (m chunks per parameter, bf16 grad -> fp32 x 1/m)
       -> ncclReduceScatter (fp32)
Ragged (this build): AG in place (views are zero-copy); RS = fused cast/scale
+ RS; both with NCCL (`--path nccl`) or the fused p2p kernels (`--path p2p`).
Copies use the library's batched ragged copy kernel (rsdb_copy_plan).

torchrun --nproc-per-node N scripts/bench_rowwise.py [--path nccl|p2p]
One JSON line per (layout, op) on rank 0: ms per step (max over ranks),
padding, bytes, and for row-wise the Copy-In / Copy-Out share.
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


def tmax(ms):
    t = torch.tensor([ms], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def timed(fns, iters, st):
    """ms per iteration of the sequence fns (each a callable), and per fn."""
    for _ in range(3):
        for f in fns:
            f()
    st.synchronize()
    dist.barrier()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(fns) + 1)] for _ in range(iters)]
    for it in range(iters):
        evs[it][0].record(st)
        for j, f in enumerate(fns):
            f()
            evs[it][j + 1].record(st)
    st.synchronize()
    per = [sum(evs[it][j].elapsed_time(evs[it][j + 1]) for it in range(iters)) / iters
           for j in range(len(fns))]
    return tmax(sum(per)), [tmax(p) for p in per]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--path", choices=["nccl", "p2p"], default="p2p")
    ap.add_argument("--rowwise-rows", type=int, default=1)
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    rank, m = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    comm = R.init_comm(rank, m, local)
    st = torch.cuda.Stream()
    unit = W.dsv3_moe_unit()
    es = [t.numel for t in unit.tensors]
    E = sum(es)
    out = []

    # ------------------------------------------------------------ ragged
    gs = [R.block_elems(t.shape, t.gran) for t in unit.tensors]
    lay = R.plan(es, gs, m)
    S = lay.S
    pf = torch.zeros(m * S, dtype=torch.bfloat16, device="cuda")
    gf = torch.randn(m * S, device="cuda").to(torch.bfloat16)
    g32 = torch.zeros(m * S, dtype=torch.float32, device="cuda")
    u = R.Unit(lay, rank, pf, gf, g32, qblock=0, comm=comm)
    p2p = R.P2P(comm, [pf, gf]) if args.path == "p2p" else None
    if p2p is None:
        ag = [lambda: R.all_gather(u, st)]
        rs = [lambda: R.unit_cast_scale(u, st), lambda: R.unit_reduce_scatter_f32(u, st)]
    else:
        ag = [lambda: R.all_gather_p2p(u, p2p, st)]
        rs = [lambda: R.reduce_scatter_p2p(u, p2p, st)]
    t_ag, _ = timed(ag, args.iters, st)
    t_rs, parts = timed(rs, args.iters, st)
    out.append({"layout": "ragged", "path": args.path, "m": m, "S": S, "padding": lay.padding,
                "pad_ratio": lay.padding / E, "ag_ms": t_ag, "rs_ms": t_rs, "copy_ms": 0.0,
                "rs_parts_ms": parts})
    if p2p is not None:
        st.synchronize()
        p2p.close()
    del u, pf, gf, g32

    # ------------------------------------------------------------ row-wise (FSDP2 Shard(0))
    q = args.rowwise_rows
    shard_rows, cols, off = [], [], []
    P = 0
    for t in unit.tensors:
        rows = t.shape[0]
        c = t.numel // rows
        sr = -(-rows // m)
        sr = -(-sr // q) * q
        shard_rows.append(sr)
        cols.append(c)
        off.append(P)
        P += sr * c
    P = -(-P // 8) * 8  # 16-B aligned rank chunks
    flat = torch.zeros(m * P, dtype=torch.bfloat16, device="cuda")       # AG buffer (rank-major)
    params = [torch.zeros(t.numel, dtype=torch.bfloat16, device="cuda") for t in unit.tensors]
    grads = [torch.randn(t.numel, device="cuda").to(torch.bfloat16) for t in unit.tensors]
    rsbuf = torch.zeros(m * P, dtype=torch.float32, device="cuda")       # RS input (rank-major)
    # Copy-Out after AllGather: chunk r of parameter t <- flat[r*P + off_t : ...]
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
    grad_dummy = torch.zeros(1, dtype=torch.bfloat16, device="cuda")
    u_rw = R.Unit(lay_rw, rank, flat, torch.zeros(m * P, dtype=torch.bfloat16, device="cuda"),
                  rsbuf, qblock=0, comm=comm)
    ag = [lambda: R.all_gather(u_rw, st), lambda: copy_out.run(st)]
    rs = [lambda: copy_in.run(st), lambda: R.unit_reduce_scatter_f32(u_rw, st)]
    t_ag, pa = timed(ag, args.iters, st)
    t_rs, pr = timed(rs, args.iters, st)
    out.append({"layout": f"rowwise{q}", "path": "nccl", "m": m, "S": P, "padding": m * P - E,
                "pad_ratio": (m * P - E) / E, "ag_ms": t_ag, "rs_ms": t_rs,
                "copy_out_ms": pa[1], "copy_in_ms": pr[0], "ag_parts_ms": pa, "rs_parts_ms": pr,
                "copy_segments": len(seg_out)})
    del grad_dummy
    if rank == 0:
        for o in out:
            print(json.dumps(o), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
