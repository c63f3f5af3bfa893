#!/usr/bin/env python
"""SURVEY N3 measurement: one distributed-Muon step (Algorithm 2,
rsdb_muon_step) over a Llama-3-8B decoder layer unit (BJ config 3 shapes;
2-D matrices updated by Muon, norms skipped) laid out by the RaggedShard
planner at element granularity (matrices straddle ranks, so Redistribute
moves real bytes).  Times the whole step and the same step with 0
Newton-Schulz iterations (momentum + gather + normalise + scatter/apply), the
difference being the Newton-Schulz GEMM time; reports the NS TFLOP/s of the
busiest root against the measured dense bf16 peak (MEASURED_PEAKS.json).
One JSON line on rank 0.  Measurement only: parity is in tests/
(test_gpu_muon.py, the parity worker at N = 2 / 4, and
test_gpu_fullsize_ext.py's k_proj check at this size) -- only tests/ execute
the oracle.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      scripts/bench_muon.py [--precision bf16|f32] [--iters 5]
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


def ns_flops(r, c, steps):
    k, L = min(r, c), max(r, c)
    return steps * (4 * k * k * L + 2 * k ** 3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", choices=["bf16", "f32"], default="bf16")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    comm = R.init_comm(rank, world, local)
    unit = W.llama3_8b_layer(0)
    shapes = [t.shape if len(t.shape) == 2 else None for t in unit.tensors]
    es = [t.numel for t in unit.tensors]
    lay = R.plan(es, [1] * len(es), world, elem_bytes=2)
    S = lay.S
    mk = lambda st: H.values_torch(7, st, rank * S, S, 14, device="cuda")  # noqa: E731
    master, buf, grad = mk(1), mk(2), mk(3)
    u = torch.zeros(S, device="cuda")
    param = torch.zeros(S, dtype=torch.bfloat16, device="cuda")
    mu = R.Muon(lay, shapes, rank, comm=comm, precision=args.precision)
    ws = torch.zeros(mu.workspace_bytes, dtype=torch.uint8, device="cuda")
    mu.bind(master, buf, grad, u, ws, param_bf16=param)
    p2p = R.P2P(comm, [u, ws]) if world > 1 else None
    st = torch.cuda.Stream()

    def timed(cfg):
        with torch.cuda.stream(st):
            for _ in range(args.warmup):
                mu.step(cfg, p2p, st)
        st.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        with torch.cuda.stream(st):
            for _ in range(args.iters):
                mu.step(cfg, p2p, st)
        e1.record(st)
        st.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.iters], dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    t_full = timed(R.MuonConfig())
    t_zero = timed(R.MuonConfig(ns_steps=0))
    roots = [mu.root(t) for t in range(len(shapes))]
    load = [0] * world
    for t, s in enumerate(shapes):
        if s is not None:
            load[roots[t]] += ns_flops(s[0], s[1], 5)
    moved = 0  # fp32 u elements gathered to roots from other ranks (= returned to owners)
    for t, s in enumerate(shapes):
        if s is None:
            continue
        l, e = lay.starts[t], es[t]
        r = roots[t]
        own = max(0, min(l + e, (r + 1) * S) - max(l, r * S))
        moved += e - own
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    except Exception:
        peak = 1590.0
    if rank == 0:
        t_ns = max(t_full - t_zero, 1e-6)
        tf = max(load) / (t_ns * 1e-3) / 1e12
        line = {"workload": "llama-3-8b layer unit, element-granularity RaggedShard", "n_gpus": world,
                "precision": args.precision, "matrices": sum(s is not None for s in shapes),
                "roots": roots, "muon_step_ms": t_full, "step_without_ns_ms": t_zero,
                "ns_ms": t_ns, "ns_tflops_busiest_root": tf,
                "ns_tensor_frac": tf / peak if args.precision == "bf16" else None,
                "peak_bf16_tflops": peak, "redistributed_elements": moved,
                "parity": "tests/test_gpu_fullsize_ext.py (k_proj), tests/dist_parity_worker.py"}
        print(json.dumps(line), flush=True)
    if p2p is not None:
        torch.cuda.synchronize()
        p2p.close()
    mu.close()
    comm.close()
    if world > 1:
        dist.destroy_process_group()
    sys.exit(0)


if __name__ == "__main__":
    main()
