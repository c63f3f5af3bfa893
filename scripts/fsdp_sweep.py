#!/usr/bin/env python
"""FSDP-size sweep and DBuffer memory accounting (P:369, P:372-373,
P:493).  For a workload and a list of FSDP sizes m, per rank 0:

  plan      S, padding % and planner time of every unit (C++ planner)
  wire      AllGather / ReduceScatter bytes into the rank per step (bf16)
  dbuffer   bytes of the batched DBuffer arenas (rsdb_arena_sizes: one
            allocation per buffer kind, 256-B aligned units)
  fsdp2     the same buffers allocated per parameter in FSDP2's per-parameter
            layout: Shard(0) pads dim 0 to a multiple of m, and every kind of
            every tensor is its own allocation, rounded to the caching
            allocator's 512 B (the request; reserved segments come on top)

--select N (host): P:493's offline choice of the FSDP group size -- among
the divisors m of N GPUs with m >= --min-fsdp (the smallest group whose
shards fit in memory; the rest of the N goes to replication, HSDP), the m
with the least LCM-induced padding; ties go to the larger m (less memory per
GPU).  One JSON line with every candidate and the choice.

With --measure (one GPU) both allocation patterns are replayed through
PyTorch's caching allocator and torch.cuda.memory_reserved() is reported --
the paper's "peak reserved" comparison (batched DBuffer -12 % vs
FSDP2's per-parameter eager allocation).  One JSON line per m.

  python scripts/fsdp_sweep.py --workload llama1b --ms 2,4,8,16,64 [--measure]
  python scripts/fsdp_sweep.py --workload gptoss128 --select 1024 --min-fsdp 256
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2602_22437_b200 as R  # noqa: E402
from synth import workloads as W  # noqa: E402

QBLOCK = 2048
KINDS = ("param_full", "grad_full", "grad_f32", "master", "m_q", "v_q", "m_absmax", "v_absmax")


def workload(name):
    return {"llama1b": lambda: W.llama32_1b(),
            "llama8b": lambda: W.llama3_8b_muon(),
            "dsv3": lambda: W.dsv3_moe(),
            "dsv3_671b_128": lambda: W.deepseek_v3_671b(128),
            "gptoss128": lambda: W.gpt_oss_120b(128)}[name]()


def padding_ratio(w, m):
    """Σ(m·S − E) / ΣE over the workload's units (C++ planner); identical
    units are planned once."""
    pad = tot = 0
    seen = {}
    for u in W.all_units(w):
        key = tuple((t.numel, R.block_elems(t.shape, t.gran)) for t in u.tensors)
        if key not in seen:
            lay = R.plan([k[0] for k in key], [k[1] for k in key], m, elem_bytes=2)
            seen[key] = (lay.m * lay.S - lay.E, lay.E)
        pad += seen[key][0]
        tot += seen[key][1]
    return pad / tot


def select_group_size(w, n_gpus, min_fsdp=2):
    """"we select the FSDP group size by offline simulation to minimize
    LCM-induced rounding".  Candidates: the divisors m >= min_fsdp of n_gpus;
    the one with the least padding wins, ties to the larger group."""
    ms = [m for m in range(max(2, min_fsdp), n_gpus + 1) if n_gpus % m == 0]
    if not ms:
        raise ValueError(f"no divisor of {n_gpus} is >= {min_fsdp}")
    table = {m: padding_ratio(w, m) for m in ms}
    best = min(ms, key=lambda m: (round(table[m], 12), -m))
    return best, table


def ceil_div(a, b):
    return -(-a // b)


def fsdp2_requests(unit, m):
    """Per-parameter allocations of FSDP2's layout (rank 0): every tensor is
    Shard(0) with dim 0 padded to a multiple of m; per kind, the same buffers
    as one DBuffer unit holds (gathered bf16 param and grad, fp32 RS buffer,
    fp32 master, 8-bit states, per-2048-block absmax)."""
    reqs = []
    for t in unit.tensors:
        rows = t.shape[0]
        rest = t.numel // rows
        s = ceil_div(rows, m) * rest  # shard elements
        nb = ceil_div(s, QBLOCK)
        reqs += [m * s * 2, m * s * 2, m * s * 4, s * 4, s, s, nb * 4, nb * 4]
    return reqs


def round512(n):
    return max(512, ceil_div(n, 512) * 512) if n > 0 else 0


def sweep_one(w, m, measure):
    units = list(W.all_units(w))
    t0 = time.perf_counter()
    lays, qspec = [], []
    for u in units:
        es = [t.numel for t in u.tensors]
        gs = [R.block_elems(t.shape, t.gran) for t in u.tensors]
        lays.append(R.plan(es, gs, m, elem_bytes=2))
        qspec.append([("flat", min(QBLOCK, g)) for g in gs])  # 8-bit state blocks stay intact
    plan_s = time.perf_counter() - t0
    E = sum(l.E for l in lays)
    padded = sum(l.m * l.S for l in lays)
    sizes, _ = R.arena_sizes(lays, 0, QBLOCK, 256, qspec=qspec)
    reqs = [r for u in units for r in fsdp2_requests(u, m)]
    fsdp2_pad_elems = sum(ceil_div(t.shape[0], m) * m * (t.numel // t.shape[0]) for u in units
                          for t in u.tensors)
    # FSDP2 Shard(0) that keeps the declared row blocks intact: rows per rank
    # rounded up to a multiple of the block's rows (SURVEY config 4 "row-wise-128")
    blk_pad_elems = 0
    for u in units:
        for t in u.tensors:
            rows, rest = t.shape[0], t.numel // t.shape[0]
            br = max(1, R.block_elems(t.shape, t.gran) // rest) if len(t.shape) > 1 else 1
            blk_pad_elems += ceil_div(ceil_div(rows, m), br) * br * m * rest
    line = {"workload": w.name, "m": m, "units": len(units), "params": E,
            "plan_s_total": plan_s,
            "ragged_padding_pct": 100.0 * (padded - E) / E,
            "fsdp2_dim0_padding_pct": 100.0 * (fsdp2_pad_elems - E) / E,
            "fsdp2_rowwise_block_padding_pct": 100.0 * (blk_pad_elems - E) / E,
            "ag_wire_bytes_per_rank": sum((l.m - 1) * l.S * 2 for l in lays),
            "rs_wire_bytes_per_rank_bf16": sum((l.m - 1) * l.S * 2 for l in lays),
            "dbuffer_bytes": sum(sizes), "dbuffer_bytes_by_kind": dict(zip(KINDS, sizes)),
            "fsdp2_requested_bytes": sum(reqs), "fsdp2_allocations": len(reqs),
            "fsdp2_rounded_bytes": sum(round512(r) for r in reqs)}
    line["fsdp2_over_dbuffer"] = line["fsdp2_rounded_bytes"] / max(1, line["dbuffer_bytes"])
    if measure:
        import torch
        torch.cuda.empty_cache()
        base = torch.cuda.memory_reserved()
        arenas = [torch.empty(max(1, s), dtype=torch.uint8, device="cuda") for s in sizes]
        line["dbuffer_reserved"] = torch.cuda.memory_reserved() - base
        del arenas
        torch.cuda.empty_cache()
        base = torch.cuda.memory_reserved()
        bufs = [torch.empty(r, dtype=torch.uint8, device="cuda") for r in reqs if r > 0]
        line["fsdp2_reserved"] = torch.cuda.memory_reserved() - base
        del bufs
        torch.cuda.empty_cache()
        line["reserved_fsdp2_over_dbuffer"] = line["fsdp2_reserved"] / max(1, line["dbuffer_reserved"])
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="llama1b",
                    choices=["llama1b", "llama8b", "dsv3", "dsv3_671b_128", "gptoss128"])
    ap.add_argument("--select", type=int, default=0, help="choose the FSDP size for N GPUs (P:493)")
    ap.add_argument("--min-fsdp", type=int, default=8, help="smallest FSDP group that fits in memory")
    ap.add_argument("--ms", default="2,4,8,16,32,64")
    ap.add_argument("--measure", action="store_true")
    args = ap.parse_args()
    w = workload(args.workload)
    if args.select:
        best, table = select_group_size(w, args.select, args.min_fsdp)
        print(json.dumps({"workload": w.name, "gpus": args.select, "fsdp_size": best,
                          "hsdp_replicas": args.select // best,
                          "padding_pct": {m: round(100 * r, 4) for m, r in table.items()}}), flush=True)
        return
    for m in [int(x) for x in args.ms.split(",")]:
        print(json.dumps(sweep_one(w, m, args.measure)), flush=True)


if __name__ == "__main__":
    main()
