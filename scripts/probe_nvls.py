#!/usr/bin/env python
"""Probe (not part of the library): NVLS -- NVSwitch multicast through
torch's symmetric memory -- for the two collectives of the step, against the
copy-engine push this library uses.  Per rank S bytes of bf16:

  nvls_ag   multimem.st of the rank's slice to the multicast address
  nvls_rs   multimem.ld_reduce (add, fp32 accumulation, bf16 result) of the
            rank's slice, stored locally
  ce_ag     cudaMemcpyAsync pushes of the slice into every peer's buffer

Checks the results once (AG: every slice holds its owner's value; RS: the
sum), then times each op device-only (a sleep kernel holds the stream while
the host enqueues 10 calls), max over ranks.  One JSON line per (op, size).

  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \\
       -o /tmp/libprobe_nvls.so scripts/probe_nvls.cu
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 scripts/probe_nvls.py
"""
import ctypes
import json
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    lib = ctypes.CDLL(os.environ.get("PROBE_NVLS_LIB", "/tmp/libprobe_nvls.so"))
    for f in (lib.probe_nvls_ag, lib.probe_nvls_rs):
        f.restype = ctypes.c_int
    lib.probe_nvls_ag.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                  ctypes.c_void_p]
    lib.probe_nvls_rs.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                  ctypes.c_void_p]
    lib.probe_ce_ag.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                ctypes.c_void_p]
    st = torch.cuda.Stream()
    sp = ctypes.c_void_p(st.cuda_stream)
    grid = 148 * 4
    for mb in (16, 64, 256):
        S = mb << 20  # bytes per rank
        n = S // 2
        t = symm.empty(world * n, dtype=torch.bfloat16, device="cuda")
        h = symm.rendezvous(t, dist.group.WORLD.group_name)
        mc = h.multicast_ptr
        peers = (ctypes.c_void_p * world)(*h.buffer_ptrs)
        dst = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        my = t[rank * n:(rank + 1) * n]
        ops = {
            "nvls_ag": lambda: lib.probe_nvls_ag(ctypes.c_void_p(my.data_ptr()), ctypes.c_void_p(mc), rank * S, S,
                                                 grid, sp),
            "nvls_rs": lambda: lib.probe_nvls_rs(ctypes.c_void_p(mc), rank * S, ctypes.c_void_p(dst.data_ptr()), S,
                                                 grid, sp),
            "ce_ag": lambda: lib.probe_ce_ag(peers, world, rank, S, sp),
        }
        # correctness once
        t.fill_(0)
        my.fill_(float(rank + 1))
        torch.cuda.synchronize()
        dist.barrier()
        ok = {}
        for name in ("nvls_ag", "ce_ag"):
            t.fill_(0)
            my.fill_(float(rank + 1))
            torch.cuda.synchronize()
            dist.barrier()
            with torch.cuda.stream(st):
                assert ops[name]() == 0
            st.synchronize()
            dist.barrier()
            exp = torch.arange(1, world + 1, device="cuda", dtype=torch.float32).repeat_interleave(n)
            ok[name] = bool(torch.equal(t.float(), exp))
        t.fill_(1.0)
        torch.cuda.synchronize()
        dist.barrier()
        with torch.cuda.stream(st):
            assert ops["nvls_rs"]() == 0
        st.synchronize()
        dist.barrier()
        ok["nvls_rs"] = bool(torch.all(dst.float() == float(world)).item())
        for name, fn in ops.items():
            with torch.cuda.stream(st):
                for _ in range(3):
                    fn()
            st.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                torch.cuda._sleep(20_000_000)
                e0.record(st)
                for _ in range(10):
                    fn()
                e1.record(st)
            st.synchronize()
            ms = torch.tensor([e0.elapsed_time(e1) / 10], dtype=torch.float64, device="cuda")
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            ms = ms.item()
            if rank == 0:
                print(json.dumps({"op": name, "m": world, "mb_per_rank": mb, "us": ms * 1e3,
                                  "bus_gbs_per_rank": (world - 1) * S / (ms * 1e-3) / 1e9,
                                  "correct": ok[name]}), flush=True)
        dist.barrier()
        del h, t
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
