"""Probe: does torch's symmetric memory give an NVLS multicast address on
this box (plumbing for an NVSwitch multicast variant of the fused kernels)?"""
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
dist.init_process_group("nccl")
try:
    t = symm.empty(1 << 20, dtype=torch.bfloat16, device="cuda")
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    print(rank, "buffer_ptrs", [hex(p) for p in h.buffer_ptrs], "multicast_ptr", hex(h.multicast_ptr),
          "signal_pad", [hex(p) for p in h.signal_pad_ptrs][:2], flush=True)
except Exception as e:
    print(rank, "symm_mem failed:", type(e).__name__, e, flush=True)
dist.barrier()
dist.destroy_process_group()
