"""torchrun worker: every multi-rank parity case (tests/parity_cases.py) with
one process per GPU -- the p2p kernels over NVLink peer memory (CUDA IPC)
plus the NCCL entry points -- against the oracle's simulated ranks.
Launched by tests/test_gpu_multi.py:

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      --master-port P tests/dist_parity_worker.py

Exit code 0 iff every check passed on every rank."""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2602_22437_b200 as R  # noqa: E402
from parity_cases import all_cases  # noqa: E402
from rank_ctx import ProcCtx, drive_proc  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    comm = R.init_comm(rank, world, local)
    msgs = []
    keep = []
    for name, fn, kw in all_cases():
        ctx = ProcCtx(rank, world, comm)
        drive_proc(fn(ctx, **kw))
        msgs += [f"{name}: {m}" for m in ctx.msgs]
        keep.append(ctx)
    torch.cuda.synchronize()
    dist.barrier()
    flag = torch.tensor([1 if msgs else 0])
    dist.all_reduce(flag)
    if msgs:
        print(f"[rank {rank}] " + "; ".join(msgs[:20]), flush=True)
    if rank == 0:
        print(f"dist parity world={world}: {'PASS' if flag.item() == 0 else 'FAIL'}", flush=True)
    del keep
    comm.close()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 0 else 1)


if __name__ == "__main__":
    main()
