"""Runs every multi-rank parity case (tests/parity_cases.py) with `world`
logical ranks on ONE device (rsdb_comm_create_local / rsdb_p2p_create_local):
the N > 1 collective kernels -- p2p AllGather / ReduceScatter, the fused
ReduceScatter + 8-bit Adam (+ AllGather) kernel, the FP8 quantize +
AllGather, the K-slot ring gather, the Muon gather / apply -- compiled for
M = world ranks, checked element by element against the oracle's simulated
ranks.  Launched by tests/test_gpu_local_ranks.py in a subprocess with
CUDA_MODULE_LOADING=EAGER (a lazily loaded kernel can need a context
synchronisation while another rank's kernel spins in a barrier -- a
deadlock; EAGER loads every kernel up front) and CUDA_DEVICE_MAX_CONNECTIONS
=32 (each logical rank's stream gets its own hardware queue).

  python tests/local_ranks_worker.py WORLD [case ...]

Prints one line per case and "PASS"/"FAIL"; exit code 0 iff all passed."""
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import torch  # noqa: E402

from parity_cases import all_cases  # noqa: E402
from rank_ctx import drive_local  # noqa: E402


def main():
    world = int(sys.argv[1])
    only = set(sys.argv[2:])
    torch.cuda.set_device(0)
    # first use of every kernel (ours, cuBLAS's, torch's) outside the
    # multi-rank phases: each case once at world 1 (a plain single-rank run)
    from rank_ctx import ProcCtx, drive_proc
    for name, fn, kw in all_cases():
        if not only or name in only:
            drive_proc(fn(ProcCtx(0, 1), **kw))
    bad = 0
    for name, fn, kw in all_cases():
        if only and name not in only:
            continue
        t0 = time.time()
        try:
            ctxs = drive_local(world, fn, **kw)
            msgs = [f"[rank {c.rank}] {m}" for c in ctxs for m in c.msgs]
            del ctxs
        except Exception as e:  # noqa: BLE001 -- report and go on to the next case
            msgs = [f"{type(e).__name__}: {e}"]
        torch.cuda.synchronize()
        bad += bool(msgs)
        print(f"world={world} {name}: {'ok' if not msgs else 'FAIL'} ({time.time() - t0:.1f} s)"
              + ("" if not msgs else "\n  " + "\n  ".join(msgs[:12])), flush=True)
    print(f"local ranks world={world}: {'PASS' if not bad else 'FAIL'}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
