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

  python tests/local_ranks_worker.py WORLD [--devices 0,1,...] [case ...]

--devices: logical rank r on GPU devices[r] (one process driving several
GPUs; the per-device kernel setup and cross-device peer mappings).

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
    rest = sys.argv[2:]
    devices = None
    if rest and rest[0] == "--devices":
        devices = [int(x) for x in rest[1].split(",")]
        rest = rest[2:]
        assert len(devices) == world
    only = set(rest)
    torch.cuda.set_device(0)
    # first use of every kernel (ours, cuBLAS's, torch's) outside the
    # multi-rank phases: each case once at world 1 (a plain single-rank run)
    from rank_ctx import ProcCtx, drive_proc
    for d in sorted(set(devices or [0])):  # on every device the ranks use
        with torch.cuda.device(d):
            for name, fn, kw in all_cases():
                if not only or name in only:
                    drive_proc(fn(ProcCtx(0, 1), **kw))
    bad = 0
    for name, fn, kw in all_cases():
        if only and name not in only:
            continue
        t0 = time.time()
        try:
            ctxs = drive_local(world, fn, devices=devices, **kw)
            msgs = [f"[rank {c.rank}] {m}" for c in ctxs for m in c.msgs]
            del ctxs
        except Exception as e:  # noqa: BLE001 -- report and go on to the next case
            msgs = [f"{type(e).__name__}: {e}"]
        for d in sorted(set(devices or [0])):
            torch.cuda.synchronize(d)
        bad += bool(msgs)
        print(f"world={world} {name}: {'ok' if not msgs else 'FAIL'} ({time.time() - t0:.1f} s)"
              + ("" if not msgs else "\n  " + "\n  ".join(msgs[:12])), flush=True)
    print(f"local ranks world={world}{' devices=' + ','.join(map(str, devices)) if devices else ''}: "
          f"{'PASS' if not bad else 'FAIL'}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
