"""-m gpu: the N > 1 path on ONE GPU.  world = 2, 3, 4, 8 logical ranks in one
process on one device run every multi-rank parity case (tests/parity_cases.py:
p2p AllGather / ReduceScatter bit exact, 8-bit Adam codes exact, fused
RS + Adam (+ AG) bit identical to the unfused kernels, long blocks and 2-D
tiles through the fused kernel, FP8 quantize + AllGather, K-slot ring,
distributed Muon) against the oracle's simulated ranks -- the same kernels,
templated on M = world, that run one rank per GPU over NVLink.  3 is a world
where fl(1/m) is inexact; 8 is the largest template instance.  Each world runs
in a subprocess under a timeout (tests/local_ranks_worker.py); barrier waits
also time out on the device (rsdb_p2p_set_timeout), so a hang fails the test
instead of wedging the GPU."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_local_ranks(world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, CUDA_MODULE_LOADING="EAGER", CUDA_DEVICE_MAX_CONNECTIONS="32")
    r = subprocess.run([sys.executable, os.path.join(HERE, "local_ranks_worker.py"), str(world)],
                       capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-6000:], r.stderr[-3000:])
    assert r.returncode == 0 and f"world={world}: PASS" in r.stdout


@pytest.mark.parametrize("devices", [[0, 1], [0, 1, 0, 1]])
def test_local_ranks_across_devices(devices):
    """The same cases with ONE process driving two GPUs (logical rank r on
    devices[r]; two ranks per device in the second case): per-device kernel
    setup (shared-memory attributes, constant tables) and peer mappings
    across devices -- the single-process multi-GPU mode the NVLink counter
    captures use (scripts/ncu_nvlink_local.py)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    world = len(devices)
    env = dict(os.environ, CUDA_MODULE_LOADING="EAGER", CUDA_DEVICE_MAX_CONNECTIONS="32")
    r = subprocess.run([sys.executable, os.path.join(HERE, "local_ranks_worker.py"), str(world), "--devices",
                        ",".join(map(str, devices))], capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-6000:], r.stderr[-3000:])
    assert r.returncode == 0 and "PASS" in r.stdout.splitlines()[-1]
