"""-m gpu parity at BASELINE's full size (Llama-3.2-1B, 1.24 B params) in the
launch configuration bench.py times, on sampled blocks of every unit (see
tests/fullsize_worker.py): world 1 in-process, 2 and 4 under torchrun when the
box has the GPUs."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,scope", [(1, "dbuffer"), (1, "unit"), (2, "unit"), (2, "dbuffer"),
                                     (2, "dbuffer+ag"), (4, "unit"), (4, "dbuffer+ag"),
                                     (4, "unit+ag")])
def test_fullsize_parity(n, scope):
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    worker = os.path.join(HERE, "fullsize_worker.py")
    if n == 1:
        cmd = [sys.executable, worker]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), worker]
    env = dict(os.environ, FULLSIZE_SCOPE=scope)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, env=env)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0 and "PASS" in r.stdout
