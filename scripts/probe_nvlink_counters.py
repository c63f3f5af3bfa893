"""Probe which NVLink traffic counters this box exposes (NVML field values,
nvidia-smi), reading them around a 4 GiB peer copy GPU0 -> GPU1."""
import subprocess

import pynvml as N
import torch

N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(0)
names = [n for n in dir(N) if n.startswith("NVML_FI_DEV_NVLINK_") and ("BYTES" in n or "THROUGHPUT" in n or "PACKETS" in n)]


def read():
    out = {}
    for n in names:
        fid = getattr(N, n)
        for scope in (None, 0):
            try:
                req = [fid] if scope is None else [(fid, scope)]
                v = N.nvmlDeviceGetFieldValues(h, req)[0]
                out[(n, scope)] = (v.nvmlReturn, int(v.value.ullVal))
            except Exception as e:
                out[(n, scope)] = ("exc", str(e)[:60])
    return out


def smi():
    r = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], capture_output=True, text=True)
    return (r.stdout + r.stderr)[:800]


a = read()
s0 = smi()
x = torch.ones(1 << 30, dtype=torch.float32, device="cuda:0")
y = torch.empty_like(x, device="cuda:1")
for _ in range(1):
    y.copy_(x)
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
b = read()
s1 = smi()
for k in a:
    print(k, a[k], b[k], (b[k][1] - a[k][1]) if isinstance(a[k][1], int) and isinstance(b[k][1], int) else None)
print("smi before:\n", s0)
print("smi after:\n", s1)
r = subprocess.run(["nvidia-smi", "nvlink", "-h"], capture_output=True, text=True)
print(r.stdout[:3000])
