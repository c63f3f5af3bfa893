"""Build librsdb.so in-tree with nvcc for sm_100a (B200).

python paper_2602_22437_b200/build.py      (or __graft_entry__.build())

Flags: -gencode arch=compute_100a,code=sm_100a (SASS only, no PTX JIT),
-O3 -lineinfo (ncu source view), -Xptxas -v (register / spill report kept in
build/ptxas.log).  Never --use_fast_math: the host scalars and the RNE
conversions must stay IEEE.  NCCL: the torch-bundled 2.28.9
from the venv (same library torch loads, one NCCL in the process).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "librsdb.so")
SOURCES = ["planner.cc", "capi.cc", "capi_ext.cc", "kernels.cu", "p2p.cu", "fp8.cu", "muon.cu", "adam_dyn.cu", "ns_umma.cu"]
HEADERS = ["planner.hpp", "capi_internal.hpp", "kernels.cuh", "adam_dev.cuh", "p2p_dev.cuh", "devmath.cuh"]


def nccl_dir() -> str:
    cands = [os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl")]
    try:
        import nvidia  # type: ignore
        for p in getattr(nvidia, "__path__", []):
            cands.append(os.path.join(p, "nccl"))
    except Exception:
        pass
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return c
    raise RuntimeError("NCCL headers not found (expected site-packages/nvidia/nccl)")


def cublas_dir() -> str:
    """The torch-bundled cuBLAS (the same library torch loads: one cuBLAS in
    the process); used for the Muon Newton-Schulz GEMMs (N3)."""
    c = os.path.join(os.path.dirname(nccl_dir()), "cublas")
    if os.path.exists(os.path.join(c, "lib", "libcublas.so.12")):
        return c
    raise RuntimeError("cuBLAS not found (expected site-packages/nvidia/cublas)")


def nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "rsdb.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    nd = nccl_dir()
    cd = cublas_dir()
    bdir = os.path.join(ROOT, "build")
    os.makedirs(bdir, exist_ok=True)
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
           "-std=c++17", "-Xcompiler", "-fPIC,-O3,-Wall", "-Xptxas", "-v", "-shared",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"),
           *[os.path.join(CSRC, s) for s in SOURCES],
           "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
           "-Xlinker", "-rpath," + os.path.join(nd, "lib"),
           "-L", os.path.join(cd, "lib"), "-l:libcublas.so.12",
           "-Xlinker", "-rpath," + os.path.join(cd, "lib"),
           "-o", OUT + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(os.path.join(bdir, "ptxas.log"), "w") as f:
        f.write(" ".join(cmd) + "\n\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building librsdb.so (see build/ptxas.log)")
    if verbose:
        sys.stdout.write(r.stderr)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
