"""Helpers for the -m gpu parity tests.

GPU-side inputs are placed with the PRODUCT layout (paper_2602_22437_b200
Layout.starts, torch slice copies); oracle-side inputs with the ORACLE layout
(oracle.dbuffer.place_logical).  Both start from the same synth logical
vectors; the planner parity (tests/test_capi_host.py) makes the layouts equal.
"""
import numpy as np
import torch

import paper_2602_22437_b200 as R
from synth import hashgen as H


def place_gpu(lay: R.Layout, flat: torch.Tensor, dtype, fill=0.0) -> torch.Tensor:
    """m*S device buffer with the logical vector at each tensor's interval."""
    buf = torch.full((lay.m * lay.S,), fill, dtype=dtype, device="cuda")
    off = 0
    for l, e in zip(lay.starts, numels(lay)):
        buf[l:l + e] = flat[off:off + e].to(dtype)
        off += e
    return buf


def numels(lay: R.Layout):
    return lay.to_json()["numel"]


def bf16_bits(t: torch.Tensor) -> np.ndarray:
    return t.detach().view(torch.int16).cpu().numpy().view(np.uint16)


def f32(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy()


def logical_params(seed, E):
    return torch.from_numpy(H.params_np(seed, 0, E))


def logical_grads(seed, rank, E):
    return torch.from_numpy(H.grads_np(seed, rank, 0, E))
