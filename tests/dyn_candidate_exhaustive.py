"""Exhaustive host check of the dynamic-codec kernel's closed-form candidate
(paper_2602_22437_b200/csrc/adam_dyn.cu dyn_candidate + clamp): for EVERY
fp32 y in [-1, 1] (signed map) and [0, 1] (unsigned map) the true hi (first
index with map >= y, clamped to [1, 255]) is within one of the candidate, so
the kernel's branch-free 4-value decision is the oracle's.  ~5 min, numpy.
Output kept in profiles/r2/dyn_candidate_exhaustive.txt.  Test infrastructure
(imports the oracle); run: python tests/dyn_candidate_exhaustive.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import codemap as CM
f32 = np.float32
TH = np.array([1e-6, 1e-5, 1e-4, 1e-3, 1e-2, 1e-1], dtype=f32)
DINV = np.array([1e6, 1e5, 1e4, 1e3, 1e2, 1e1, 1.0], dtype=f32)
K9 = f32(1.0) / f32(0.9)
def cand(a, signed):
    W = 0 if signed else 1
    i = np.zeros(a.shape, np.int32)
    for t in TH: i += (a >= t)
    cnt = (1 << (i + W)).astype(np.int32)
    u = (a * DINV[i]).astype(f32)
    u = (u - f32(0.1)).astype(f32)
    u = (u * cnt.astype(f32)).astype(f32)
    u = (u * K9).astype(f32)
    t = (u - f32(0.5)).astype(f32)
    j = np.rint(t).astype(np.int64)
    j = np.clip(j, 0, cnt - 1)
    return (127 if signed else 0) + cnt + j
def check(signed, neg):
    mp = CM.dynamic_map(signed)
    bad = 0; n = 0
    hi_bits = 0x3F800000
    step = 1 << 24
    for s in range(0, hi_bits + 1, step):
        bits = np.arange(s, min(s + step, hi_bits + 1), dtype=np.uint32)
        a = bits.view(f32)
        y = -a if neg else a
        p = cand(a, signed)
        c = (255 - p) if neg else p
        c = np.clip(c, 2, 254)
        true_hi = np.clip(np.searchsorted(mp, y, side='left'), 1, 255)
        ok = (true_hi >= c - 1) & (true_hi <= c + 1)
        bad += int((~ok).sum()); n += a.size
        if (~ok).any():
            idx = np.nonzero(~ok)[0][:3]
            print("BAD", signed, neg, y[idx], c[idx], true_hi[idx], flush=True)
    print("signed" if signed else "unsigned", "neg" if neg else "pos", n, "bad", bad, flush=True)
if __name__ == "__main__":
    t0 = time.time()
    check(True, False)
    check(True, True)
    check(False, False)
    print("time", time.time() - t0)
