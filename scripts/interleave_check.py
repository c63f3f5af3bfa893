#!/usr/bin/env python
"""Cross-check of the experimental interleaved optimizer-state layout
(RSDB_STATE_LAYOUT=interleaved): the same fused DBuffer steps on a small
3-unit workload from the same logical state, in whichever layout the
environment selects; prints a hash of the final bf16 parameters and of every
block's master / codes / absmax read back in logical order.  Run once per
layout and compare the two lines (they must be equal)."""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_22437_b200 as R  # noqa: E402
from synth import hashgen as H  # noqa: E402

UNITS = [[2048 * 100, 300, 2048 * 7 + 16], [2048 * 33], [4096 * 10, 1024]]
Q = 2048


def main():
    inter = os.environ.get("RSDB_STATE_LAYOUT") == "interleaved"
    torch.cuda.set_device(0)
    lays = [R.plan(es, [min(Q, e) for e in es], 1) for es in UNITS]
    sizes, offs = R.arena_sizes(lays, 0, Q, 256)
    arenas = [torch.zeros(max(1, s), dtype=torch.uint8, device="cuda") for s in sizes]
    db = R.DBuffer(lays, 0, arenas, qblock=Q, align=256)
    runs = []  # per unit: list of (block off, len, master byte, mq byte, vq byte)
    for ui, l in enumerate(lays):
        S, off = l.S, offs[ui]
        blocks = l.rank_blocks(0, Q)
        p = H.params_torch(ui, 0, l.E, device="cuda")
        full = torch.zeros(S, device="cuda")
        o = 0
        for st_, e in zip(l.starts, UNITS[ui]):
            full[st_:st_ + e] = p[o:o + e]
            o += e
        arenas[0][off[0]:off[0] + S * 2].view(torch.bfloat16).copy_(full.to(torch.bfloat16))
        arenas[1][off[1]:off[1] + S * 2].view(torch.bfloat16).copy_(
            H.grads_torch(ui, 0, 0, S, device="cuda").to(torch.bfloat16))
        mc = H.codes_torch(ui, H.STREAM_MCODE, 0, S, True, device="cuda").view(torch.uint8)
        vc = H.codes_torch(ui, H.STREAM_VCODE, 0, S, False, device="cuda")
        ib = off[3]
        rl = []
        for bo, n in blocks:
            if inter:
                mb, qm, qv = ib, ib + 4 * n, ib + 5 * n
                ib += (6 * n + 15) // 16 * 16
            else:
                mb, qm, qv = off[3] + 4 * bo, off[4] + bo, off[5] + bo
            rl.append((bo, n, mb, qm, qv))
            arenas[3][mb:mb + 4 * n].view(torch.float32).copy_(full[bo:bo + n])
            arenas[4 if not inter else 3][qm:qm + n].copy_(mc[bo:bo + n])
            arenas[5 if not inter else 3][qv:qv + n].copy_(vc[bo:bo + n])
        runs.append(rl)
        nb = len(blocks)
        arenas[6][off[6]:off[6] + nb * 4].view(torch.float32).copy_(
            H.absmax_torch(ui, H.STREAM_ABSM, 0, nb, 14, device="cuda"))
        arenas[7][off[7]:off[7] + nb * 4].view(torch.float32).copy_(
            H.absmax_torch(ui, H.STREAM_ABSV, 0, nb, 22, device="cuda"))
    cfg = R.AdamConfig()
    for t in range(1, 4):
        db.reduce_scatter_adam(cfg, t, None)
    torch.cuda.synchronize()
    h = hashlib.sha256()
    for ui, l in enumerate(lays):
        off = offs[ui]
        h.update(arenas[0][off[0]:off[0] + l.S * 2].cpu().numpy().tobytes())
        for bo, n, mb, qm, qv in runs[ui]:
            h.update(arenas[3][mb:mb + 4 * n].cpu().numpy().tobytes())
            h.update(arenas[4 if not inter else 3][qm:qm + n].cpu().numpy().tobytes())
            h.update(arenas[5 if not inter else 3][qv:qv + n].cpu().numpy().tobytes())
        nb = len(runs[ui])
        h.update(arenas[6][off[6]:off[6] + nb * 4].cpu().numpy().tobytes())
        h.update(arenas[7][off[7]:off[7] + nb * 4].cpu().numpy().tobytes())
    print(json.dumps({"layout": "interleaved" if inter else "split", "sha256": h.hexdigest()}))
    db.close()


if __name__ == "__main__":
    main()
