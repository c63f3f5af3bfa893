#!/usr/bin/env python
"""Fig. 9 of the paper: RaggedShard padding of DeepSeek-V3-671B
and GPT-OSS-120B per-layer FSDP units when the expert FFN weights are sharded
at 1 / 16 / 128-row granularity, over FSDP sizes m, with the C++ planner
(Algorithm 1).  Padding ratio of a model = sum over units of (m*S - E) /
sum of E; also the ratio of each distinct unit kind (root, dense layer, MoE
layer), since a whole-model figure mixes them, and the padding with the best
of P:279's tensor orders (the paper adopts the default order).  Also the planner time ("< 0.3 s").  One JSON line per
(model, rows, m); host only.

  python scripts/fig9_padding.py > profiles/r1/fig9_padding.jsonl
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2602_22437_b200 as R  # noqa: E402
from synth import workloads as W  # noqa: E402

MS = (8, 16, 24, 32, 48, 64, 96, 128, 192, 256, 384, 512, 768, 1024)


def main():
    for name, mk in (("deepseek-v3-671b", W.deepseek_v3_671b), ("gpt-oss-120b", W.gpt_oss_120b)):
        for rows in (1, 16, 128):
            wl = mk(rows)
            # identical layer units plan identically: plan each distinct unit once
            kinds = {}  # key -> [first unit name, count]
            for u in wl.units:
                key = tuple((t.numel, R.block_elems(t.shape, t.gran)) for t in u.tensors)
                kinds.setdefault(key, [u.name, 0])[1] += 1
            for m in MS:
                pad = tot = pad_best = 0
                t_max = 0.0
                per_kind = {}
                for key, (uname, count) in kinds.items():
                    es = [k[0] for k in key]
                    gs = [k[1] for k in key]
                    t0 = time.perf_counter()
                    lay = R.plan(es, gs, m, elem_bytes=2)
                    t_max = max(t_max, time.perf_counter() - t0)
                    pad += count * (m * lay.S - lay.E)
                    tot += count * lay.E
                    best = R.plan_ordered(es, gs, m, "best", elem_bytes=2)  # P:279 orders (N4)
                    pad_best += count * (m * best.S - best.E)
                    per_kind[f"{uname} (x{count})"] = round(100.0 * (m * lay.S - lay.E) / lay.E, 3)
                print(json.dumps({"model": name, "rows": rows, "m": m, "units": len(wl.units),
                                  "params": tot, "padding_pct": 100.0 * pad / tot,
                                  "padding_pct_best_order": 100.0 * pad_best / tot,
                                  "unit_padding_pct": per_kind,
                                  "max_plan_s_per_unit": t_max}), flush=True)


if __name__ == "__main__":
    main()
