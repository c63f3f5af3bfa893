#!/usr/bin/env python
"""Kernel micro-benchmark (1 GPU): the Adam and cast kernels on the
Llama-3.2-1B DBuffer of bench.py, timed with CUDA events over KB_REPS
repetitions (default 20).  Prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_22437_b200 as R  # noqa: E402


def main():
    reps = int(os.environ.get("KB_REPS", "20"))
    torch.cuda.set_device(0)
    comm = R.init_comm(0, 1, 0)
    units = bench.build_units(16)
    lays, db, arenas, views, plan_ms, sizes = bench.setup(0, 1, 0, units, comm)
    ab = bench.algorithmic_bytes(lays, 0)
    cfg = R.AdamConfig()
    st = torch.cuda.Stream()
    for t in range(1, 4):
        db.step_8bit_adam(cfg, t, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.synchronize()
    e0.record(st)
    for t in range(4, 4 + reps):
        db.step_8bit_adam(cfg, t, st)
    e1.record(st)
    st.synchronize()
    adam_ms = e0.elapsed_time(e1) / reps
    # cast over every unit
    for u in db.units:
        R.unit_cast_scale(u, st)
    e0.record(st)
    for _ in range(reps):
        for u in db.units:
            R.unit_cast_scale(u, st)
    e1.record(st)
    st.synchronize()
    cast_ms = e0.elapsed_time(e1) / reps
    # 8-bit Adam with the dynamic (tree) code map (N2, R25) on the same DBuffer
    # (the warm linear codes are valid uint8 map indices too)
    for t in range(1, 3):
        db.step_8bit_adam_dynamic(cfg, t, st)
    st.synchronize()
    e0.record(st)
    for t in range(3, 3 + reps):
        db.step_8bit_adam_dynamic(cfg, t, st)
    e1.record(st)
    st.synchronize()
    dyn_ms = e0.elapsed_time(e1) / reps
    peak, _ = bench.load_peaks()
    out = {"adam_ms": adam_ms, "adam_gbs": ab["adam"] / adam_ms / 1e6,
           "adam_frac": ab["adam"] / adam_ms / 1e6 / peak,
           "cast_ms": cast_ms, "cast_gbs": ab["cast"] / cast_ms / 1e6,
           "cast_frac": ab["cast"] / cast_ms / 1e6 / peak,
           "adam_dynamic_ms": dyn_ms, "adam_dynamic_gbs": ab["adam"] / dyn_ms / 1e6,
           "adam_dynamic_frac": ab["adam"] / dyn_ms / 1e6 / peak}
    print(json.dumps(out), flush=True)
    db.close()
    comm.close()


if __name__ == "__main__":
    main()
