#!/usr/bin/env python
"""Benchmark of the RaggedShard/DBuffer collective step (veScale-FSDP, arxiv
2602.22437) on B200.  Contract: see DESIGN.md "Measurement".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
        --master-addr 127.0.0.1 --master-port P bench.py --gpus N ...

Workload (BASELINE.json configs[1]): Llama-3.2-1B-shaped bf16 parameter set,
one FSDP unit per decoder layer plus a root unit (embed + final norm), 2048-
element 8-bit-Adam blocks, all 17 units in one batched DBuffer per rank.
Synthetic, seeded inputs (synth/), random-init weights.

One step (all per-step rows of SURVEY §8(a); a1-a3 planning is one-time at
init, reported as plan_ms):
    for unit in units:            a4  AllGather (in place, zero-copy views a5)
    for unit in reversed(units):  a6  cast bf16->fp32 x 1/m, padding 0
                                  a7  ReduceScatter
                                  a8  block-wise 8-bit Adam (+ bf16 shard)
  --collectives p2p (default): the step is ONE kernel over NVLink peer memory
      for the whole DBuffer (rsdb_dbuffer_reduce_scatter_adam_gather): a6+a7
      (rank-order sum of every rank's bf16 gradient slice), a8 (8-bit Adam of
      the owned blocks) and a4 (each updated bf16 parameter stored into every
      peer's gathered buffer -- the AllGather the next step's forward needs;
      the first step's AllGather runs once at setup).  Variants:
      --no-fuse-ag: rsdb_all_gather_p2p per unit + the fused RS+Adam kernel;
      --fused-scope unit: one fused kernel per unit (FSDP backward order);
      --no-fuse-adam: a6+a7 kernel per unit, then one a8 launch.
  --collectives nccl: ncclAllGather; cast kernel + ncclReduceScatter (fp32) per
      unit; one a8 launch over every shard.

value = BJ's metric as named, from PHYSICAL bytes / max-rank step time:
        N = 1: "8-bit Adam shard HBM GB/s" -- the HBM bytes the step moves
               (fused kernel: 16 B per owned element + 16 B per block);
        N > 1: "AG+RS bus GB/s" -- the NVLink bytes every rank receives for
               the unit AllGathers and ReduceScatters, summed over ranks.
        value_composite_gbs keeps SURVEY §8(d)'s unfused work-normalised
        accounting (24 B per element at N = 1), which is not a physical rate.
extras = scripts/bench_extras.py (configs 3-5, N2 rows, per-unit bus GB/s,
        ZeRO-3 overlap); --no-extras skips them.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AG+RS bus GB/s per FSDP unit at 1/2/4/8 B200; 8-bit Adam shard HBM GB/s"
UNIT = "GB/s"
WORKLOAD = "llama-3.2-1b"
QBLOCK = 2048
ALIGN = 256
L2_BYTES = 126 * 2 ** 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--layers", type=int, default=16)
    ap.add_argument("--e2e-steps", type=int, default=0, help="0: max(3, steps // 10)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the extra measurements (configs 3-5, tiles, dynamic codec, "
                         "per-unit collectives, ZeRO-3 overlap; scripts/bench_extras.py)")
    ap.add_argument("--extras", default="",
                    help="comma-separated subset of the extras to run (default: all)")
    ap.add_argument("--no-fuse-adam", action="store_true",
                    help="p2p path: separate ReduceScatter kernel + one 8-bit Adam launch instead "
                         "of the fused ReduceScatter+Adam kernel")
    ap.add_argument("--fused-scope", choices=["unit", "dbuffer"], default="dbuffer",
                    help="fused kernel per unit (FSDP backward order, 17 launches) or one launch "
                         "over the whole DBuffer (default)")
    ap.add_argument("--fuse-ag", action=argparse.BooleanOptionalAction, default=True,
                    help="p2p + fused Adam: the AllGather is fused into the RS+Adam kernel too "
                         "(each rank pushes its updated bf16 shard into every peer's gathered "
                         "buffer); the step's AllGather is the one the previous step's kernel "
                         "did (default on)")
    ap.add_argument("--collectives", choices=["p2p", "nccl"], default="p2p",
                    help="p2p: fused single-kernel collectives over NVLink peer memory "
                         "(SURVEY N1); nccl: ncclAllGather / cast kernel + ncclReduceScatter")
    ap.add_argument("--watchdog", type=float, default=1800.0,
                    help="after this many seconds every rank prints all its Python stacks and "
                         "exits (faulthandler) instead of hanging until killed; 0 = off (the "
                         "default run takes a few minutes)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


NVLINK_PEAK_GBS = 770.0  # measured per-direction peer bandwidth, B200_PROFILING.md
NVLINK_SPEC_GBS = 900.0  # NVLink 5 per direction per GPU (nominal)
HBM_SPEC_GBS = 8000.0    # B200 HBM3e (nominal)


# ---------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampler (the B200_PROFILING.md clocks line) started before the
    warm-up -- nvidia-smi needs ~0.1-0.3 s to start -- and filtered to samples
    whose own timestamps fall inside [begin(), end()] (the timed region)."""
    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        import threading
        self.gpus = set(gpus)
        self.p = None
        self.t0 = self.t1 = None
        self.lines = []
        self.live = threading.Event()
        try:
            self.p = subprocess.Popen(["nvidia-smi", "--query-gpu=" + self.FIELDS,
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.lines.append(line)
            self.live.set()

    def ready(self):
        """Blocks until the sampler produces lines (nvidia-smi takes 0.1-1 s to
        start; a short N=1 timed region could otherwise end first).  Called
        before the pre-timing barrier so no rank's timing includes the wait."""
        if self.p is not None:
            self.live.wait(timeout=10.0)

    def begin(self):
        self.t0 = time.time()

    def end(self):
        self.t1 = time.time()

    def stop(self):
        if self.p is None:
            return None
        import datetime
        time.sleep(0.12)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        time.sleep(0.05)
        out = "".join(self.lines)
        sm, mx, reasons, n = [], 0.0, set(), 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 10 or not f[1].isdigit() or int(f[1]) not in self.gpus:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            if ts is not None and self.t0 is not None and not (self.t0 - 0.06 <= ts <= self.t1 + 0.06):
                continue
            f = f[1:]
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            n += 1
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": n}


# ---------------------------------------------------------------- NVLink counters
class NvlinkCounters:
    """Cumulative NVLink data counters of this rank's GPU through NVML
    (pynvml field values, summed over links): read around the timed region so
    the wire bytes the line claims are backed by hardware counters
    (VERDICT r1 "NVLink GB/s backed by captures").  Tries the
    per-link data-throughput counters (KiB) and the raw byte counters."""
    FIELDS = (("data", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX", 1024),
              ("bytes", "NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES", 1))

    def __init__(self, device):
        self.ok = False
        self.err = None
        try:
            import pynvml as N
            import torch
            N.nvmlInit()
            self.N = N
            uuid = str(torch.cuda.get_device_properties(device).uuid)
            self.h = N.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            self.ok = True
        except Exception as e:  # recorded in the line
            self.err = f"{type(e).__name__}: {e}"

    def read(self):
        if not self.ok:
            return None
        N, out = self.N, {}
        for name, ftx, frx, unit in self.FIELDS:
            try:
                for d, f in (("tx", ftx), ("rx", frx)):
                    fid = getattr(N, f)
                    vals = N.nvmlDeviceGetFieldValues(self.h, [(fid, link) for link in range(18)])
                    tot, n = 0, 0
                    codes = set()
                    for v in vals:
                        codes.add(int(v.nvmlReturn))
                        if v.nvmlReturn == 0:
                            tot += int(v.value.ullVal)
                            n += 1
                    out[f"{name}_{d}"] = tot * unit if n else None
                    if not n:
                        out[f"{name}_{d}_nvml_return"] = sorted(codes)  # 3 = NOT_SUPPORTED
            except Exception as e:
                out[f"{name}_error"] = f"{type(e).__name__}: {e}"
        return out

    @staticmethod
    def delta(a, b, steps):
        if not a or not b:
            return None
        d = {}
        for k in a:
            if k in b and isinstance(a[k], int) and isinstance(b[k], int):
                d[k + "_bytes_per_step"] = (b[k] - a[k]) / steps
        return d


# ---------------------------------------------------------------- setup
def build_units(n_layers):
    from synth import workloads as W
    wl = W.llama32_1b(QBLOCK, n_layers)
    return wl.units


def setup(rank, world, local, units, comm):
    import torch

    import paper_2602_22437_b200 as R
    from synth import hashgen as H

    t0 = time.perf_counter()
    lays = []
    for u in units:
        es = [t.numel for t in u.tensors]
        gs = [R.block_elems(t.shape, t.gran) for t in u.tensors]
        lays.append(R.plan(es, gs, world, elem_bytes=2))
    plan_ms = (time.perf_counter() - t0) * 1e3
    sizes, offs = R.arena_sizes(lays, rank, QBLOCK, ALIGN)
    dev = torch.device("cuda", local)
    arenas = [torch.zeros(max(1, s), dtype=torch.uint8, device=dev) for s in sizes]
    db = R.DBuffer(lays, rank, arenas, qblock=QBLOCK, align=ALIGN, comm=comm)
    # fill: logical params / grads from the counter hash, placed through the views
    views = []
    for ui, (u, lay) in enumerate(zip(units, lays)):
        S, m = lay.S, lay.m
        off = offs[ui]
        nb = len(lay.rank_blocks(rank, QBLOCK))
        v = {
            "param_full": arenas[0][off[0]:off[0] + m * S * 2].view(torch.bfloat16),
            "grad_full": arenas[1][off[1]:off[1] + m * S * 2].view(torch.bfloat16),
            "grad_f32": arenas[2][off[2]:off[2] + m * S * 4].view(torch.float32),
            "master": arenas[3][off[3]:off[3] + S * 4].view(torch.float32),
            "mq": arenas[4][off[4]:off[4] + S].view(torch.int8),
            "vq": arenas[5][off[5]:off[5] + S],
            "ma": arenas[6][off[6]:off[6] + nb * 4].view(torch.float32),
            "va": arenas[7][off[7]:off[7] + nb * 4].view(torch.float32),
        }
        E = lay.E
        p = H.params_torch(ui, 0, E, device=dev)
        g = H.grads_torch(ui, rank, 0, E, device=dev)
        full_p = torch.zeros(m * S, dtype=torch.float32, device=dev)
        o = 0
        for l, e in zip(lay.starts, [t.numel for t in u.tensors]):
            full_p[l:l + e] = p[o:o + e]
            v["grad_full"][l:l + e] = g[o:o + e].to(torch.bfloat16)
            o += e
        v["param_full"].copy_(full_p.to(torch.bfloat16))
        v["master"].copy_(full_p[rank * S:(rank + 1) * S])
        # warm synthetic 8-bit Adam state (codes + per-block absmax)
        v["mq"].copy_(H.codes_torch(ui, H.STREAM_MCODE, rank * S, S, True, device=dev))
        v["vq"].copy_(H.codes_torch(ui, H.STREAM_VCODE, rank * S, S, False, device=dev))
        v["ma"].copy_(H.absmax_torch(ui, H.STREAM_ABSM, rank * 10 ** 7, nb, 14, device=dev))
        v["va"].copy_(H.absmax_torch(ui, H.STREAM_ABSV, rank * 10 ** 7, nb, 22, device=dev))
        del p, g, full_p
        views.append(v)
    torch.cuda.synchronize()
    return lays, db, arenas, views, plan_ms, sizes


def algorithmic_bytes(lays, rank):
    """Per-rank algorithmic bytes of one step, by row."""
    ag = rs = cast = adam = 0
    n_el = n_blk = 0
    for lay in lays:
        m, S = lay.m, lay.S
        ag += (m - 1) * S * 2
        rs += (m - 1) * S * 4
        cast += m * S * 6
        blocks = lay.rank_blocks(rank, QBLOCK)
        el = sum(n for _, n in blocks)
        n_el += el
        n_blk += len(blocks)
    adam = 18 * n_el + 16 * n_blk
    return {"ag": ag, "rs": rs, "cast": cast, "adam": adam, "adam_elems": n_el,
            "adam_blocks": n_blk}


# ---------------------------------------------------------------- step
class Timers:
    """CUDA event pairs on the launching stream around each op kind."""

    def __init__(self):
        self.pairs = {"ag": [], "cast": [], "rs": [], "adam": []}

    def rec(self, kind, stream):
        import torch
        a = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        return a

    def add(self, kind, a, b):
        self.pairs[kind].append((a, b))

    def totals_ms(self):
        return {k: sum(a.elapsed_time(b) for a, b in v) for k, v in self.pairs.items()}

    def counts(self):
        return {k: len(v) for k, v in self.pairs.items()}


def step(R, db, cfg, t, stream, timers=None, p2p=None, fuse=False):
    """One step.  p2p=None: NCCL AllGather, cast kernel + NCCL fp32
    ReduceScatter, one 8-bit Adam launch.  p2p given: the single-kernel
    collectives over NVLink peer memory; the cast is inside the
    ReduceScatter kernel, and with fuse=True the 8-bit Adam update of each
    unit's shard is inside it too (rsdb_reduce_scatter_adam_p2p)."""
    import torch
    units = db.units

    def timed(kind, fn):
        if timers is None:
            fn()
            return
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        timers.add(kind, a, b)

    if p2p is None:
        for u in units:
            timed("ag", lambda u=u: R.all_gather(u, stream))
        for u in reversed(units):
            timed("cast", lambda u=u: R.unit_cast_scale(u, stream))
            timed("rs", lambda u=u: R.unit_reduce_scatter_f32(u, stream))
    else:
        if fuse not in ("dbuffer+ag", "unit+ag"):  # else fused into the previous step
            for u in units:
                timed("ag", lambda u=u: R.all_gather_p2p(u, p2p, stream))
        if fuse == "dbuffer":  # a6 + a7 + a8 for every unit in ONE launch
            timed("rs", lambda: db.reduce_scatter_adam(cfg, t, p2p if db.units[0].layout.m > 1
                                                       else None, stream))
            return
        if fuse == "dbuffer+ag":  # a6 + a7 + a8 + (next) a4, every unit, ONE launch
            timed("rs", lambda: db.reduce_scatter_adam_gather(
                cfg, t, p2p if db.units[0].layout.m > 1 else None, stream))
            return
        if fuse == "unit+ag":  # a6 + a7 + a8 + (next) a4, one kernel per unit
            for u in reversed(units):
                timed("rs", lambda u=u: R.reduce_scatter_adam_gather_p2p(u, p2p, cfg, t,
                                                                           stream=stream))
            return
        if fuse:  # a6 + a7 + a8: one kernel per unit (FSDP backward order), no optimizer launch
            for u in reversed(units):
                timed("rs", lambda u=u: R.reduce_scatter_adam_p2p(u, p2p, cfg, t, stream=stream))
            return
        for u in reversed(units):
            timed("rs", lambda u=u: R.reduce_scatter_p2p(u, p2p, stream))
    timed("adam", lambda: db.step_8bit_adam(cfg, t, stream))


def barrier(world):
    import torch.distributed as dist
    if world > 1:
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def sum_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.item()


def profile_traffic(kernel):
    """dram bytes per launch of `kernel` from the committed ncu summary (or None)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(kernel)
        if e and e.get("workload") == WORKLOAD and e.get("n_gpus") == 1:
            return e["dram_bytes_per_launch"]
    except Exception:
        pass
    return None


def profile_nvlink(kernel, world):
    """NVLink bytes per launch of `kernel` at this world size from the
    committed ncu capture (profiles/ncu_nvlink.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_nvlink.json")
    try:
        with open(p) as f:
            es = json.load(f).get(kernel)
        for e in (es if isinstance(es, list) else [es]):  # one capture per world size
            if e and e.get("workload") == WORKLOAD and e.get("n_gpus") == world:
                return e
    except Exception:
        pass
    return None


# ---------------------------------------------------------------- CPU baseline (oracle)
_ORACLE_INPUTS = {}


def oracle_sample_step(world, n_blocks, seed=0, phases=None):
    """The oracle (as it stands) on a bounded sample of the workload: a slice
    of n_blocks 2048-element blocks of the layer unit, planned for `world`
    simulated ranks; AG, cast/scale, RS and 8-bit Adam for EVERY rank.
    Inputs are generated once per (world, n_blocks) outside the timing.
    Returns (seconds, whole-job algorithmic bytes, elements); `phases`, if a
    dict, receives the seconds of each op."""
    import numpy as np

    from oracle import adam8 as OA
    from oracle import dbuffer as OD
    from oracle import planner as OP
    from synth import hashgen as H

    key = (world, n_blocks, seed)
    if key not in _ORACLE_INPUTS:
        _ORACLE_INPUTS.clear()
        E = n_blocks * QBLOCK
        o = OP.plan([E], [QBLOCK], world, OP.gcoll_elems(2))
        p_log = H.params_np(seed, 0, E)
        grads = [OD.to_bf16_rne(OD.place_logical(o, H.grads_np(seed, r, 0, E)))
                 for r in range(world)]
        _ORACLE_INPUTS[key] = (o, grads, OD.to_bf16_rne(OD.place_logical(o, p_log)),
                               OD.place_logical(o, p_log))
    o, grads, params16, master = _ORACLE_INPUTS[key]
    E, S = o.E, o.S
    t0 = time.perf_counter()
    OD.all_gather([OD.shard(o, params16, k) for k in range(world)])
    t1 = time.perf_counter()
    xs = [OD.grouped_cast_scale(o, g, True) for g in grads]
    t2 = time.perf_counter()
    ys = OD.reduce_scatter(o, xs)
    t3 = time.perf_counter()
    for r in range(world):
        blocks = OP.rank_blocks(o, r, QBLOCK)
        nb = len(blocks)
        OA.step_8bit_adam(OD.shard(o, master, r), ys[r], np.zeros(S, np.int8),
                          np.zeros(S, np.uint8), np.zeros(nb, np.float32),
                          np.zeros(nb, np.float32), blocks, OA.AdamCfg(), 1)
    t4 = time.perf_counter()
    if phases is not None:
        phases.update({"ag_s": t1 - t0, "cast_s": t2 - t1, "rs_s": t3 - t2, "adam_s": t4 - t3})
    dt = t4 - t0
    return dt, metric_bytes(world, S, E, n_blocks), E


def metric_bytes(world, S, E, n_blocks):
    """Bytes the line's `value` counts for one step of work (run_ours's value
    definition, so both arms report the same metric for the same work):
    world 1 -- the fused step's HBM bytes, 16 B per element + 16 B per block;
    world m > 1 -- every rank's AG + RS wire bytes, m * 2 (m-1) S 2."""
    if world == 1:
        return 16 * E + 16 * n_blocks
    return world * 2 * (world - 1) * S * 2


def _mp_worker(args):
    world, n_blocks, seed = args
    dt, nb, E = oracle_sample_step(world, n_blocks, seed)  # inputs (untimed), then warm
    t0 = time.perf_counter()
    dt, nb, E = oracle_sample_step(world, n_blocks, seed)
    return t0, time.perf_counter(), nb, E


def cpu_baseline(world, target_s=10.0, procs=8):
    """The oracle on the host cores (SURVEY §8(d) 'oracle beside it'):
    one process, numpy single thread, on a calibrated sample of the layer
    unit; per-op seconds of that sample; the oracle planner's time per unit
    (the two unit kinds of the workload); and a multi-process variant
    (`procs` worker processes, one core each, every worker running the same
    single-process oracle step on its own slice of the workload)."""
    import multiprocessing as mp

    from oracle import planner as OP
    dt, nb, E = oracle_sample_step(world, 256)
    blocks = max(256, int(256 * target_s / max(dt, 1e-3)))
    blocks = min(blocks, 1 << 16)
    ph = {}
    dt, nb, E = oracle_sample_step(world, blocks, phases=ph)
    _ORACLE_INPUTS.clear()
    # planner per unit (one-time, host): the oracle's Algorithm 1
    plan_s = {}
    for name, u in (("layer", build_units(1)[1]), ("root", build_units(1)[0])):
        es = [t.numel for t in u.tensors]
        gs = [min(QBLOCK, e) for e in es]
        t0 = time.perf_counter()
        OP.plan(es, gs, world, OP.gcoll_elems(2))
        plan_s[name] = time.perf_counter() - t0
    # multi-process: `procs` workers, each 1/procs of the sample
    mp_res = None
    try:
        per = max(16, blocks // procs)
        ctx = mp.get_context("fork")
        with ctx.Pool(procs) as pool:
            rs = pool.map(_mp_worker, [(world, per, 100 + i) for i in range(procs)])
        t_beg, t_end = min(r[0] for r in rs), max(r[1] for r in rs)
        mp_bytes = sum(r[2] for r in rs)
        mp_res = {"value": mp_bytes / (t_end - t_beg) / 1e9, "unit": UNIT, "cores": procs,
                  "sample": f"{procs} processes x {per} blocks (2048 elem) each, the same "
                            f"single-process oracle step per worker, {t_end - t_beg:.1f} s wall"}
    except Exception as e:  # recorded, not hidden
        mp_res = {"error": f"{type(e).__name__}: {e}"}
    return {"value": nb / dt / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{E} params ({blocks} x 2048-elem blocks of the layer unit), "
                      f"{world} simulated rank(s), AG+cast+RS+8-bit Adam, numpy single thread, "
                      f"{dt:.1f} s", "host": host_info(),
            "per_op_s": ph, "per_op_gbs": {
                "adam": (18 * E + 16 * blocks) / ph["adam_s"] / 1e9,
                "cast": world * world * (E // world) * 6 / ph["cast_s"] / 1e9},
            "planner_s_per_unit": plan_s, "multiprocess": mp_res}


def host_info():
    """CPU model and the cores this process may use (SURVEY §8(d) 'oracle beside it')."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = os.cpu_count()
    return {"cpu_model": model, "affinity_cores": aff}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    # calibrate: the whole --steps K --warmup W run should take ~2 minutes
    dt, _, _ = oracle_sample_step(world, 64)
    per_step = 120.0 / max(1, args.steps + args.warmup)
    blocks = max(16, min(1 << 15, int(64 * per_step / max(dt, 1e-4))))
    for _ in range(args.warmup):
        oracle_sample_step(world, blocks)
    tot_t = tot_b = 0.0
    E = 0
    for _ in range(args.steps):
        dt, nb, E = oracle_sample_step(world, blocks)
        tot_t += dt
        tot_b += nb
    value = tot_b / tot_t / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot_t / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(workload_config(args, world),
                           sample="bounded oracle sample of the layer unit, every simulated rank"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{E} params per step ({blocks} blocks), {world} "
                                       "simulated rank(s), numpy single thread",
                             "host": host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# The paper's own results (whole training systems, not this kernel metric): context only
PAPER_CONTEXT = {
    "throughput": "+5 % (LLaMA-3-70B) to +66 % (MoE) vs DeepSpeed / FSDP1 / FSDP2 / Megatron-FSDP (P:27, P:369)",
    "memory": "-16 % to -30 % peak reserved memory (P:372)",
    "ablation": "DBuffer off: 92.8 % of full throughput; planner off: 65.4 % (GPT-OSS-style model, "
                "8-bit Adam, 32 GPUs; P:511-527)",
    "hardware": "H800 cluster (8 GPUs per node, 400 GB/s NVLink), 128-1,024 GPUs (P:336, P:362, P:367)",
    "note": "no per-collective or per-kernel number in the paper (BASELINE.md §1): vs_baseline stays null",
}


def workload_config(args, world):
    """config keys shared by both arms (the reference arm runs the oracle on a
    bounded sample of THIS workload; its `cpu_baseline.sample` says which)."""
    units = build_units(args.layers)
    E = sum(t.numel for u in units for t in u.tensors)
    return {"workload": f"{WORKLOAD}: {len(units)} FSDP units (root + {args.layers} layers), {E} params, "
                        "bf16 params/grads, 2048-elem 8-bit Adam blocks, warm synthetic states",
            "units": len(units), "params": E, "qblock": QBLOCK, "parallelism": f"fsdp{world}"}


# ---------------------------------------------------------------- main arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2602_22437_b200 as R

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    comm = R.init_comm(rank, world, local)
    units = build_units(args.layers)
    lays, db, arenas, views, plan_ms, sizes = setup(rank, world, local, units, comm)
    p2p = None
    if args.collectives == "p2p":
        p2p = R.P2P(comm, [arenas[0], arenas[1]])  # PARAM_FULL, GRAD_FULL arenas
    fuse = p2p is not None and not args.no_fuse_adam
    if fuse:
        scope = args.fused_scope
        fuse = "dbuffer" if scope == "dbuffer" else True
        if args.fuse_ag:
            fuse = "dbuffer+ag" if scope == "dbuffer" else "unit+ag"
            for u in db.units:  # the first step's AllGather (steady state: the previous step's)
                R.all_gather_p2p(u, p2p)
            torch.cuda.synchronize()
    ab = algorithmic_bytes(lays, rank)
    per_rank_bytes = ab["ag"] + ab["rs"] + ab["cast"] + ab["adam"]
    job_bytes = sum_over_ranks(per_rank_bytes, world)
    cfg = R.AdamConfig()
    stream = torch.cuda.Stream()
    clocks = Clocks(range(world)) if rank == 0 else None  # started early: nvidia-smi is slow to start
    t = 1
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step(R, db, cfg, t, stream, p2p=p2p, fuse=fuse)
            t += 1
    stream.synchronize()
    # ---------------- timed region: inputs resident in HBM
    timers = Timers()
    if clocks:
        clocks.ready()
    barrier(world)
    torch.cuda.synchronize()
    if clocks:
        clocks.begin()
    nvl = NvlinkCounters(local) if world > 1 else None
    nvl0 = nvl.read() if nvl else None
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if p2p is not None and world > 1:
        # align the ranks' streams ON THE DEVICE before the first event: the
        # host barrier + synchronize leave the ranks' launch times skewed by
        # milliseconds, which would otherwise be charged to the first step
        p2p.barrier(stream)
    ev0.record(stream)
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            if i:
                step_ev[i - 1].record(stream)  # step boundaries: per-step distribution
            step(R, db, cfg, t, stream, timers, p2p=p2p, fuse=fuse)
            t += 1
    ev1.record(stream)
    torch.cuda.synchronize()
    nvl1 = nvl.read() if nvl else None
    if clocks:
        clocks.end()
    barrier(world)
    clk = clocks.stop() if clocks else None
    ms_local = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms_local, world)
    bounds = [ev0] + step_ev[:args.steps - 1] + [ev1]
    per_step = sorted(bounds[i].elapsed_time(bounds[i + 1]) for i in range(args.steps))
    pct = lambda q: per_step[min(len(per_step) - 1, int(q * (len(per_step) - 1) + 0.5))]  # noqa: E731
    step_dist = {"p10": pct(0.1), "p50": pct(0.5), "p90": pct(0.9), "rank": rank,
                 "note": "rank 0's per-step CUDA-event times inside the timed region"}
    tot = timers.totals_ms()
    cnt = timers.counts()
    K = args.steps
    # per-op rates on this rank (per launch averages)
    adam_ms = tot["adam"] / max(1, cnt["adam"])
    cast_ms = tot["cast"] / K
    ag_ms, rs_ms = tot["ag"] / K, tot["rs"] / K
    fuse_ag = fuse in ("dbuffer+ag", "unit+ag")
    adam_gbs = ab["adam"] / (adam_ms * 1e-3) / 1e9 if adam_ms > 0 else None  # fused: inside RS
    cast_gbs = ab["cast"] / (cast_ms * 1e-3) / 1e9 if cast_ms > 0 else None  # p2p: fused into RS
    # physical bytes crossing NVLink into each rank per step: AG (m-1) S 2;
    # RS (m-1) S 4 on the NCCL fp32 path, (m-1) S 2 on the fused p2p path
    wire_ag = ab["ag"]
    wire_rs = ab["rs"] if p2p is None else ab["rs"] // 2
    ag_bus = wire_ag / (ag_ms * 1e-3) / 1e9 if world > 1 and ag_ms > 0 else None
    rs_bus = wire_rs / (rs_ms * 1e-3) / 1e9 if world > 1 else None
    hbm_peak, peak_src = load_peaks()
    # fused kernel (a6+a7+a8): HBM bytes per rank per step = every element of
    # this rank's bf16 gradient buffer read once (by whichever rank owns it)
    # + 14 B per owned element (fp32 master R+W, codes R+W, bf16 shard W)
    # + 16 B of absmax per block
    fused_hbm = (sum(l.m * l.S * 2 for l in lays) + 14 * ab["adam_elems"] + 16 * ab["adam_blocks"])
    fused_gbs = fused_hbm / (rs_ms * 1e-3) / 1e9 if fuse else None
    # dominant kernel of the step (largest share of device time)
    names = ({"ag": "nccl_all_gather", "rs": "nccl_reduce_scatter"} if p2p is None else
             {"ag": "ag_p2p (copy engines)", "rs": "rs_adam_tma_kernel" if fuse else "rs_tma_kernel"})
    adam_name = "adam8_tma_kernel"
    shares = {adam_name: tot["adam"], "cast_scale_kernel": tot["cast"],
              names["rs"]: tot["rs"], names["ag"]: tot["ag"]}
    dom = max(shares, key=shares.get)
    if fuse and dom == names["rs"]:
        if world == 1:
            roof = {"kernel": dom, "bound": "hbm", "achieved": fused_gbs, "peak": hbm_peak,
                    "unit": "GB/s", "frac": fused_gbs / hbm_peak,
                    "traffic": profile_traffic(dom), "peak_source": peak_src,
                    "bytes": "16 B per owned element (bf16 grad 2, master 8, codes 4, bf16 out 2) "
                             "+ 16 B absmax per block"}
        else:
            # bytes entering each rank over NVLink per launch: the peers' gradient
            # slices it reads ((m-1) S 2); with the AllGather fused in, also the
            # peers' updated parameter shards pushed into it ((m-1) S 2 more).
            # The outbound direction carries the same amount (its slices read by
            # the peers + its own pushes), so this is the per-direction load.
            wire_in = wire_rs + (wire_ag if fuse_ag else 0)
            ach = wire_in / (rs_ms * 1e-3) / 1e9
            nv = profile_nvlink(dom, world)
            roof = {"kernel": dom, "bound": "nvlink", "achieved": ach, "peak": NVLINK_PEAK_GBS,
                    "unit": "GB/s", "frac": ach / NVLINK_PEAK_GBS,
                    "traffic": nv["nvlrx_bytes_per_launch"] if nv else None,
                    "traffic_user": nv["nvlrx_user_bytes_per_launch"] if nv else None,
                    "traffic_source": (nv["source"] + ": ncu nvlrx__bytes (all NVLink bytes in, protocol "
                                       "included) / nvlrx__bytes_data_user (payload)") if nv else None,
                    "bytes": "physical wire bytes into each rank per launch: (m-1) S 2 gradient "
                             "reads" + (" + (m-1) S 2 parameter pushes from the peers (the fused "
                                        "AllGather)" if fuse_ag else ""),
                    "hbm_achieved": fused_gbs, "hbm_frac": fused_gbs / hbm_peak,
                    "peak_source": "measured peer copy per direction (B200_PROFILING.md)"}
    elif dom in (adam_name, "cast_scale_kernel") or world == 1:
        if dom not in (adam_name, "cast_scale_kernel"):
            dom = adam_name
        ach = adam_gbs if dom == adam_name else cast_gbs
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                "frac": ach / hbm_peak, "traffic": profile_traffic(dom), "peak_source": peak_src}
    else:
        ach = rs_bus if dom == names["rs"] else ag_bus
        roof = {"kernel": dom, "bound": "nvlink", "achieved": ach, "peak": NVLINK_PEAK_GBS,
                "unit": "GB/s", "frac": ach / NVLINK_PEAK_GBS, "traffic": None,
                "bytes": "physical wire bytes into each rank per launch",
                "peak_source": "measured peer copy per direction (B200_PROFILING.md)"}
    roof["share_of_step"] = shares[dom] / max(1e-9, ms_local)
    spec = HBM_SPEC_GBS if roof["bound"] == "hbm" else NVLINK_SPEC_GBS
    roof["frac_vs_spec"] = roof["achieved"] / spec
    roof["spec_peak"] = spec
    # value = BJ's metric as named, physical bytes only (never above the peaks):
    #   N = 1: 8-bit Adam shard HBM GB/s -- the HBM bytes the step's kernels
    #          move (fused: 16 B per owned element + 16 B per block; unfused:
    #          cast m S 6 + Adam 18 B per element + 16 B per block), summed
    #          over ranks, / step time;
    #   N > 1: AG+RS bus GB/s -- the bytes each rank receives over NVLink for
    #          the unit collectives (AG (m-1) S 2; RS (m-1) S 2 on the fused
    #          p2p path (bf16 wire), (m-1) S 4 for NCCL's fp32 RS), summed over
    #          ranks, / step time.
    if fuse:
        hbm_rank = fused_hbm
    else:
        hbm_rank = ab["cast"] + ab["adam"]
    wire_rank = wire_ag + wire_rs
    if world == 1:
        value_bytes = sum_over_ranks(hbm_rank, world)
        value_def = ("8-bit Adam shard HBM GB/s (whole job): physical HBM bytes of the step "
                     "(fused: 16 B/owned elem + 16 B/block) / step time")
    else:
        value_bytes = sum_over_ranks(wire_rank, world)
        value_def = ("AG+RS bus GB/s (whole job, sum over ranks): NVLink bytes into each rank "
                     "for the unit AllGathers and ReduceScatters / step time")
    value = value_bytes / (ms / K * 1e-3) / 1e9
    nvlink = None
    if nvl is not None:
        nvlink = {"rank": rank, "counters": NvlinkCounters.delta(nvl0, nvl1, K),
                  "error": nvl.err, "nvml_raw": nvl1, "algorithmic_wire_in_bytes_per_step": wire_rank,
                  "ncu": "profiles/ncu_nvlink.json (nvlrx__bytes / nvltx__bytes of the fused kernel at "
                         "N = 2 and 4, one process driving the GPUs: scripts/ncu_nvlink_local.py)",
                  "note": "NVML NVLink counters of this rank's GPU around the timed region "
                          "(all links; data = payload KiB counters, bytes = raw link bytes)"}
        if nvlink["counters"]:
            for k, v in list(nvlink["counters"].items()):
                nvlink[k.replace("_bytes_per_step", "_gbs")] = v / (ms / K * 1e-3) / 1e9
    composite = job_bytes / (ms / K * 1e-3) / 1e9
    hbm_job = sum_over_ranks(hbm_rank, world) / (ms / K * 1e-3) / 1e9
    bus_job = sum_over_ranks(wire_rank, world) / (ms / K * 1e-3) / 1e9 if world > 1 else None

    # ---------------- e2e: host buffers through the C-ABI, copies inside
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(R, db, lays, views, cfg, t, stream, world, rank, args, value_bytes, p2p, fuse)
    # ---------------- extras (scripts/bench_extras.py): configs 3-5, N2 rows, per-unit bus
    extras = None
    if not args.no_extras:
        import importlib.util
        spec_ = importlib.util.spec_from_file_location(
            "bench_extras", os.path.join(ROOT, "scripts", "bench_extras.py"))
        BX = importlib.util.module_from_spec(spec_)
        spec_.loader.exec_module(BX)
        ctx = {"rank": rank, "world": world, "comm": comm, "stream": stream, "db": db,
               "lays": lays, "cfg": cfg, "t": t + 1000, "p2p": p2p, "reps": 10}
        which = set(x for x in args.extras.split(",") if x) or None
        extras = BX.run_all(R, ctx, which)
    # ---------------- CPU baseline (oracle) on rank 0
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(world)
    barrier(world)
    if rank == 0:
        E = sum(l.E for l in lays)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {**workload_config(args, world),
                       "collectives": args.collectives,
                       "fused": {"dbuffer": "rs+adam, one launch per step",
                                 True: "rs+adam, one launch per unit",
                                 "dbuffer+ag": "rs+adam+allgather, one launch per step",
                                 "unit+ag": "rs+adam+allgather, one launch per unit",
                                 False: "none"}[fuse],
                       "l2": f"no flush: per-step working set {sum(sizes) / 2 ** 30:.1f} GiB "
                             f"per rank >> L2 ({L2_BYTES >> 20} MiB)",
                       "plan_ms": plan_ms},
            "value_definition": value_def,
            "value_composite_gbs": composite,
            "value_composite_definition": "SURVEY §8(d) unfused algorithmic bytes (AG (m-1)S2 + "
                                          "RS (m-1)S4 + cast mS6 + Adam 18/elem + 16/block) / step "
                                          "time: work-normalised, NOT a physical rate (the fused "
                                          "kernel moves fewer bytes)",
            "hbm_gbs_job": hbm_job, "ag_rs_bus_gbs_job": bus_job,
            "params_updated_per_s": sum(l.E for l in lays) / (ms / K * 1e-3),
            "paper_context": PAPER_CONTEXT,
            "scaling_note": ("value is BJ's metric as named: HBM GB/s at N = 1, AG+RS bus GB/s at N > 1 "
                             "(no collective bytes exist at N = 1), so value_N / value_1 is not a scaling "
                             "ratio; compare ag_rs_bus_gbs_job across N > 1 and params_updated_per_s "
                             "(the same 1.24 B-parameter step at every N) across all N"),
            "step_ms": step_dist,
            "per_op": {"adam_hbm_gbs": adam_gbs, "adam_ms_per_launch": adam_ms,
                       "cast_hbm_gbs": cast_gbs, "cast_ms_per_step": cast_ms,
                       "ag_wire_gbs": ag_bus, "rs_wire_gbs": rs_bus,
                       "fused_rs_adam": fuse, "fused_hbm_gbs": fused_gbs,
                       "ag_wire_bytes_per_rank": wire_ag, "rs_wire_bytes_per_rank": wire_rs,
                       "ag_ms_per_step": ag_ms, "rs_ms_per_step": rs_ms,
                       "bytes_per_rank": ab},
            "roofline": roof,
            "nvlink_counters": nvlink,
            "clocks": clk,
            # this library's kernels in the timed region (world 1: the p2p
            # AllGather is the identity and launches nothing)
            "gpu_launches": (cnt["cast"] + cnt["adam"] +
                             (0 if p2p is None else (cnt["ag"] if world > 1 else 0) + cnt["rs"])),
            "nccl_calls": 0 if p2p is not None else cnt["ag"] + cnt["rs"],
            "cpu_baseline": cpu,
            "e2e": e2e,
            "extras": extras,
        }
        print(json.dumps(line), flush=True)
    if p2p is not None:
        torch.cuda.synchronize()
        p2p.close()
    db.close()
    comm.close()
    if world > 1:
        dist.destroy_process_group()


def run_e2e(R, db, lays, views, cfg, t, stream, world, rank, args, job_bytes, p2p=None, fuse=False):
    """Same metric (job_bytes per step), end to end through the public C-ABI
    with HOST buffers: every step copies this rank's bf16 gradient buffers in
    from pinned host memory and the updated bf16 parameter shards back out,
    inside the timed region.  Fused p2p paths: ONE library call per step,
    rsdb_dbuffer_step_host, which pipelines per unit (H2D copy stream | fused
    kernel | D2H copy stream) inside the library; other paths: the copies and
    the step's calls serially on one stream."""
    import torch
    K = args.e2e_steps or max(3, args.steps // 10)
    host_g, host_p = [], []
    for v, lay in zip(views, lays):
        host_g.append(v["grad_full"].cpu().pin_memory())
        host_p.append(torch.empty(lay.S, dtype=torch.bfloat16).pin_memory())
    h2d = sum_over_ranks(sum(h.numel() * 2 for h in host_g), world)  # whole job
    d2h = sum_over_ranks(sum(h.numel() * 2 for h in host_p), world)

    def e2e_step(tt):
        for v, h in zip(views, host_g):
            v["grad_full"].copy_(h, non_blocking=True)
        for u in db.units:
            if p2p is None:
                R.all_gather(u, stream)
            elif fuse not in ("dbuffer+ag", "unit+ag"):
                R.all_gather_p2p(u, p2p, stream)
        if fuse == "dbuffer":
            db.reduce_scatter_adam(cfg, tt, p2p if world > 1 else None, stream)
        elif fuse == "dbuffer+ag":
            db.reduce_scatter_adam_gather(cfg, tt, p2p if world > 1 else None, stream)
        elif fuse == "unit+ag":
            for u in reversed(db.units):
                R.reduce_scatter_adam_gather_p2p(u, p2p, cfg, tt, stream=stream)
        else:
            for u in reversed(db.units):
                if p2p is None:
                    R.reduce_scatter(u, stream)
                elif fuse:
                    R.reduce_scatter_adam_p2p(u, p2p, cfg, tt, stream=stream)
                else:
                    R.reduce_scatter_p2p(u, p2p, stream)
        if not fuse:
            db.step_8bit_adam(cfg, tt, stream)
        for v, h, lay in zip(views, host_p, lays):
            h.copy_(v["param_full"][rank * lay.S:(rank + 1) * lay.S], non_blocking=True)

    pipelined = p2p is not None and fuse in (True, "unit+ag", "dbuffer", "dbuffer+ag")

    def e2e_step_host(tt):  # the library's host-buffer entry point
        db.step_host(cfg, tt, host_g, host_p, p2p if world > 1 else None, stream)

    if pipelined:
        for u in db.units:  # the first step's AllGather (the kernels push the following ones)
            R.all_gather_p2p(u, p2p, stream)
    run = e2e_step_host if pipelined else e2e_step
    with torch.cuda.stream(stream):
        run(t)
        t += 1
    torch.cuda.synchronize()
    barrier(world)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    with torch.cuda.stream(stream):
        for _ in range(K):
            run(t)
            t += 1
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(ev0.elapsed_time(ev1), world)
    return {"value": job_bytes / (ms / K * 1e-3) / 1e9, "unit": UNIT, "steps": K,
            "ms_per_step": ms / K, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "api": "rsdb_dbuffer_step_host (host buffers through the C-ABI)" if pipelined
                   else "rsdb_* device calls + torch pinned copies",
            "schedule": ("per-unit pipeline inside the library: H2D copy stream | fused kernel | "
                         "D2H copy stream" if pipelined else "serial on one stream")}


def main():
    args = parse()
    if args.watchdog > 0:
        import faulthandler
        faulthandler.dump_traceback_later(args.watchdog, exit=True)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
