"""Full-size parity (BASELINE config 2, Llama-3.2-1B, 1,235,814,400 params) in
the launch configuration bench.py times: bench.setup builds the DBuffer,
bench.step runs ONE step (default path), and sampled quantization blocks of
every unit are checked against the oracle, block by block:

  oracle input  = the block's pre-step master / codes / absmax and every
                  rank's bf16 gradient, regenerated from synth (the values
                  bench.setup placed; nothing is read back from the device)
  oracle        = grouped_cast_scale -> reduce_scatter (rank order) ->
                  step_8bit_adam on the block
  check         = codes +-1, params 1e-5 (|p|+lr), absmax 1e-6, bf16 shard

Plus, after a second AllGather (or the one fused into the step for the "+ag"
scopes): every rank's gathered buffer holds, at every other rank's checked
blocks, the oracle's updated bf16 parameters (element-wise, same tolerance),
and the whole gathered arena is byte-identical on every rank (rank 0's
broadcast over gloo, compared element by element).  FULLSIZE_SCOPE = unit | dbuffer | unit+ag | dbuffer+ag.  Runs standalone (world 1) or under
torchrun.  Exit 0 iff all checks pass on every rank.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2602_22437_b200 as R  # noqa: E402
from oracle import adam8 as OA  # noqa: E402
from oracle import dbuffer as OD  # noqa: E402
from oracle import planner as OP  # noqa: E402
from synth import hashgen as H  # noqa: E402

SAMPLES_PER_UNIT = int(os.environ.get("FULLSIZE_SAMPLES", "6"))


def main():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    comm = R.init_comm(rank, world, local)
    units = bench.build_units(16)
    lays, db, arenas, views, _, _ = bench.setup(rank, world, local, units, comm)
    p2p = R.P2P(comm, [arenas[0], arenas[1]])
    rng = np.random.default_rng(1234 + rank)
    picks = []  # (unit, block index, off, len, logical start, pre-step inputs)
    for ui, (u, lay) in enumerate(zip(units, lays)):
        blocks = lay.rank_blocks(rank, bench.QBLOCK)
        if not blocks:
            continue
        idx = sorted(set([0, len(blocks) - 1] +
                         list(rng.integers(0, len(blocks), SAMPLES_PER_UNIT))))
        starts = lay.starts
        numel = [t.numel for t in u.tensors]
        flat0 = np.cumsum([0] + numel)
        v = views[ui]
        for b in idx:
            off, n = blocks[b]
            pos = rank * lay.S + off
            t = max(i for i in range(len(starts)) if starts[i] <= pos)
            logical = int(flat0[t] + pos - starts[t])
            # the oracle's inputs regenerated from synth (what bench.setup placed
            # in the arenas), never read back from the device
            pre = (H.params_np(ui, logical, n),
                   H.codes_np(ui, H.STREAM_MCODE, rank * lay.S + off, n, True),
                   H.codes_np(ui, H.STREAM_VCODE, rank * lay.S + off, n, False),
                   H.absmax_np(ui, H.STREAM_ABSM, rank * 10 ** 7 + b, 1, 14),
                   H.absmax_np(ui, H.STREAM_ABSV, rank * 10 ** 7 + b, 1, 22))
            picks.append((ui, b, off, n, logical, pre))
    cfg = R.AdamConfig()
    st = torch.cuda.Stream()
    scope = os.environ.get("FULLSIZE_SCOPE", "unit")
    with torch.cuda.stream(st):
        bench.step(R, db, cfg, 1, st, p2p=p2p, fuse={"unit": True}.get(scope, scope))
    st.synchronize()
    ok, msgs = True, []
    checked = []  # (unit, global position, len, oracle bf16 bits, oracle master) of every checked block
    ocfg = OA.AdamCfg()
    for ui, b, off, n, logical, pre in picks:
        v = views[ui]
        # oracle: every rank's bf16 gradient for this block, cast/scale, rank-order RS
        mini = OP.Layout(world, 1, [world * n], [1], n, [0])
        bufs = []
        for r in range(world):
            g = np.zeros(world * n, np.float32)
            g[rank * n:(rank + 1) * n] = H.grads_np(ui, r, logical, n)
            bufs.append(OD.grouped_cast_scale(mini, OD.to_bf16_rne(g), True))
        gred = OD.reduce_scatter(mini, bufs)[rank]
        ref = OA.step_8bit_adam(pre[0], gred, pre[1], pre[2], pre[3], pre[4], [(0, n)], ocfg, 1)
        gm = v["master"][off:off + n].cpu().numpy()
        err = np.abs(gm - ref[0]) / (np.abs(ref[0]) + cfg.lr)
        dm = np.abs(v["mq"][off:off + n].cpu().numpy().astype(int) - ref[1].astype(int))
        dv = np.abs(v["vq"][off:off + n].cpu().numpy().astype(int) - ref[2].astype(int))
        ma = v["ma"][b:b + 1].cpu().numpy()
        va = v["va"][b:b + 1].cpu().numpy()
        lay = lays[ui]
        bf = v["param_full"][rank * lay.S + off:rank * lay.S + off + n]
        bfv = OD.bf16_to_f32(bf.view(torch.int16).cpu().numpy().view(np.uint16)).astype(np.float64)
        rv = OD.bf16_to_f32(ref[5]).astype(np.float64)
        r0 = np.abs(ref[0]).astype(np.float64)
        good = (err.max() <= 1e-5 and dm.max() <= 1 and dv.max() <= 1
                and np.all(np.abs(ma - ref[3]) <= 1e-6 * np.abs(ref[3]) + 1e-30)
                and np.all(np.abs(va - ref[4]) <= 1e-6 * np.abs(ref[4]) + 1e-30)
                and np.all(np.abs(bfv - rv) <= 1e-5 * (r0 + cfg.lr) + 2.0 ** -7 * r0))
        if not good:
            ok = False
            msgs.append(f"unit {ui} block {b}: err {err.max():.2e} dm {dm.max()} dv {dv.max()}")
        checked.append((ui, rank * lay.S + off, n, ref[5], ref[0]))
    # AllGather: every rank ends with the same full parameter buffers (the
    # "+ag" scopes already did it inside the fused kernel)
    if not scope.endswith("+ag"):
        with torch.cuda.stream(st):
            for u in db.units:
                R.all_gather_p2p(u, p2p, st)
    st.synchronize()
    # (1) element-wise against the oracle: every rank's checked blocks, read
    # from THIS rank's gathered buffer at the owner's shard position
    allc = [checked]
    if world > 1:
        allc = [None] * world
        dist.all_gather_object(allc, checked)
    for owner, lst in enumerate(allc):
        for ui, pos, n, ref16, ref32 in lst:
            got = views[ui]["param_full"][pos:pos + n].view(torch.int16).cpu().numpy().view(np.uint16)
            gv = OD.bf16_to_f32(got).astype(np.float64)
            rv = OD.bf16_to_f32(ref16).astype(np.float64)
            r0 = np.abs(ref32).astype(np.float64)
            if not np.all(np.abs(gv - rv) <= 1e-5 * (r0 + cfg.lr) + 2.0 ** -7 * r0):
                ok = False
                msgs.append(f"gathered block of rank {owner} (unit {ui}, pos {pos}) differs from the oracle")
    # (2) the whole gathered parameter arena identical on every rank, byte for byte
    if world > 1:
        mine = arenas[0].cpu()
        ref_arena = mine.clone() if rank == 0 else torch.empty_like(mine)
        dist.broadcast(ref_arena, src=0)
        if not torch.equal(mine, ref_arena):
            ok = False
            msgs.append("full parameter buffers differ across ranks after AllGather")
    p2p.close()
    db.close()
    comm.close()
    flag = torch.tensor([0 if ok else 1])
    if world > 1:
        dist.all_reduce(flag)
    if msgs:
        print(f"[rank {rank}] " + "; ".join(msgs[:10]), flush=True)
    if rank == 0:
        print(f"fullsize parity world={world} blocks checked={len(picks)} (rank 0): "
              f"{'PASS' if flag.item() == 0 else 'FAIL'}", flush=True)
    if world > 1:
        dist.destroy_process_group()
    sys.exit(0 if flag.item() == 0 else 1)


if __name__ == "__main__":
    main()
