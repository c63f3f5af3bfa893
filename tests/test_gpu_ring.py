"""-m gpu: the K-slot unsharded ring (rsdb_ring_*,
rsdb_unit_set_shard / rsdb_unit_rebind / rsdb_all_gather_shards_p2p).

Three units share K = 2 ring slots.  Forward: each unit acquires a slot, is
rebound to it, gathers every rank's persistent shard into it (checked bit
exact against the full parameters) and releases it.  Backward (reverse
order): acquire, gather again, write the gradients into the slot, run the
fused ReduceScatter + 8-bit Adam writing the persistent shard, release.  The
shards and optimizer states must equal, bit for bit, the same step on
dedicated (non-ring) buffers.  World 1 here; N = 2/4 in the parity worker."""
import pytest
import torch

import paper_2602_22437_b200 as R
from oracle import dbuffer as OD
from oracle import planner as OP

from gpu_helpers import logical_grads, logical_params, place_gpu

pytestmark = pytest.mark.gpu

UNITS = [[2048 * 20, 300, 2048 * 3], [2048 * 7 + 5, 2048 * 2], [2048 * 33]]


def ring_case(world, rank, comm=None, p2p_factory=None, k=2):
    msgs = []
    q = 2048
    lays = [R.plan(es, [min(q, e) for e in es], world, elem_bytes=2) for es in UNITS]
    olays = [OP.plan(es, [min(q, e) for e in es], world, OP.gcoll_elems(2)) for es in UNITS]
    max_full = max(l.m * l.S for l in lays)
    dev = "cuda"
    slots = [(torch.zeros(max_full, dtype=torch.bfloat16, device=dev),
              torch.zeros(max_full, dtype=torch.bfloat16, device=dev),
              torch.zeros(max_full, dtype=torch.float32, device=dev)) for _ in range(k)]
    shard_off, acc = [], 0
    for l in lays:
        shard_off.append(acc)
        acc += (l.S + 7) // 8 * 8  # 16-B aligned shards in one arena
    shards = torch.zeros(max(acc, 8), dtype=torch.bfloat16, device=dev)
    p2p_ring = p2p_factory([t for sl in slots for t in sl[:2]] + [shards]) if p2p_factory else None
    units, refs, states, ref_states, fulls, grads = [], [], [], [], [], []
    for ui, (es, l, o) in enumerate(zip(UNITS, lays, olays)):
        E, S = sum(es), l.S
        p_log = logical_params(20 + ui, E)
        full = place_gpu(l, p_log, torch.bfloat16)
        fulls.append(full)
        grads.append(place_gpu(l, logical_grads(20 + ui, rank, E), torch.bfloat16))
        shard = shards[shard_off[ui]:shard_off[ui] + S]
        shard.copy_(full[rank * S:(rank + 1) * S])
        u = R.Unit(l, rank, *slots[0], qblock=q, comm=comm)
        u.set_shard(shard)
        units.append(u)
        nb = u.num_blocks
        master = torch.from_numpy(OD.shard(o, OD.place_logical(o, p_log.numpy()), rank).copy()).to(dev)
        st = [master, torch.zeros(S, dtype=torch.int8, device=dev), torch.zeros(S, dtype=torch.uint8, device=dev),
              torch.zeros(max(nb, 1), device=dev), torch.zeros(max(nb, 1), device=dev)]
        states.append(st)
        ref_states.append([t.clone() for t in st])
        # reference: dedicated buffers, the same fused step
        pf = full.clone()
        gf = grads[-1].clone()
        refs.append((R.Unit(l, rank, pf, gf, torch.zeros(world * S, device=dev), qblock=q, comm=comm), pf, gf))
    stream = torch.cuda.Stream()
    cfg = R.AdamConfig()
    # reference step
    for (ru, pf, gf), st in zip(refs, ref_states):
        p2p_ref = p2p_factory([pf, gf]) if p2p_factory else None
        R.reduce_scatter_adam_p2p(ru, p2p_ref, cfg, 1, state=st, stream=stream)
        stream.synchronize()
        if p2p_ref is not None:
            p2p_ref.close()
    ring = R.Ring(k)
    with torch.cuda.stream(stream):
        for ui, u in enumerate(units):  # forward: gather, use, release
            s = ring.acquire(stream)
            u.rebind(*slots[s])
            R.all_gather_shards_p2p(u, p2p_ring, stream)
            l = lays[ui]
            got = slots[s][0][:l.m * l.S].clone()
            ring.release(s, stream)
            stream.synchronize()
            if not torch.equal(got.view(torch.int16), fulls[ui].view(torch.int16)):
                msgs.append(f"unit {ui}: gathered shards differ from the full parameters")
        for ui in reversed(range(len(units))):  # backward: gather, grads, RS+Adam into the shard
            u, l = units[ui], lays[ui]
            s = ring.acquire(stream)
            u.rebind(*slots[s])
            R.all_gather_shards_p2p(u, p2p_ring, stream)
            slots[s][1][:l.m * l.S].copy_(grads[ui])
            R.reduce_scatter_adam_p2p(u, p2p_ring, cfg, 1, state=states[ui], stream=stream)
            ring.release(s, stream)
    stream.synchronize()
    for ui, l in enumerate(lays):
        S = l.S
        shard = shards[shard_off[ui]:shard_off[ui] + S]
        ref_shard = refs[ui][1][rank * S:(rank + 1) * S]
        if not torch.equal(shard.view(torch.int16), ref_shard.view(torch.int16)):
            msgs.append(f"unit {ui}: ring shard differs from the dedicated-buffer step")
        for a, b in zip(states[ui], ref_states[ui]):
            if not torch.equal(a.view(torch.uint8), b.view(torch.uint8)):
                msgs.append(f"unit {ui}: ring optimizer state differs")
                break
    ring.close()
    if p2p_ring is not None:
        torch.cuda.synchronize()
        p2p_ring.close()
    return not msgs, msgs


def test_ring_world1():
    ok, msgs = ring_case(1, 0)
    assert ok, msgs


def test_ring_single_slot_world1():
    ok, msgs = ring_case(1, 0, k=1)
    assert ok, msgs
