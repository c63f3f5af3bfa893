"""Rank contexts for the multi-rank parity cases (tests/parity_cases.py).

A parity case is a generator function ``case(ctx)`` written once, SPMD style,
for one rank: it issues that rank's calls and ``yield``s at every point where
the ranks must meet (after issuing a collective, before reading its result).
Two drivers run it:

* ``drive_proc`` -- one process per GPU (torchrun; tests/dist_parity_worker.py)
  or world 1: at each yield the device is synchronised and the processes meet
  at a torch.distributed barrier.
* ``drive_local`` -- ``world`` logical ranks in ONE process on ONE device
  (rsdb_comm_create_local / rsdb_p2p_create_local), so the driver's 1-GPU
  test box runs the N > 1 collective kernels.  Each rank's calls go to its own
  stream; the driver advances every rank to its next yield, then synchronises
  the device.  Rank code must therefore never block on the device between
  two yields (no .cpu() / torch.equal / synchronize after issuing a
  collective) and must not free library objects (cudaFree synchronises the
  device) until after a yield.
"""
from __future__ import annotations

import torch

import paper_2602_22437_b200 as R


class ProcCtx:
    """One process per rank (or world 1)."""
    local = False

    def __init__(self, rank, world, comm=None, p2p_factory=None):
        self.rank, self.world, self.comm = rank, world, comm
        self._factory = p2p_factory
        self.msgs = []
        self.p2ps = []

    @property
    def has_nccl(self):
        return self.comm is not None

    def fail(self, msg):
        self.msgs.append(msg)

    def p2p(self, bufs):
        """P2P over `bufs` (collective: every rank calls it at the same point);
        None at world 1 without a factory."""
        if False:  # noqa: SIM108 -- keeps this a generator
            yield
        if self._factory is None and self.world == 1:
            return None
        p = self._factory(bufs) if self._factory else R.P2P(self.comm, bufs)
        self.p2ps.append(p)
        return p

    def allgather(self, obj):
        """Every rank's obj, in rank order."""
        yield
        if self.world == 1:
            return [obj]
        import torch.distributed as dist
        out = [None] * self.world
        dist.all_gather_object(out, obj)
        return out


class LocalCtx:
    """Logical rank `rank` of `world` ranks sharing this process and device."""
    local = True
    has_nccl = False

    def __init__(self, rank, world, comm, comms, shared, stream):
        self.rank, self.world, self.comm = rank, world, comm
        self._comms, self._shared, self.stream = comms, shared, stream
        self._n_p2p = 0
        self._n_ag = 0
        self.msgs = []
        self.p2ps = []

    def fail(self, msg):
        self.msgs.append(msg)

    def p2p(self, bufs):
        key = ("p2p", self._n_p2p)
        self._n_p2p += 1
        self._shared.setdefault(key, {})[self.rank] = list(bufs)
        yield
        grp = self._shared.get(key + ("grp",))
        if grp is None:
            tabs = self._shared[key]
            grp = R.P2P.local_group(self._comms, [tabs[r] for r in range(self.world)])
            for p in grp:
                p.set_timeout(20.0)
            self._shared[key + ("grp",)] = grp
        self.p2ps.append(grp[self.rank])
        return grp[self.rank]

    def allgather(self, obj):
        key = ("ag", self._n_ag)
        self._n_ag += 1
        self._shared.setdefault(key, {})[self.rank] = obj
        yield
        return [self._shared[key][r] for r in range(self.world)]


def drive_proc(gen):
    """Run one rank's case in this process: sync (+ barrier) at every yield."""
    import torch.distributed as dist
    for _ in gen:
        torch.cuda.synchronize()
        if dist.is_available() and dist.is_initialized():
            dist.barrier()
    torch.cuda.synchronize()


def _sync_all(devs):
    for d in sorted(set(devs)):
        torch.cuda.synchronize(d)


def drive_local(world, case, *args, devices=None, **kw):
    """Run `case` for `world` logical ranks on the current device -- or rank r
    on devices[r] (one process driving several GPUs, peer access over
    NVLink); returns the contexts (their .msgs hold the failures).  Raises if
    the ranks' yield counts differ (an SPMD bug) or a p2p barrier timed out."""
    devs = list(devices) if devices else [torch.cuda.current_device()] * world
    comms, streams = [], []
    for r in range(world):
        with torch.cuda.device(devs[r]):
            comms.append(R.Comm.local(world, r))
            streams.append(torch.cuda.Stream())
    shared = {}
    ctxs = [LocalCtx(r, world, comms[r], comms, shared, streams[r]) for r in range(world)]
    _sync_all(devs)
    gens = []
    for r, c in enumerate(ctxs):
        with torch.cuda.device(devs[r]):
            gens.append(case(c, *args, **kw))
    alive = [True] * world
    steps = [0] * world
    while any(alive):
        for r in range(world):
            if not alive[r]:
                continue
            with torch.cuda.device(devs[r]), torch.cuda.stream(streams[r]):
                try:
                    next(gens[r])
                    steps[r] += 1
                except StopIteration:
                    alive[r] = False
        _sync_all(devs)
        if any(alive) and not all(alive):
            raise RuntimeError(f"ranks left the case at different yields: {steps}")
    for r, c in enumerate(ctxs):
        with torch.cuda.device(devs[r]):
            for p in c.p2ps:
                p.check()  # raises if one of its barriers timed out
    _sync_all(devs)
    return ctxs
