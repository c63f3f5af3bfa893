"""paper_2602_22437_b200 -- the RaggedShard/DBuffer collective step of
veScale-FSDP (arxiv 2602.22437) for B200.

Thin Python binding over librsdb.so (include/rsdb.h): argument marshalling
only; every step of the path runs in the library's C++ planner, sm_100a
kernels and NCCL calls.  PyTorch supplies device memory, streams and the
torch.distributed bootstrap -- plumbing, not the product.  There is no CPU
fallback: importing fails loudly if the library is missing.

Names follow the C ABI without the ``rsdb_`` prefix.
"""
from __future__ import annotations

import ctypes as C
import json
from typing import List, Optional, Sequence, Tuple

from . import _capi as _c
from ._capi import (RSDB_BF16, RSDB_F32, RSDB_GRAN_ELEM, RSDB_GRAN_FLAT,  # noqa: F401
                    RSDB_GRAN_ROWS, RSDB_GRAN_WHOLE, RsdbError)

lib = _c.lib
check = _c.check

__all__ = ["block_elems", "plan", "Layout", "tensor_views", "Comm", "Unit", "DBuffer", "CopyPlan", "AdamConfig",
           "all_gather", "reduce_scatter", "step_8bit_adam", "unit_cast_scale", "RsdbError",
           "init_comm"]

_GRAN = {"flat": RSDB_GRAN_FLAT, "rows": RSDB_GRAN_ROWS, "whole": RSDB_GRAN_WHOLE,
         "elem": RSDB_GRAN_ELEM}


def _ptr(t) -> Optional[int]:
    """device pointer of a torch tensor (or an int / None)."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ---------------------------------------------------------------- quantization specs
def qspecs(specs) -> "C.Array":
    """Per-tensor quantization block specs -> rsdb_qspec[]:
    ("flat", q) contiguous q-element blocks; ("tile", row_len, rows, cols)
    2-D tiles of the [numel/row_len, row_len] view (N2, P:419 32x32)."""
    arr = (_c.QSpec * max(1, len(specs)))()
    for i, sp in enumerate(specs):
        if sp[0] == "flat":
            arr[i] = _c.QSpec(0, 0, int(sp[1]))
        elif sp[0] == "tile":
            arr[i] = _c.QSpec(int(sp[1]), int(sp[2]), int(sp[3]))
        else:
            raise ValueError(f"unknown quantization spec {sp!r}")
    return arr


# ---------------------------------------------------------------- a1
def block_elems(shape: Sequence[int], gran: Tuple) -> int:
    """g_t for a granularity declaration ("flat", q) | ("rows", r) | ("whole",) | ("elem",)."""
    kind = _GRAN[gran[0]]
    param = int(gran[1]) if len(gran) > 1 else 0
    sh = _c.i64_array(shape)
    out = C.c_int64()
    check(lib.rsdb_block_elems(len(shape), sh, kind, param, C.byref(out)))
    return out.value


# ---------------------------------------------------------------- a2/a3
class Layout:
    """Planned FSDP unit layout (library-owned rsdb_layout*)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and lib is not None:  # lib is None at interpreter exit
            lib.rsdb_layout_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def S(self) -> int:
        return lib.rsdb_layout_shard_numel(self._h)

    @property
    def padding(self) -> int:
        return lib.rsdb_layout_padding(self._h)

    @property
    def E(self) -> int:
        return lib.rsdb_layout_total_numel(self._h)

    @property
    def m(self) -> int:
        return lib.rsdb_layout_world(self._h)

    @property
    def n(self) -> int:
        return lib.rsdb_layout_ntensors(self._h)

    @property
    def elem_bytes(self) -> int:
        return lib.rsdb_layout_elem_bytes(self._h)

    @property
    def starts(self) -> List[int]:
        arr = (C.c_int64 * max(1, self.n))()
        check(lib.rsdb_layout_starts(self._h, arr))
        return list(arr[: self.n])

    def validate(self) -> int:
        v = C.c_int64()
        check(lib.rsdb_layout_validate(self._h, C.byref(v)))
        return v.value

    def padding_intervals(self) -> List[Tuple[int, int]]:
        n = C.c_int64(0)
        check(lib.rsdb_layout_padding_intervals(self._h, C.byref(n), None, None))
        lo, hi = (C.c_int64 * max(1, n.value))(), (C.c_int64 * max(1, n.value))()
        check(lib.rsdb_layout_padding_intervals(self._h, C.byref(n), lo, hi))
        return [(lo[i], hi[i]) for i in range(n.value)]

    def rank_segments(self, rank: int) -> List[Tuple[int, int, int, int]]:
        n = C.c_int64(0)
        check(lib.rsdb_layout_rank_segments(self._h, rank, C.byref(n), None, None, None, None))
        k = max(1, n.value)
        t, lo, ln, to = (C.c_int32 * k)(), (C.c_int64 * k)(), (C.c_int64 * k)(), (C.c_int64 * k)()
        check(lib.rsdb_layout_rank_segments(self._h, rank, C.byref(n), t, lo, ln, to))
        return [(t[i], lo[i], ln[i], to[i]) for i in range(n.value)]

    def rank_blocks(self, rank: int, qblock: int) -> List[Tuple[int, int]]:
        n = C.c_int64(0)
        check(lib.rsdb_layout_rank_blocks(self._h, rank, qblock, C.byref(n), None, None))
        k = max(1, n.value)
        off, ln = (C.c_int64 * k)(), (C.c_int32 * k)()
        check(lib.rsdb_layout_rank_blocks(self._h, rank, qblock, C.byref(n), off, ln))
        return [(off[i], ln[i]) for i in range(n.value)]

    def rank_tiles(self, rank: int, specs) -> List[Tuple[int, int, int, int]]:
        """(offset of first element, rows, cols, pitch) of rank's blocks (N2)."""
        sp = qspecs(specs)
        n = C.c_int64(0)
        check(lib.rsdb_layout_rank_tiles(self._h, rank, sp, C.byref(n), None, None, None, None))
        k = max(1, n.value)
        off, rw, cl, pt = (C.c_int64 * k)(), (C.c_int32 * k)(), (C.c_int32 * k)(), (C.c_int64 * k)()
        check(lib.rsdb_layout_rank_tiles(self._h, rank, sp, C.byref(n), off, rw, cl, pt))
        return [(off[i], rw[i], cl[i], pt[i]) for i in range(n.value)]

    def to_json(self) -> dict:
        need = C.c_int64(0)
        check(lib.rsdb_layout_to_json(self._h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        check(lib.rsdb_layout_to_json(self._h, buf, need.value, C.byref(need)))
        return json.loads(buf.value.decode())


def plan(numel: Sequence[int], block: Sequence[int], world: int, elem_bytes: int = 2,
         gcoll_bytes: int = 16) -> Layout:
    """plan(tensors, block_sizes, world) -> layout (Algorithm 1)."""
    h = C.c_void_p()
    check(lib.rsdb_plan(len(numel), _c.i64_array(numel), _c.i64_array(block), world,
                        elem_bytes, gcoll_bytes, C.byref(h)))
    return Layout(h.value)


ORDER = {"default": 0, "block": 1, "shape": 2, "best": 3}


def plan_ordered(numel: Sequence[int], block: Sequence[int], world: int, ordering="default",
                 shape_keys: Optional[Sequence[int]] = None, elem_bytes: int = 2,
                 gcoll_bytes: int = 16) -> Layout:
    """Algorithm 1 on one of the tensor orders of P:279 (N4)."""
    h = C.c_void_p()
    keys = _c.i64_array(shape_keys) if shape_keys is not None else None
    check(lib.rsdb_plan_ordered(len(numel), _c.i64_array(numel), _c.i64_array(block), world,
                                elem_bytes, gcoll_bytes, ORDER[ordering], keys, C.byref(h)))
    return Layout(h.value)


def layout_from_starts(numel, block, world, S, starts, elem_bytes=2, gcoll_bytes=16,
                       require_gcoll=True) -> Layout:
    h = C.c_void_p()
    check(lib.rsdb_layout_from_starts(len(numel), _c.i64_array(numel), _c.i64_array(block),
                                      world, elem_bytes, gcoll_bytes, S, _c.i64_array(starts),
                                      int(require_gcoll), C.byref(h)))
    return Layout(h.value)


# ---------------------------------------------------------------- comm
def tensor_views(layout: Layout, full, shapes: Sequence[Sequence[int]]) -> list:
    """a5 ("zero-copy access before and after communication"): the
    tensors of a unit as views of its m*S buffer (PARAM_FULL, GRAD_FULL or
    GRAD_F32 of any dtype): tensor t = full[l_t : l_t + e_t] reshaped to
    shapes[t].  No bytes move; writes through a view land in the buffer the
    collectives read.  Padding is never covered by a view."""
    numel = layout.to_json()["numel"]
    if len(shapes) != len(numel):
        raise ValueError(f"{len(shapes)} shapes for a unit of {len(numel)} tensors")
    if full.dim() != 1 or full.numel() != layout.m * layout.S:
        raise ValueError(f"buffer must be flat with m*S = {layout.m * layout.S} elements")
    out = []
    for t, (l, e, shp) in enumerate(zip(layout.starts, numel, shapes)):
        n = 1
        for d in shp:
            n *= int(d)
        if n != e:
            raise ValueError(f"tensor {t}: shape {tuple(shp)} has {n} elements, the layout {e}")
        out.append(full[l:l + e].view(*[int(d) for d in shp]))
    return out


class Comm:
    def __init__(self, uid: bytes, world: int, rank: int, device: int):
        h = C.c_void_p()
        check(lib.rsdb_comm_init(uid, world, rank, device, C.byref(h)))
        self._h = h

    @classmethod
    def local(cls, world: int, rank: int) -> "Comm":
        """Logical rank `rank` of `world` ranks living in this process on the
        current device (rsdb_comm_create_local; no NCCL)."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        check(lib.rsdb_comm_create_local(world, rank, C.byref(h)))
        self._h = h
        return self

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib.rsdb_unique_id(buf))
        return buf.raw

    @property
    def handle(self):
        return self._h

    @property
    def rank(self) -> int:
        return lib.rsdb_comm_rank(self._h)

    @property
    def world(self) -> int:
        return lib.rsdb_comm_world(self._h)

    def close(self):
        if self._h is not None and self._h.value:
            lib.rsdb_comm_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def init_comm(rank: int, world: int, device: int, group=None) -> Comm:
    """Bootstrap: rank 0 makes the NCCL unique id, torch.distributed
    broadcasts its 128 bytes (plumbing), every rank joins."""
    import torch.distributed as dist
    obj = [Comm.unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0, group=group)
    return Comm(obj[0], world, rank, device)


# ---------------------------------------------------------------- unit
class Unit:
    """One FSDP unit bound to caller-owned device buffers (torch tensors)."""

    def __init__(self, layout: Layout, rank: int, param_full, grad_full, grad_f32,
                 qblock: int = 2048, comm: Optional[Comm] = None, _handle=None, _keep=None,
                 qspec=None):
        self.layout = layout
        self.rank = rank
        self.comm = comm
        self._keep = _keep if _keep is not None else (param_full, grad_full, grad_f32)
        self._owned = _handle is None
        if _handle is None:
            bufs = _c.UnitBufs(_ptr(param_full), _ptr(grad_full), _ptr(grad_f32))
            h = C.c_void_p()
            if qspec is None:
                check(lib.rsdb_unit_create(layout.handle, comm.handle if comm else None, rank,
                                           C.byref(bufs), qblock, C.byref(h)))
            else:
                check(lib.rsdb_unit_create_q(layout.handle, comm.handle if comm else None, rank,
                                             C.byref(bufs), qspecs(qspec), C.byref(h)))
            self._h = h
        else:
            self._h = C.c_void_p(_handle)

    @property
    def handle(self):
        return self._h

    @property
    def num_blocks(self) -> int:
        return lib.rsdb_unit_num_blocks(self._h)

    def set_shard(self, shard) -> None:
        """K-slot ring mode: the persistent parameter shard (S elements) the
        optimizer writes; None turns ring mode off."""
        self._shard = shard
        check(lib.rsdb_unit_set_shard(self._h, _ptr(shard) if shard is not None else None))

    def rebind(self, param_full, grad_full, grad_f32) -> None:
        """Point the unit at other gathered buffers (e.g. a ring slot)."""
        self._keep = (param_full, grad_full, grad_f32)
        bufs = _c.UnitBufs(_ptr(param_full), _ptr(grad_full), _ptr(grad_f32))
        check(lib.rsdb_unit_rebind(self._h, C.byref(bufs)))

    def close(self):
        if self._owned and self._h is not None and self._h.value:
            lib.rsdb_unit_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class AdamConfig(_c.AdamCfg):
    def __init__(self, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=1e-2):
        super().__init__(lr, beta1, beta2, eps, weight_decay)


def all_gather(unit: Unit, stream=None) -> None:
    """a4: in-place AllGather of the unit buffer (ncclAllGather)."""
    check(lib.rsdb_all_gather(unit.handle, _stream(stream)))


def unit_cast_scale(unit: Unit, stream=None) -> None:
    """a6: the fused group op alone (cast bf16->fp32, x1/m, padding 0)."""
    check(lib.rsdb_unit_cast_scale(unit.handle, _stream(stream)))


def reduce_scatter(unit: Unit, stream=None) -> None:
    """a6 + a7: fused cast/scale, then in-place fp32 ReduceScatter."""
    check(lib.rsdb_reduce_scatter(unit.handle, _stream(stream)))


def unit_reduce_scatter_f32(unit: Unit, stream=None) -> None:
    """a7 alone: in-place fp32 ReduceScatter of grad_f32 as it stands."""
    check(lib.rsdb_unit_reduce_scatter_f32(unit.handle, _stream(stream)))


def step_8bit_adam(unit: Unit, master, m_q, v_q, m_absmax, v_absmax, cfg: AdamConfig,
                   step: int, stream=None) -> None:
    """a8: block-wise 8-bit Adam on the unit's local ragged shard."""
    st = _c.AdamState(_ptr(master), _ptr(m_q), _ptr(v_q), _ptr(m_absmax), _ptr(v_absmax))
    check(lib.rsdb_step_8bit_adam(unit.handle, C.byref(st), C.byref(cfg), step, _stream(stream)))


def step_8bit_adam_dynamic(unit: Unit, master, m_q, v_q, m_absmax, v_absmax, cfg: AdamConfig,
                           step: int, stream=None) -> None:
    """a8 with the dynamic (tree) code map (N2, R25): m_q / v_q are uint8 map indices."""
    st = _c.AdamState(_ptr(master), _ptr(m_q), _ptr(v_q), _ptr(m_absmax), _ptr(v_absmax))
    check(lib.rsdb_step_8bit_adam_dynamic(unit.handle, C.byref(st), C.byref(cfg), step,
                                          _stream(stream)))


def dynamic_code_maps():
    """The two 256-value maps (signed for m, unsigned for v) of the dynamic codec."""
    m = (C.c_float * 256)()
    v = (C.c_float * 256)()
    check(lib.rsdb_dynamic_code_maps(m, v))
    return list(m), list(v)


def dynamic_code_tables():
    """The code tables the dynamic codec's kernels decide with
    (rsdb_dynamic_code_tables: layout in include/rsdb.h), as two lists of uint32."""
    m = (C.c_uint32 * _c.RSDB_DYN_TABLE_M_LEN)()
    v = (C.c_uint32 * _c.RSDB_DYN_TABLE_V_LEN)()
    check(lib.rsdb_dynamic_code_tables(m, v))
    return list(m), list(v)


# ---------------------------------------------------------------- N1: NVLink peer memory
def ipc_handle(t) -> bytes:
    buf = C.create_string_buffer(_c.RSDB_IPC_BYTES)
    check(lib.rsdb_ipc_handle(_ptr(t), buf))
    return buf.raw


class P2P:
    """Every rank's `bufs` (torch tensors, e.g. the GRAD_FULL and PARAM_FULL
    arenas) mapped into this process over NVLink (CUDA IPC), plus a signal
    buffer, for the fused p2p collectives.  The IPC handles are exchanged with
    torch.distributed.all_gather_object (plumbing).  Keeps the tensors alive."""

    def __init__(self, comm: Comm, bufs: Sequence, group=None):
        import torch
        import torch.distributed as dist
        dev = bufs[0].device
        self.signal = torch.zeros(_c.RSDB_P2P_SIGNAL_BYTES, dtype=torch.uint8, device=dev)
        self.bufs = [self.signal] + list(bufs)
        mine = b"".join(ipc_handle(t) for t in self.bufs)
        allh = [None] * comm.world
        if comm.world > 1:
            dist.all_gather_object(allh, mine, group=group)
        else:
            allh = [mine]
        n = len(self.bufs)
        ptrs = (C.c_void_p * n)(*[t.data_ptr() for t in self.bufs])
        sizes = (C.c_int64 * n)(*[t.numel() * t.element_size() for t in self.bufs])
        h = C.c_void_p()
        check(lib.rsdb_p2p_create(comm.handle, n, ptrs, sizes, b"".join(allh), C.byref(h)))
        self._h = h
        self.comm = comm

    @classmethod
    def local_group(cls, comms: Sequence[Comm], bufs_per_rank: Sequence[Sequence]) -> List["P2P"]:
        """Local mode: one P2P per logical rank (comms from Comm.local) over
        every rank's buffers, all on the current device
        (rsdb_p2p_create_local).  bufs_per_rank[r] = rank r's tensors."""
        import torch
        world = len(comms)
        tables = []
        for bufs in bufs_per_rank:
            sig = torch.zeros(_c.RSDB_P2P_SIGNAL_BYTES, dtype=torch.uint8, device=bufs[0].device)
            tables.append([sig] + list(bufs))
        n = len(tables[0])
        ptrs = (C.c_void_p * (world * n))(*[t.data_ptr() for tb in tables for t in tb])
        sizes = (C.c_int64 * n)(*[t.numel() * t.element_size() for t in tables[0]])
        out = []
        for r in range(world):
            self = cls.__new__(cls)
            h = C.c_void_p()
            check(lib.rsdb_p2p_create_local(comms[r].handle, n, ptrs, sizes, C.byref(h)))
            self._h = h
            self.comm = comms[r]
            self.signal = tables[r][0]
            self.bufs = tables  # keeps every rank's tensors alive
            out.append(self)
        return out

    def channel(self, c: int) -> "P2P":
        """rsdb_p2p_channel: an independent collective channel (own epoch and
        signal words) over the same mappings, for collectives that overlap on
        different streams.  Close it before this object."""
        h = C.c_void_p()
        check(lib.rsdb_p2p_channel(self._h, int(c), C.byref(h)))
        ch = P2P.__new__(P2P)
        ch._h = h
        ch.comm = self.comm
        ch.signal = self.signal
        ch.bufs = self.bufs
        ch.parent = self
        return ch

    def barrier(self, stream=None) -> None:
        """rsdb_p2p_barrier: device-side barrier of every rank on `stream`."""
        check(lib.rsdb_p2p_barrier(self._h, _stream(stream)))

    def set_max_ctas(self, n: int) -> None:
        """rsdb_p2p_set_max_ctas: CTA budget of this object's kernels (0 = all SMs)."""
        check(lib.rsdb_p2p_set_max_ctas(self._h, int(n)))

    def set_timeout(self, seconds: float) -> None:
        check(lib.rsdb_p2p_set_timeout(self._h, float(seconds)))

    def check(self) -> int:
        """Synchronise; raise if a barrier of this rank timed out."""
        f = C.c_int64(0)
        check(lib.rsdb_p2p_check(self._h, C.byref(f)))
        return f.value

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.rsdb_p2p_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def reduce_scatter_p2p(unit: Unit, p2p: Optional[P2P], stream=None) -> None:
    """a6 + a7 fused in one kernel over NVLink peer memory (bf16 on the wire)."""
    check(lib.rsdb_reduce_scatter_p2p(unit.handle, p2p.handle if p2p is not None else None,
                                      _stream(stream)))


def reduce_scatter_adam_p2p(unit: Unit, p2p: Optional[P2P], cfg: AdamConfig, step: int,
                            state=None, stream=None) -> None:
    """a6 + a7 + a8 in one kernel: ReduceScatter over NVLink feeding the 8-bit
    Adam update of this rank's shard.  state = (master, m_q, v_q, m_absmax,
    v_absmax) tensors, or None for a unit of a DBuffer.  p2p may be None at
    world 1."""
    st = None
    if state is not None:
        st = C.byref(_c.AdamState(*[_ptr(t) for t in state]))
    check(lib.rsdb_reduce_scatter_adam_p2p(unit.handle, p2p.handle if p2p is not None else None,
                                           st, C.byref(cfg), step, _stream(stream)))


def reduce_scatter_adam_gather_p2p(unit: Unit, p2p: Optional[P2P], cfg: AdamConfig, step: int,
                                   state=None, stream=None) -> None:
    """reduce_scatter_adam_p2p with the next AllGather fused in: the updated
    bf16 shard is also stored into every peer's param_full (p2p must map it)."""
    st = None
    if state is not None:
        st = C.byref(_c.AdamState(*[_ptr(t) for t in state]))
    check(lib.rsdb_reduce_scatter_adam_gather_p2p(unit.handle,
                                                  p2p.handle if p2p is not None else None,
                                                  st, C.byref(cfg), step, _stream(stream)))


def all_gather_p2p(unit: Unit, p2p: Optional[P2P], stream=None) -> None:
    """a4 as one kernel pulling every peer's shard over NVLink."""
    check(lib.rsdb_all_gather_p2p(unit.handle, p2p.handle if p2p is not None else None, _stream(stream)))


# ---------------------------------------------------------------- DBuffer
KINDS = ("param_full", "grad_full", "grad_f32", "master", "m_q", "v_q", "m_absmax", "v_absmax")


def _spec_ptrs(qspec_per_unit):
    keep = [qspecs(sp) for sp in qspec_per_unit]
    ptrs = (C.POINTER(_c.QSpec) * max(1, len(keep)))(
        *[C.cast(a, C.POINTER(_c.QSpec)) for a in keep])
    return ptrs, keep


def arena_sizes(layouts: Sequence[Layout], rank: int, qblock: int = 2048, align: int = 256,
                qspec=None):
    """qspec: None (flat qblock) or one per-tensor spec list per unit (N2)."""
    arr = (C.c_void_p * max(1, len(layouts)))(*[l.handle.value for l in layouts])
    sizes = (C.c_int64 * _c.RSDB_NKINDS)()
    offs = (C.c_int64 * max(1, len(layouts) * _c.RSDB_NKINDS))()
    if qspec is None:
        check(lib.rsdb_arena_sizes(arr, len(layouts), rank, qblock, align, sizes, offs))
    else:
        ptrs, _keep = _spec_ptrs(qspec)
        check(lib.rsdb_arena_sizes_q(arr, len(layouts), rank, ptrs, align, sizes, offs))
    K = _c.RSDB_NKINDS
    return list(sizes), [list(offs[u * K:(u + 1) * K]) for u in range(len(layouts))]


class DBuffer:
    """Batched DBuffer: one caller-allocated arena per
    buffer kind holding every unit; per-unit zero-copy views; one optimizer
    launch over all units."""

    def __init__(self, layouts: Sequence[Layout], rank: int, arenas: Sequence, qblock=2048,
                 align=256, comm: Optional[Comm] = None, qspec=None):
        self.layouts = list(layouts)
        self.rank = rank
        self.comm = comm
        self.arenas = list(arenas)
        arr = (C.c_void_p * max(1, len(layouts)))(*[l.handle.value for l in layouts])
        bases = (C.c_void_p * _c.RSDB_NKINDS)(*[_ptr(a) if a is not None and a.numel() > 0
                                                else None for a in arenas])
        h = C.c_void_p()
        if qspec is None:
            check(lib.rsdb_dbuffer_create(arr, len(layouts), comm.handle if comm else None, rank,
                                          qblock, align, bases, C.byref(h)))
        else:
            ptrs, _keep = _spec_ptrs(qspec)
            check(lib.rsdb_dbuffer_create_q(arr, len(layouts), comm.handle if comm else None, rank,
                                            ptrs, align, bases, C.byref(h)))
        self._h = h
        self.units = [Unit(l, rank, None, None, None, comm=comm,
                           _handle=lib.rsdb_dbuffer_unit(h, i), _keep=())
                      for i, l in enumerate(layouts)]

    @property
    def handle(self):
        return self._h

    @property
    def num_blocks(self) -> int:
        return lib.rsdb_dbuffer_num_blocks(self._h)

    def step_8bit_adam(self, cfg: AdamConfig, step: int, stream=None) -> None:
        check(lib.rsdb_dbuffer_step_8bit_adam(self._h, C.byref(cfg), step, _stream(stream)))

    def reduce_scatter_adam(self, cfg: AdamConfig, step: int, p2p: Optional["P2P"] = None,
                            stream=None) -> None:
        """a6 + a7 + a8 for every unit in one launch (p2p None iff world 1)."""
        check(lib.rsdb_dbuffer_reduce_scatter_adam(self._h, p2p.handle if p2p is not None else None,
                                                   C.byref(cfg), step, _stream(stream)))

    def reduce_scatter_adam_gather(self, cfg: AdamConfig, step: int, p2p: Optional["P2P"] = None,
                                   stream=None) -> None:
        """a6 + a7 + a8 + a4 for every unit in one launch: on return every rank
        holds the full updated parameters (p2p maps GRAD_FULL and PARAM_FULL)."""
        check(lib.rsdb_dbuffer_reduce_scatter_adam_gather(
            self._h, p2p.handle if p2p is not None else None, C.byref(cfg), step, _stream(stream)))

    def step_8bit_adam_dynamic(self, cfg: AdamConfig, step: int, stream=None) -> None:
        """One launch of 8-bit Adam with the dynamic code map over every unit."""
        check(lib.rsdb_dbuffer_step_8bit_adam_dynamic(self._h, C.byref(cfg), step, _stream(stream)))

    def step_host(self, cfg: AdamConfig, step: int, host_grads, host_shards,
                  p2p: Optional["P2P"] = None, stream=None) -> None:
        """rsdb_dbuffer_step_host: per unit (backward order) H2D of host_grads[u]
        (pinned host tensor, m*S bf16), the fused RS + 8-bit Adam (+ AllGather
        push) kernel, D2H of the rank's updated bf16 shard into host_shards[u]."""
        n = len(self.units)
        if len(host_grads) != n or len(host_shards) != n:
            raise ValueError("one host gradient and one host shard buffer per unit")
        g = (C.c_void_p * n)(*[_ptr(t) for t in host_grads])
        s = (C.c_void_p * n)(*[_ptr(t) for t in host_shards])
        check(lib.rsdb_dbuffer_step_host(self._h, p2p.handle if p2p is not None else None,
                                         C.byref(cfg), step, g, s, _stream(stream)))

    def zero_grads(self, stream=None) -> None:
        check(lib.rsdb_dbuffer_zero_grads(self._h, _stream(stream)))

    def close(self):
        for u in getattr(self, "units", []):
            u._h = None
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.rsdb_dbuffer_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- copies
class CopyPlan:
    """Persistent batched ragged copy (FSDP2 Copy-In / Copy-Out baseline)."""

    def __init__(self, segments: Sequence[Tuple[object, object, int]], src_dtype=RSDB_BF16,
                 dst_dtype=RSDB_BF16, scale: float = 1.0):
        arr = (_c.Segment * max(1, len(segments)))(
            *[_c.Segment(_ptr(s), _ptr(d), int(n)) for s, d, n in segments])
        h = C.c_void_p()
        check(lib.rsdb_copy_plan_create(arr, len(segments), src_dtype, dst_dtype, scale,
                                        C.byref(h)))
        self._h = h

    def run(self, stream=None) -> None:
        check(lib.rsdb_copy_run(self._h, _stream(stream)))

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.rsdb_copy_plan_free(self._h)
            self._h = None


# ---------------------------------------------------------------- N2: FP8 AllGather
class Fp8Unit:
    """FP8 (E4M3) 128x128 block quantization of a unit's fp32 master shard
    fused with the AllGather of the codes (1 B/element) and per-tile scales
    (rsdb_fp8_*, R18-R20).  `layout` is planned with elem_bytes=1
    at 128-row granularity; `specs` = [("tile", row_len, 128, 128), ...]."""

    def __init__(self, layout: Layout, specs, rank: int, master_shard, codes_full, scales_full,
                 comm: Optional[Comm] = None):
        self._keep = (layout, master_shard, codes_full, scales_full)
        self._specs = qspecs(specs)
        h = C.c_void_p()
        check(lib.rsdb_fp8_unit_create(layout.handle, self._specs, comm.handle if comm else None,
                                       rank, _ptr(master_shard), _ptr(codes_full),
                                       _ptr(scales_full), C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    @property
    def num_tiles(self) -> int:
        return lib.rsdb_fp8_unit_num_tiles(self._h)

    @property
    def first_slot(self) -> int:
        return lib.rsdb_fp8_unit_first_slot(self._h)

    def quantize_all_gather(self, p2p: Optional["P2P"] = None, stream=None) -> None:
        check(lib.rsdb_fp8_quantize_all_gather(self._h, p2p.handle if p2p is not None else None,
                                               _stream(stream)))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.rsdb_fp8_unit_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- N3: distributed Muon
class MuonConfig(_c.MuonCfg):
    """R21-R23 defaults: eta 0.02, Nesterov momentum 0.95, NS eps 1e-7, 5 steps."""

    def __init__(self, lr=0.02, momentum=0.95, eps=1e-7, ns_steps=5):
        super().__init__(lr, momentum, eps, ns_steps)


def muon_select_roots(layout: Layout, shapes) -> List[int]:
    """SelectRoot (R24) on the host: the root rank of every matrix (-1: skipped)."""
    rows = _c.i64_array([s[0] if s else 0 for s in shapes])
    cols = _c.i64_array([s[1] if s else 0 for s in shapes])
    out = (C.c_int32 * max(1, len(shapes)))()
    check(lib.rsdb_muon_select_roots(layout.handle, rows, cols, out))
    return list(out[:len(shapes)])


class Muon:
    """Distributed Muon over a RaggedShard unit (Algorithm 2; rsdb_muon_*).
    shapes[t] = (rows, cols) for the matrices Muon updates, None otherwise.
    precision "f32" (SGEMM Newton-Schulz) or "bf16" (tensor cores)."""

    def __init__(self, layout: Layout, shapes, rank: int, comm: Optional[Comm] = None,
                 precision: str = "f32"):
        rows = _c.i64_array([s[0] if s else 0 for s in shapes])
        cols = _c.i64_array([s[1] if s else 0 for s in shapes])
        prec = {"f32": RSDB_F32, "bf16": RSDB_BF16}[precision]
        h = C.c_void_p()
        check(lib.rsdb_muon_create(layout.handle, rows, cols, comm.handle if comm else None, rank, prec,
                                   C.byref(h)))
        self._h = h
        self._keep = (layout,)
        self.n = len(shapes)

    @property
    def workspace_bytes(self) -> int:
        return lib.rsdb_muon_workspace_bytes(self._h)

    def root(self, t: int) -> int:
        return lib.rsdb_muon_root(self._h, t)

    def bind(self, master, momentum, grad, u, workspace, param_bf16=None) -> None:
        self._bufs = (master, momentum, grad, u, workspace, param_bf16)
        b = _c.MuonBufs(_ptr(master), _ptr(momentum), _ptr(grad), _ptr(u), _ptr(param_bf16),
                        _ptr(workspace))
        check(lib.rsdb_muon_bind(self._h, C.byref(b)))

    def step(self, cfg: Optional[MuonConfig] = None, p2p: Optional["P2P"] = None, stream=None) -> None:
        cfg = cfg or MuonConfig()
        check(lib.rsdb_muon_step(self._h, p2p.handle if p2p is not None else None, C.byref(cfg),
                                 _stream(stream)))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.rsdb_muon_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- K-slot unsharded ring
def ns_gemm_bf16(A, B, C, alpha=1.0, beta=0.0, D=None, CT=None, stream=None) -> None:
    """rsdb_ns_gemm_bf16: C = alpha A B^T + beta D (and CT = C^T), bf16 2-D
    torch tensors, row-major with unit column stride (the tcgen05 Newton-Schulz
    GEMM of Muon's bf16 mode)."""
    M, K = A.shape
    N = B.shape[0]
    check(lib.rsdb_ns_gemm_bf16(M, N, K, _ptr(A), A.stride(0), _ptr(B), B.stride(0), float(alpha),
                                float(beta), _ptr(D), D.stride(0) if D is not None else 0, _ptr(C),
                                C.stride(0), _ptr(CT), CT.stride(0) if CT is not None else 0,
                                _stream(stream)))


def ns_gemm_bf16_sym(A, B, C, alpha=1.0, beta=0.0, D=None, stream=None) -> None:
    """rsdb_ns_gemm_bf16_sym: C = alpha A B^T + beta D for a product known to
    be symmetric (M x M): upper-triangle tiles computed, lower mirrored."""
    M, K = A.shape
    check(lib.rsdb_ns_gemm_bf16_sym(M, K, _ptr(A), A.stride(0), _ptr(B), B.stride(0), float(alpha), float(beta),
                                    _ptr(D), D.stride(0) if D is not None else 0, _ptr(C), C.stride(0),
                                    _stream(stream)))


def all_gather_shards_p2p(unit: Unit, p2p: Optional["P2P"] = None, stream=None) -> None:
    """AllGather of every rank's persistent shard into the unit's param_full."""
    check(lib.rsdb_all_gather_shards_p2p(unit.handle, p2p.handle if p2p is not None else None,
                                         _stream(stream)))


class Ring:
    """K slots handed out round robin (same slot sequence on every rank); the
    stream waits for the slot's previous release."""

    def __init__(self, k: int):
        h = C.c_void_p()
        check(lib.rsdb_ring_create(k, C.byref(h)))
        self._h = h
        self.k = k

    def acquire(self, stream=None) -> int:
        out = C.c_int32()
        check(lib.rsdb_ring_acquire(self._h, _stream(stream), C.byref(out)))
        return out.value

    def release(self, slot: int, stream=None) -> None:
        check(lib.rsdb_ring_release(self._h, slot, _stream(stream)))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.rsdb_ring_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
