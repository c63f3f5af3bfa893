"""ctypes declarations of include/rsdb.h (argument marshalling only).

Every function here is the C symbol of the same name; no arithmetic of the
method is done in Python.  Loading fails loudly if librsdb.so is missing:
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librsdb.so")

RSDB_OK, RSDB_EINVAL, RSDB_EMISMATCH, RSDB_ECUDA, RSDB_ENCCL, RSDB_EINTERNAL = range(6)
RSDB_BF16, RSDB_F32 = 0, 1
RSDB_GRAN_FLAT, RSDB_GRAN_ROWS, RSDB_GRAN_WHOLE, RSDB_GRAN_ELEM = range(4)
(RSDB_KIND_PARAM_FULL, RSDB_KIND_GRAD_FULL, RSDB_KIND_GRAD_F32, RSDB_KIND_MASTER,
 RSDB_KIND_MQ, RSDB_KIND_VQ, RSDB_KIND_MABS, RSDB_KIND_VABS) = range(8)
RSDB_NKINDS = 8
RSDB_IPC_BYTES = 72
RSDB_P2P_SIGNAL_BYTES = 4096
RSDB_DYN_TABLE_M_LEN = RSDB_DYN_TABLE_V_LEN = 3584

i32, i64, vp = C.c_int32, C.c_int64, C.c_void_p
P_i64, P_i32 = C.POINTER(C.c_int64), C.POINTER(C.c_int32)


class UnitBufs(C.Structure):
    _fields_ = [("param_full", vp), ("grad_full", vp), ("grad_f32", vp)]


class AdamCfg(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("weight_decay", C.c_double)]


class AdamState(C.Structure):
    _fields_ = [("master_f32", vp), ("m_q", vp), ("v_q", vp), ("m_absmax", vp), ("v_absmax", vp)]


class QSpec(C.Structure):
    _fields_ = [("row_len", i64), ("tile_rows", i32), ("tile_cols", i32)]


class Segment(C.Structure):
    _fields_ = [("src", vp), ("dst", vp), ("numel", i64)]


class MuonCfg(C.Structure):
    _fields_ = [("lr", C.c_double), ("momentum", C.c_double), ("eps", C.c_double),
                ("ns_steps", i32)]


class MuonBufs(C.Structure):
    _fields_ = [("master", vp), ("momentum", vp), ("grad", vp), ("u", vp), ("param_bf16", vp),
                ("workspace", vp)]


# name: (restype, argtypes)
_SIGS = {
    "rsdb_last_error": (C.c_char_p, []),
    "rsdb_abi_version": (i32, []),
    "rsdb_block_elems": (i32, [i32, P_i64, i32, i64, P_i64]),
    "rsdb_plan": (i32, [i32, P_i64, P_i64, i32, i32, i32, C.POINTER(vp)]),
    "rsdb_plan_ordered": (i32, [i32, P_i64, P_i64, i32, i32, i32, i32, P_i64, C.POINTER(vp)]),
    "rsdb_layout_from_starts": (i32, [i32, P_i64, P_i64, i32, i32, i32, i64, P_i64, i32,
                                      C.POINTER(vp)]),
    "rsdb_layout_shard_numel": (i64, [vp]),
    "rsdb_layout_padding": (i64, [vp]),
    "rsdb_layout_total_numel": (i64, [vp]),
    "rsdb_layout_world": (i32, [vp]),
    "rsdb_layout_ntensors": (i32, [vp]),
    "rsdb_layout_elem_bytes": (i32, [vp]),
    "rsdb_layout_starts": (i32, [vp, P_i64]),
    "rsdb_layout_validate": (i32, [vp, P_i64]),
    "rsdb_layout_padding_intervals": (i32, [vp, P_i64, P_i64, P_i64]),
    "rsdb_layout_rank_segments": (i32, [vp, i32, P_i64, P_i32, P_i64, P_i64, P_i64]),
    "rsdb_layout_rank_blocks": (i32, [vp, i32, i64, P_i64, P_i64, P_i32]),
    "rsdb_layout_to_json": (i32, [vp, C.c_char_p, i64, P_i64]),
    "rsdb_layout_rank_tiles": (i32, [vp, i32, C.POINTER(QSpec), P_i64, P_i64, P_i32, P_i32, P_i64]),
    "rsdb_unit_create_q": (i32, [vp, vp, i32, C.POINTER(UnitBufs), C.POINTER(QSpec), C.POINTER(vp)]),
    "rsdb_arena_sizes_q": (i32, [C.POINTER(vp), i32, i32, C.POINTER(C.POINTER(QSpec)), i64, P_i64,
                                 P_i64]),
    "rsdb_dbuffer_create_q": (i32, [C.POINTER(vp), i32, vp, i32, C.POINTER(C.POINTER(QSpec)), i64,
                                    C.POINTER(vp), C.POINTER(vp)]),
    "rsdb_layout_free": (None, [vp]),
    "rsdb_unique_id": (i32, [C.c_char_p]),
    "rsdb_comm_init": (i32, [C.c_char_p, i32, i32, i32, C.POINTER(vp)]),
    "rsdb_comm_rank": (i32, [vp]),
    "rsdb_comm_world": (i32, [vp]),
    "rsdb_comm_free": (None, [vp]),
    "rsdb_comm_create_local": (i32, [i32, i32, C.POINTER(vp)]),
    "rsdb_unit_create": (i32, [vp, vp, i32, C.POINTER(UnitBufs), i64, C.POINTER(vp)]),
    "rsdb_unit_num_blocks": (i64, [vp]),
    "rsdb_unit_free": (None, [vp]),
    "rsdb_all_gather": (i32, [vp, vp]),
    "rsdb_unit_cast_scale": (i32, [vp, vp]),
    "rsdb_reduce_scatter": (i32, [vp, vp]),
    "rsdb_unit_reduce_scatter_f32": (i32, [vp, vp]),
    "rsdb_step_8bit_adam": (i32, [vp, C.POINTER(AdamState), C.POINTER(AdamCfg), i64, vp]),
    "rsdb_ipc_handle": (i32, [vp, C.c_char_p]),
    "rsdb_p2p_create": (i32, [vp, i32, C.POINTER(vp), P_i64, C.c_char_p, C.POINTER(vp)]),
    "rsdb_p2p_free": (None, [vp]),
    "rsdb_p2p_channel": (i32, [vp, i32, C.POINTER(vp)]),
    "rsdb_p2p_set_max_ctas": (i32, [vp, i32]),
    "rsdb_p2p_barrier": (i32, [vp, vp]),
    "rsdb_p2p_create_local": (i32, [vp, i32, C.POINTER(vp), P_i64, C.POINTER(vp)]),
    "rsdb_p2p_set_timeout": (i32, [vp, C.c_double]),
    "rsdb_p2p_check": (i32, [vp, P_i64]),
    "rsdb_reduce_scatter_p2p": (i32, [vp, vp, vp]),
    "rsdb_all_gather_p2p": (i32, [vp, vp, vp]),
    "rsdb_reduce_scatter_adam_p2p": (i32, [vp, vp, C.POINTER(AdamState), C.POINTER(AdamCfg), i64,
                                           vp]),
    "rsdb_reduce_scatter_adam_gather_p2p": (i32, [vp, vp, C.POINTER(AdamState), C.POINTER(AdamCfg),
                                                  i64, vp]),
    "rsdb_arena_sizes": (i32, [C.POINTER(vp), i32, i32, i64, i64, P_i64, P_i64]),
    "rsdb_dbuffer_create": (i32, [C.POINTER(vp), i32, vp, i32, i64, i64, C.POINTER(vp),
                                  C.POINTER(vp)]),
    "rsdb_dbuffer_unit": (vp, [vp, i32]),
    "rsdb_dbuffer_num_blocks": (i64, [vp]),
    "rsdb_dbuffer_step_8bit_adam": (i32, [vp, C.POINTER(AdamCfg), i64, vp]),
    "rsdb_dbuffer_step_8bit_adam_dynamic": (i32, [vp, C.POINTER(AdamCfg), i64, vp]),
    "rsdb_step_8bit_adam_dynamic": (i32, [vp, C.POINTER(AdamState), C.POINTER(AdamCfg), i64, vp]),
    "rsdb_dynamic_code_maps": (i32, [C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "rsdb_dynamic_code_tables": (i32, [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "rsdb_dbuffer_zero_grads": (i32, [vp, vp]),
    "rsdb_dbuffer_step_host": (i32, [vp, vp, C.POINTER(AdamCfg), i64, C.POINTER(vp), C.POINTER(vp), vp]),
    "rsdb_dbuffer_reduce_scatter_adam": (i32, [vp, vp, C.POINTER(AdamCfg), i64, vp]),
    "rsdb_dbuffer_reduce_scatter_adam_gather": (i32, [vp, vp, C.POINTER(AdamCfg), i64, vp]),
    "rsdb_dbuffer_free": (None, [vp]),
    "rsdb_copy_plan_create": (i32, [C.POINTER(Segment), i64, i32, i32, C.c_float,
                                    C.POINTER(vp)]),
    "rsdb_copy_run": (i32, [vp, vp]),
    "rsdb_copy_plan_free": (None, [vp]),
    "rsdb_fp8_unit_create": (i32, [vp, C.POINTER(QSpec), vp, i32, vp, vp, vp, C.POINTER(vp)]),
    "rsdb_fp8_unit_num_tiles": (i64, [vp]),
    "rsdb_fp8_unit_first_slot": (i64, [vp]),
    "rsdb_fp8_quantize_all_gather": (i32, [vp, vp, vp]),
    "rsdb_fp8_unit_free": (None, [vp]),
    "rsdb_muon_create": (i32, [vp, P_i64, P_i64, vp, i32, i32, C.POINTER(vp)]),
    "rsdb_muon_select_roots": (i32, [vp, P_i64, P_i64, P_i32]),
    "rsdb_muon_root": (i32, [vp, i32]),
    "rsdb_muon_workspace_bytes": (i64, [vp]),
    "rsdb_muon_bind": (i32, [vp, C.POINTER(MuonBufs)]),
    "rsdb_muon_step": (i32, [vp, vp, C.POINTER(MuonCfg), vp]),
    "rsdb_muon_free": (None, [vp]),
    "rsdb_ns_gemm_bf16": (i32, [i32, i32, i32, vp, i64, vp, i64, C.c_float, C.c_float, vp, i64, vp, i64, vp, i64, vp]),
    "rsdb_ns_gemm_bf16_sym": (i32, [i32, i32, vp, i64, vp, i64, C.c_float, C.c_float, vp, i64, vp, i64, vp]),
    "rsdb_unit_set_shard": (i32, [vp, vp]),
    "rsdb_unit_rebind": (i32, [vp, C.POINTER(UnitBufs)]),
    "rsdb_all_gather_shards_p2p": (i32, [vp, vp, vp]),
    "rsdb_ring_create": (i32, [i32, C.POINTER(vp)]),
    "rsdb_ring_acquire": (i32, [vp, vp, P_i32]),
    "rsdb_ring_release": (i32, [vp, i32, vp]),
    "rsdb_ring_free": (None, [vp]),
}
EXPORTED = tuple(_SIGS)


class RsdbError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"rsdb status {status}: {msg}")
        self.status = status


def load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2602_22437_b200/build.py` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()


def check(status: int) -> None:
    if status != RSDB_OK:
        raise RsdbError(status, lib.rsdb_last_error().decode(errors="replace"))


def i64_array(vals):
    arr = (C.c_int64 * max(1, len(vals)))(*[int(v) for v in vals])
    return arr
