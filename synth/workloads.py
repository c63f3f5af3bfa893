"""Synthetic parameter sets shaped like BASELINE.json's configs.

Each workload is a list of FSDP units; each unit an ordered list of
``TensorDecl(name, shape, gran)`` where ``gran`` is the user's granularity
*declaration* (P:419 ``orig_param_policy``), one of

  ("flat", q)   quantization blocks of q contiguous elements of the flattened
                tensor; the sharding block is min(q, numel)
  ("rows", r)   r rows of the last dimension (row-wise RaggedShard)
  ("whole",)    the whole tensor is one block (Muon whole-matrix)
  ("elem",)     element granularity (the paper's default)

Resolving a declaration into a block size g_t is method step a1; the oracle
(oracle/planner.py) and the product (C-ABI rsdb_block_elems) each do it.

Shapes are the public model configurations (HF config.json values), written
out by hand; nothing is downloaded.  Unit order and tensor order follow the
HF module registration order.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from math import prod
from typing import List, Sequence, Tuple

import numpy as np


@dataclass(frozen=True)
class TensorDecl:
    name: str
    shape: Tuple[int, ...]
    gran: Tuple

    @property
    def numel(self) -> int:
        return int(prod(self.shape))


@dataclass
class Unit:
    name: str
    tensors: List[TensorDecl]
    elem_bytes: int = 2  # bf16 unless stated

    @property
    def numel(self) -> int:
        return sum(t.numel for t in self.tensors)


@dataclass
class Workload:
    name: str
    units: List[Unit] = field(default_factory=list)

    @property
    def numel(self) -> int:
        return sum(u.numel for u in self.units)


def _T(name, shape, gran):
    return TensorDecl(name, tuple(int(s) for s in shape), tuple(gran))


# ----------------------------------------------------------------------------
# BJ config 1: tiny toy: 6 x (W[256,128] fp32, b[256] fp32)
# ----------------------------------------------------------------------------
def toy(q: int = 2048) -> Workload:
    ts = []
    for i in range(6):
        ts.append(_T(f"w{i}", (256, 128), ("flat", q)))
        ts.append(_T(f"b{i}", (256,), ("flat", q)))
    return Workload("toy-6x(256x128+256)-fp32", [Unit("toy", ts, elem_bytes=4)])


# ----------------------------------------------------------------------------
# BJ config 2: Llama-3.2-1B (hidden 2048, inter 8192, 32 q heads, 8 kv heads,
# head_dim 64, 16 layers, vocab 128256, tied embeddings)
# ----------------------------------------------------------------------------
def llama32_1b_layer(i: int, q: int = 2048) -> Unit:
    h, f, kv = 2048, 8192, 512
    g = ("flat", q)
    return Unit(f"layers.{i}", [
        _T("self_attn.q_proj.weight", (h, h), g),
        _T("self_attn.k_proj.weight", (kv, h), g),
        _T("self_attn.v_proj.weight", (kv, h), g),
        _T("self_attn.o_proj.weight", (h, h), g),
        _T("mlp.gate_proj.weight", (f, h), g),
        _T("mlp.up_proj.weight", (f, h), g),
        _T("mlp.down_proj.weight", (h, f), g),
        _T("input_layernorm.weight", (h,), g),
        _T("post_attention_layernorm.weight", (h,), g),
    ])


def llama32_1b_root(q: int = 2048) -> Unit:
    g = ("flat", q)
    return Unit("root", [_T("embed_tokens.weight", (128256, 2048), g),
                         _T("norm.weight", (2048,), g)])


def llama32_1b(q: int = 2048, n_layers: int = 16) -> Workload:
    units = [llama32_1b_root(q)] + [llama32_1b_layer(i, q) for i in range(n_layers)]
    return Workload("llama-3.2-1b", units)


# ----------------------------------------------------------------------------
# BJ config 3: Llama-3-8B with Muon whole-matrix blocks (hidden 4096, inter
# 14336, 32 q heads, 8 kv heads, head_dim 128, 32 layers, vocab 128256, untied)
# ----------------------------------------------------------------------------
def llama3_8b_layer(i: int) -> Unit:
    h, f, kv = 4096, 14336, 1024
    W, E = ("whole",), ("elem",)
    return Unit(f"layers.{i}", [
        _T("self_attn.q_proj.weight", (h, h), W),
        _T("self_attn.k_proj.weight", (kv, h), W),
        _T("self_attn.v_proj.weight", (kv, h), W),
        _T("self_attn.o_proj.weight", (h, h), W),
        _T("mlp.gate_proj.weight", (f, h), W),
        _T("mlp.up_proj.weight", (f, h), W),
        _T("mlp.down_proj.weight", (h, f), W),
        _T("input_layernorm.weight", (h,), E),
        _T("post_attention_layernorm.weight", (h,), E),
    ])


def llama3_8b_root() -> Unit:
    E = ("elem",)  # Muon excludes embeddings / head
    return Unit("root", [_T("embed_tokens.weight", (128256, 4096), E),
                         _T("norm.weight", (4096,), E),
                         _T("lm_head.weight", (128256, 4096), E)])


def llama3_8b_muon(n_layers: int = 32) -> Workload:
    return Workload("llama-3-8b-muon", [llama3_8b_root()] +
                    [llama3_8b_layer(i) for i in range(n_layers)])


# ----------------------------------------------------------------------------
# BJ config 4: DeepSeek-V3-style MoE layer unit with 8 local routed experts
# (EP=32 over 256), 128-row block granularity on 2-D weights, element on 1-D.
# ----------------------------------------------------------------------------
def dsv3_moe_unit(n_local_experts: int = 8, rows: int = 128) -> Unit:
    h, qa, qb, kva, kvb, o_in, mi = 7168, 1536, 24576, 576, 32768, 16384, 2048
    R, E = ("rows", rows), ("elem",)
    ts = [
        _T("self_attn.q_a_proj.weight", (qa, h), R),
        _T("self_attn.q_a_layernorm.weight", (qa,), E),
        _T("self_attn.q_b_proj.weight", (qb, qa), R),
        _T("self_attn.kv_a_proj_with_mqa.weight", (kva, h), R),
        _T("self_attn.kv_a_layernorm.weight", (512,), E),
        _T("self_attn.kv_b_proj.weight", (kvb, 512), R),
        _T("self_attn.o_proj.weight", (h, o_in), R),
        _T("mlp.gate.weight", (256, h), R),
        _T("mlp.gate.e_score_correction_bias", (256,), E),
        _T("mlp.shared_experts.gate_proj.weight", (mi, h), R),
        _T("mlp.shared_experts.up_proj.weight", (mi, h), R),
        _T("mlp.shared_experts.down_proj.weight", (h, mi), R),
    ]
    for e in range(n_local_experts):
        ts += [_T(f"mlp.experts.{e}.gate_proj.weight", (mi, h), R),
               _T(f"mlp.experts.{e}.up_proj.weight", (mi, h), R),
               _T(f"mlp.experts.{e}.down_proj.weight", (h, mi), R)]
    ts += [_T("input_layernorm.weight", (h,), E),
           _T("post_attention_layernorm.weight", (h,), E)]
    return Unit("moe_layer", ts)


def dsv3_ffn_fp8_unit(n_local_experts: int = 8) -> Unit:
    """The FFN weights of the config-4 MoE unit (shared + routed expert
    gate/up/down projections, 27 matrices, 396,361,728 params) -- the tensors a
    DeepSeek-style scheme quantizes to FP8 in 128x128 tiles -- as a
    1-byte-element unit at 128-row granularity (DESIGN R20)."""
    ts = [t for t in dsv3_moe_unit(n_local_experts, 128).tensors
          if t.name.startswith("mlp.") and t.name.endswith("_proj.weight")]
    return Unit("ffn_fp8", ts, elem_bytes=1)


def dsv3_moe(rows: int = 128) -> Workload:
    return Workload(f"dsv3-moe-unit-{rows}rows", [dsv3_moe_unit(8, rows)])


# ----------------------------------------------------------------------------
# BJ config 5: bucket sweep
# ----------------------------------------------------------------------------
def bucket(total_mb: int, seed: int = 0, elem_bytes: int = 2) -> Unit:
    """2-D [r_i, 2048] tensors, r_i in 64*{1..64}, until ~total_mb, + one [2049]."""
    rng = np.random.default_rng(seed + 7919 * total_mb)
    target = total_mb * (1 << 20) // elem_bytes
    ts, acc, i = [], 0, 0
    while acc < target:
        r = 64 * int(rng.integers(1, 65))
        if acc + r * 2048 > target:          # last tensor: fill to target (64-row steps)
            r = max(64, (target - acc) // (64 * 2048) * 64)
        ts.append(_T(f"t{i}", (r, 2048), ("elem",)))
        acc += r * 2048
        i += 1
        if r * 2048 < 64 * 2048 or acc + 64 * 2048 > target:
            break
    ts.append(_T("tail", (2049,), ("elem",)))
    return Unit(f"bucket{total_mb}MB", ts, elem_bytes=elem_bytes)


# ----------------------------------------------------------------------------
# Fig. 9 models: only FFN (MLP) weights take the row granularity;
# all other tensors element granularity.  Per-layer units + root unit.
# ----------------------------------------------------------------------------
def deepseek_v3_671b(rows: int) -> Workload:
    h, qa, qb, kva, kvb, o_in = 7168, 1536, 24576, 576, 32768, 16384
    dense_f, mi, n_exp, vocab = 18432, 2048, 256, 129280
    R, E = ("rows", rows), ("elem",)
    units = [Unit("root", [_T("embed_tokens.weight", (vocab, h), E),
                           _T("norm.weight", (h,), E),
                           _T("lm_head.weight", (vocab, h), E)])]
    for i in range(61):
        ts = [
            _T("q_a_proj", (qa, h), E), _T("q_a_layernorm", (qa,), E),
            _T("q_b_proj", (qb, qa), E), _T("kv_a_proj_with_mqa", (kva, h), E),
            _T("kv_a_layernorm", (512,), E), _T("kv_b_proj", (kvb, 512), E),
            _T("o_proj", (h, o_in), E),
        ]
        if i < 3:
            ts += [_T("gate_proj", (dense_f, h), R), _T("up_proj", (dense_f, h), R),
                   _T("down_proj", (h, dense_f), R)]
        else:
            ts += [_T("gate", (n_exp, h), E), _T("e_score_correction_bias", (n_exp,), E),
                   _T("shared.gate_proj", (mi, h), R), _T("shared.up_proj", (mi, h), R),
                   _T("shared.down_proj", (h, mi), R)]
            for e in range(n_exp):
                ts += [_T(f"experts.{e}.gate_proj", (mi, h), R),
                       _T(f"experts.{e}.up_proj", (mi, h), R),
                       _T(f"experts.{e}.down_proj", (h, mi), R)]
        ts += [_T("input_layernorm", (h,), E), _T("post_attention_layernorm", (h,), E)]
        units.append(Unit(f"layers.{i}", ts))
    return Workload(f"deepseek-v3-671b-{rows}rows", units)


def gpt_oss_120b(rows: int) -> Workload:
    """GPT-OSS-120B: experts fused into one tensor per projection."""
    h, n_exp, inter, heads, kvh, hd, vocab = 2880, 128, 2880, 64, 8, 64, 201088
    R, E = ("rows", rows), ("elem",)
    units = [Unit("root", [_T("embed_tokens.weight", (vocab, h), E),
                           _T("norm.weight", (h,), E),
                           _T("lm_head.weight", (vocab, h), E)])]
    for i in range(36):
        ts = [
            _T("q_proj.weight", (heads * hd, h), E), _T("q_proj.bias", (heads * hd,), E),
            _T("k_proj.weight", (kvh * hd, h), E), _T("k_proj.bias", (kvh * hd,), E),
            _T("v_proj.weight", (kvh * hd, h), E), _T("v_proj.bias", (kvh * hd,), E),
            _T("o_proj.weight", (h, heads * hd), E), _T("o_proj.bias", (h,), E),
            _T("sinks", (heads,), E),
            _T("router.weight", (n_exp, h), E), _T("router.bias", (n_exp,), E),
            _T("experts.gate_up_proj", (n_exp, h, 2 * inter), R),
            _T("experts.gate_up_proj_bias", (n_exp, 2 * inter), E),
            _T("experts.down_proj", (n_exp, inter, h), R),
            _T("experts.down_proj_bias", (n_exp, h), E),
            _T("input_layernorm.weight", (h,), E),
            _T("post_attention_layernorm.weight", (h,), E),
        ]
        units.append(Unit(f"layers.{i}", ts))
    return Workload(f"gpt-oss-120b-{rows}rows", units)


def all_units(w: Workload) -> Sequence[Unit]:
    return w.units
