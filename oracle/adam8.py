"""Oracle block-wise 8-bit Adam: step a8.  SURVEY.md §8(c) O4.
TEST INFRASTRUCTURE ONLY.

PAPER.md P:419: "8-bit Adam applies *block-wise* INT8 quantization to the
gradient statistics ... each device quantizes its local shard independently
without any communication".  P:344: FP32 master weights.  The paper does not
print the update; the readings are SURVEY R9 (linear absmax code, zero absmax
-> zero codes), R10 (contiguous q-element blocks per tensor), R11 (torch
AdamW order, host fp64 scalars rounded to fp32, the update uses the fresh
fp32 m, v before requantization).

Per quant block (block = contiguous elements of one tensor, tail shorter),
every op below is one IEEE fp32 operation (RN = round to nearest even once;
steps 3 and 4 round once per fused multiply-add, as torch's lerp_ and
addcmul_ do -- reading R26), in this order:
  1. mt = q_m * fl(A_m / 127)                 dequantize first moment (signed)
  2. vt = q_v * fl(A_v / 255)                 dequantize second moment (unsigned)
  3. m  = RN(mt + w1 * fl(g - mt))            w1 = fl(1 - beta1)   (torch lerp_, weight < 0.5)
  4. v  = RN(fl(w2 * g) * g + fl(b2 * vt))    b2 = fl(beta2), w2 = fl(1 - beta2)
                                              (torch mul_(beta2).addcmul_(g, g, 1 - beta2))
  5. p  = p * c_wd                            c_wd = fl(1 - lr * wd)   (decoupled decay)
  6. p  = p + (-step_size * m) / (sqrt(v) / bc2s + eps)
                                              step_size = fl(lr / (1 - beta1^t)),
                                              bc2s = fl(sqrt(1 - beta2^t))
                                              (torch addcdiv_(m, denom, -step_size), R11)
  7. A_m' = max |m|,  A_v' = max v            over the block (NaN-propagating
                                              max: one NaN makes A' NaN, reading R27)
  8. q_m = clamp(rint(fl(m / fl(A_m' / 127))), -127, 127)   (int8)
     q_v = clamp(rint(fl(v / fl(A_v' / 255))),    0, 255)   (uint8)
     SURVEY.md §8(c) O4 step 8 as written there (before any kernel existed):
     one IEEE fp32 division by the dequantization step d = fl(A'/L), then
     round half to even.  Total for every A' (reading R27): a NaN quotient
     (0/0 when A' = 0 or d underflows to 0; anything / NaN) gives code 0,
     +-inf (x/0) saturates -- so A' = 0 gives all-zero codes, and a
     block whose A' is NaN or +inf (a non-finite gradient) gets all-zero
     codes and keeps A' (its next dequantization is then NaN: the block's
     state is visibly poisoned instead of silently wrong).
  9. param shard for the next AllGather = bf16_RNE(p)  (or p itself for fp32 units)

Parity pins (tests/test_oracle_adam8.py): step-1 closed form from the zero
state, the identity-codec variant equals torch.optim.AdamW (library routine:
m and v bit for bit, p bit for bit wherever torch's CPU sqrt is correctly
rounded), fma32 against exact rational arithmetic,
codec round trip / error bound / zero block, shard-local = unsharded result
(containment).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence, Tuple

import numpy as np

from . import codemap as CM
from .dbuffer import to_bf16_rne

f32 = np.float32


@dataclass(frozen=True)
class AdamCfg:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 1e-2


def host_scalars(cfg: AdamCfg, step: int) -> dict:
    """Per-step scalars, computed in fp64 then rounded to fp32 (R11)."""
    if step < 1:
        raise ValueError("step must be >= 1")
    return {
        "w1": f32(1.0 - cfg.beta1),
        "b2": f32(cfg.beta2),
        "w2": f32(1.0 - cfg.beta2),
        "eps": f32(cfg.eps),
        "c_wd": f32(1.0 - cfg.lr * cfg.weight_decay),
        "step_size": f32(cfg.lr / (1.0 - cfg.beta1 ** step)),
        "bc2s": f32(np.sqrt(1.0 - cfg.beta2 ** step)),
    }


def fma32(a, b, c) -> np.ndarray:
    """RN32(a*b + c) for fp32 a, b, c: the exact value rounded once to fp32
    (a fused multiply-add).  a*b is exact in fp64 (24 + 24 <= 53 bits); the
    fp64 sum s and its exact error e (TwoSum) give exact = s + e.  RN32(s)
    equals RN32(exact) unless s lies exactly on a midpoint between two fp32
    values while e != 0 -- then the sign of e picks the side."""
    a, b, c = (np.asarray(x, np.float32).astype(np.float64) for x in (a, b, c))
    ab = a * b
    s = ab + c
    bv = s - ab
    e = (ab - (s - bv)) + (c - bv)
    r = s.astype(np.float32)
    r64 = r.astype(np.float64)
    other = np.nextafter(r, np.where(s > r64, np.inf, -np.inf).astype(np.float32)).astype(np.float64)
    on_mid = (s != r64) & (s == (r64 + other) / 2) & (e != 0)
    fix = np.where(e > 0, np.maximum(r64, other), np.minimum(r64, other)).astype(np.float32)
    return np.where(on_mid, fix, r).astype(np.float32)


def dequantize(codes: np.ndarray, absmax: f32, signed: bool) -> np.ndarray:
    levels = f32(127.0) if signed else f32(255.0)
    with np.errstate(invalid="ignore", under="ignore"):  # 0 * inf = NaN (R27)
        scale = f32(f32(absmax) / levels)
        return (codes.astype(np.float32) * scale).astype(np.float32)


def quantize(x: np.ndarray, signed: bool) -> Tuple[np.ndarray, f32]:
    """Linear absmax code of one block (R9; step 8 above, R27); returns
    (codes, absmax)."""
    x = np.asarray(x, dtype=np.float32)
    a = f32(np.max(np.abs(x))) if x.size else f32(0)  # numpy's max propagates NaN
    levels = f32(127.0) if signed else f32(255.0)
    lo, hi = (-127, 127) if signed else (0, 255)
    with np.errstate(divide="ignore", invalid="ignore", over="ignore", under="ignore"):
        d = f32(a / levels)
        y = (x / d).astype(np.float32)  # IEEE fp32 division (correctly rounded)
    q = np.where(np.isnan(y), f32(0), np.clip(np.rint(y), lo, hi))
    return q.astype(np.int8 if signed else np.uint8), a


def adam_block_update(p, g, mt, vt, sc):
    """Steps 3-6 on fp32 arrays (shared by the 8-bit and identity-codec
    variants); returns (p_new, m, v)."""
    g = np.asarray(g, dtype=np.float32)
    m = fma32(sc["w1"], (g - mt).astype(np.float32), mt)
    v = fma32((sc["w2"] * g).astype(np.float32), g, (sc["b2"] * vt).astype(np.float32))
    p = (p * sc["c_wd"]).astype(np.float32)
    denom = ((np.sqrt(v).astype(np.float32) / sc["bc2s"]).astype(np.float32) + sc["eps"]).astype(np.float32)
    p = (p + ((-sc["step_size"] * m).astype(np.float32) / denom).astype(np.float32)).astype(np.float32)
    return p, m, v


def step_8bit_adam(master: np.ndarray, grad: np.ndarray, m_q: np.ndarray, v_q: np.ndarray,
                   m_abs: np.ndarray, v_abs: np.ndarray, blocks: Sequence[Tuple[int, int]],
                   cfg: AdamCfg, step: int, out_bf16: bool = True, codec: str = "linear"):
    """One 8-bit Adam step on a rank's local shard, block by block.

    master/grad: fp32 [S]; m_q int8 [S]; v_q uint8 [S]; m_abs/v_abs fp32
    [len(blocks)]; blocks = rank_blocks(...) table of (local offset, len), or
    rank_tiles(...) table of 2-D tiles (offset of first element, rows, cols,
    pitch) -- a block is the set of its elements, the update is the same.
    Returns new copies (master, m_q, v_q, m_abs, v_abs, param_shard) where
    param_shard is bf16 bit patterns (uint16) or fp32; positions outside any
    block are left unchanged (param shard: 0).  codec "dynamic": both moments
    use the dynamic tree maps of oracle/codemap.py (R25; m_q holds uint8 map
    indices) instead of the linear absmax codes (R9)."""
    if codec not in ("linear", "dynamic"):
        raise ValueError(codec)
    sc = host_scalars(cfg, step)
    with np.errstate(all="ignore"):  # non-finite gradients propagate as IEEE says (R27)
        return _step_8bit_adam(master, grad, m_q, v_q, m_abs, v_abs, blocks, sc, out_bf16, codec)


def _step_8bit_adam(master, grad, m_q, v_q, m_abs, v_abs, blocks, sc, out_bf16, codec):
    master = np.array(master, dtype=np.float32, copy=True)
    m_q, v_q = np.array(m_q, copy=True), np.array(v_q, copy=True)
    m_abs = np.array(m_abs, dtype=np.float32, copy=True)
    v_abs = np.array(v_abs, dtype=np.float32, copy=True)
    param = np.zeros(master.shape, np.uint16 if out_bf16 else np.float32)
    for b, blk in enumerate(blocks):
        if len(blk) == 2:
            s = slice(blk[0], blk[0] + blk[1])
        else:  # 2-D tile: element (a, c) at off + a * pitch + c
            off, rows, cols, pitch = blk
            s = (off + np.arange(rows)[:, None] * pitch + np.arange(cols)[None, :]).ravel()
        if codec == "linear":
            mt = dequantize(m_q[s], m_abs[b], signed=True)
            vt = dequantize(v_q[s], v_abs[b], signed=False)
        else:
            mt = CM.dyn_dequantize(m_q[s], m_abs[b], signed=True)
            vt = CM.dyn_dequantize(v_q[s], v_abs[b], signed=False)
        p, m, v = adam_block_update(master[s], grad[s], mt, vt, sc)
        master[s] = p
        if codec == "linear":
            m_q[s], m_abs[b] = quantize(m, signed=True)
            v_q[s], v_abs[b] = quantize(v, signed=False)
        else:
            m_q[s], m_abs[b] = CM.dyn_quantize(m, signed=True)
            v_q[s], v_abs[b] = CM.dyn_quantize(v, signed=False)
        param[s] = to_bf16_rne(p) if out_bf16 else p
    return master, m_q, v_q, m_abs, v_abs, param


def step_adam_fp32_states(master, grad, m, v, cfg: AdamCfg, step: int):
    """Identity-codec variant (states kept in fp32, no quantization): the
    special case that must reduce to torch.optim.AdamW (pin)."""
    sc = host_scalars(cfg, step)
    return adam_block_update(np.asarray(master, np.float32), grad,
                             np.asarray(m, np.float32), np.asarray(v, np.float32), sc)
