"""Oracle distributed Muon over RaggedShard (Algorithm 2):
SURVEY.md §8(f) N3.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Algorithm 2, for every 2-D parameter w:
    g <- grad(w)
    u <- MomentumUpdate(g, m)
    p <- placement(u)                       (the RaggedShard layout)
    r <- SelectRoot()                       ("load balancing")
    o <- Redistribute(u, RaggedShard(r))    (the whole matrix on rank r)
    o <- NewtonSchulz(o)                    (on the root only)
    o <- Redistribute(o, p)                 (back to the owners)
    w <- w - eta * o
P:456: "after redistribution, only the root rank holds the full 2D parameter,
so the Newton-Schulz update becomes a no-op on other ranks".

The paper prints neither MomentumUpdate, NewtonSchulz nor SelectRoot; the
readings (R21-R24) take Muon's public definition (Jordan et al.
2024, the paper's [jordan2024muon]):
  R21  MomentumUpdate (Nesterov): buf <- mu * buf + g;  u <- g + mu * buf;
       mu = 0.95.
  R22  NewtonSchulz: X <- U / (||U||_F + eps), eps = 1e-7; if rows > cols work
       on the transpose; 5 times: A <- X X^T;  B <- b A + c A A;
       X <- a X + B X;  (a, b, c) = (3.4445, -4.7750, 2.0315); transpose back.
       It maps each singular value s of U/(||U||_F+eps) to phi^5(s) with
       phi(s) = a s + b s^3 + c s^5 and keeps the singular vectors.
  R23  Update: w <- w - eta * sqrt(max(1, rows / cols)) * o   (Muon's shape
       scale), eta = 0.02.
  R24  SelectRoot: matrices in decreasing Newton-Schulz cost
       rows * cols * min(rows, cols) (stable for ties), each to the rank with
       the least cost assigned so far; ties -> the rank owning most of the
       matrix's elements, then the lowest rank (greedy LPT, deterministic).
Redistribute(u, RaggedShard(r)) concatenates every owner's piece of the
matrix in rank order -- the matrix itself (O2); Redistribute(o, p) cuts it
back at the same boundaries.  So the sharded step equals Muon applied to each
logical matrix; the pins check the pieces against that.

Pins (tests/test_oracle_muon.py): NewtonSchulz against the SVD closed form
U diag(phi^5(s)) V^T (numpy.linalg.svd, library routine) and transpose
equivariance; momentum against its closed form under a constant gradient;
SelectRoot against brute-force optimal assignment and Graham's LPT bound
(4/3 - 1/(3m)) OPT; the sharded step against the per-matrix step.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from itertools import product
from typing import List, Sequence, Tuple

import numpy as np

from .planner import Layout

NS_COEFFS = (3.4445, -4.7750, 2.0315)


@dataclass(frozen=True)
class MuonCfg:
    lr: float = 0.02
    momentum: float = 0.95
    ns_steps: int = 5
    eps: float = 1e-7


def momentum_update(buf: np.ndarray, g: np.ndarray, mu: float):
    """R21 (fp64): returns (new buf, u)."""
    buf = mu * np.asarray(buf, np.float64) + np.asarray(g, np.float64)
    return buf, np.asarray(g, np.float64) + mu * buf


def newton_schulz(G: np.ndarray, steps: int = 5, eps: float = 1e-7) -> np.ndarray:
    """R22, fp64, step by step."""
    a, b, c = NS_COEFFS
    X = np.asarray(G, np.float64)
    tall = X.shape[0] > X.shape[1]
    if tall:
        X = X.T
    X = X / (np.linalg.norm(X) + eps)
    for _ in range(steps):
        A = X @ X.T
        B = b * A + c * (A @ A)
        X = a * X + B @ X
    return X.T if tall else X


def shape_scale(rows: int, cols: int) -> float:
    """R23: sqrt(max(1, rows / cols))."""
    return math.sqrt(max(1.0, rows / cols))


def ns_cost(rows: int, cols: int) -> int:
    return rows * cols * min(rows, cols)


def owned(lay: Layout, t: int, rank: int) -> int:
    """Elements of tensor t inside rank's shard."""
    l, e = lay.starts[t], lay.numel[t]
    lo, hi = rank * lay.S, (rank + 1) * lay.S
    return max(0, min(l + e, hi) - max(l, lo))


def select_roots(lay: Layout, shapes: Sequence[Tuple[int, int]]) -> List[int]:
    """R24.  shapes[t] = (rows, cols) for matrices, None for tensors Muon
    skips (root -1)."""
    m = lay.m
    order = sorted([t for t, s in enumerate(shapes) if s is not None],
                   key=lambda t: -ns_cost(*shapes[t]))  # sorted() is stable
    load = [0] * m
    roots = [-1] * len(shapes)
    for t in order:
        r = min(range(m), key=lambda k: (load[k], -owned(lay, t, k), k))
        roots[t] = r
        load[r] += ns_cost(*shapes[t])
    return roots


def pieces(lay: Layout, t: int) -> List[Tuple[int, int, int]]:
    """(rank, offset inside the tensor, length) of every owner's piece, rank order."""
    l, e = lay.starts[t], lay.numel[t]
    out = []
    for k in range(lay.m):
        a, b = max(l, k * lay.S), min(l + e, (k + 1) * lay.S)
        if a < b:
            out.append((k, a - l, b - a))
    return out


def muon_step_sharded(lay: Layout, shapes, master: np.ndarray, buf: np.ndarray,
                      grad: np.ndarray, cfg: MuonCfg = MuonCfg()):
    """One step of Algorithm 2 over the m*S buffers (fp64; padding untouched).
    Every rank's piece is updated from its own shard (momentum), gathered to
    the root, orthogonalised there and cut back.  Returns (master, buf, roots,
    o_full) with o_full the Newton-Schulz output placed in the buffer."""
    master = np.asarray(master, np.float64).copy()
    buf = np.asarray(buf, np.float64).copy()
    o_full = np.zeros_like(master)
    roots = select_roots(lay, shapes)
    for t, sh in enumerate(shapes):
        if sh is None:
            continue
        rows, cols = sh
        l, e = lay.starts[t], lay.numel[t]
        u_pieces = []
        for k, off, n in pieces(lay, t):           # owners: momentum on their piece
            sl = slice(l + off, l + off + n)
            buf[sl], u = momentum_update(buf[sl], grad[sl], cfg.momentum)
            u_pieces.append(u)
        U = np.concatenate(u_pieces).reshape(rows, cols)  # Redistribute to the root
        O = newton_schulz(U, cfg.ns_steps, cfg.eps)       # root only
        o = O.reshape(-1)
        for k, off, n in pieces(lay, t):           # Redistribute back, owners apply
            sl = slice(l + off, l + off + n)
            o_full[sl] = o[off:off + n]
            master[sl] = master[sl] - cfg.lr * shape_scale(rows, cols) * o[off:off + n]
    return master, buf, roots, o_full


def brute_force_makespan(costs: Sequence[int], m: int) -> int:
    """Optimal max load over all assignments (tiny inputs only)."""
    best = None
    for assign in product(range(m), repeat=len(costs)):
        load = [0] * m
        for c, r in zip(costs, assign):
            load[r] += c
        mk = max(load)
        best = mk if best is None else min(best, mk)
    return best or 0
