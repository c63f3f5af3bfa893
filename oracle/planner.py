"""Oracle planner: steps a1 (granularity), a2 (Alg. 1), a3 (per-rank tables).

Written from PAPER.md §5 (Algorithm 1 at P:244-275) with the
readings of SURVEY.md §8(c) O1 / R1-R8 (restated in DESIGN.md "Readings").
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Notation follows the paper: tensors t with e_t elements and block size g_t,
m devices, per-device shard size S, interval [l_t, r_t) in a global buffer of
m*S elements; device k (0-based here) owns [k*S, (k+1)*S).

Parity pins (tests/test_oracle_planner.py):
  * validate(): the three constraints of P:226-229 -- hand-built violating
    layouts, SPEC worked examples S:175-177.
  * plan(): closed form for element granularity; textbook linear-partition
    optimum for whole-tensor blocks; brute force (exact DP over every start
    position) on >=1000 random tiny instances with the 2-approximation bound
    of P:287; SPEC worked examples S:145-146/156/165-167/186-187/195-196;
    Fig. 9 padding claims P:489; planner time P:491.
  * brute_force_min_shard(): hand-derived optima of SPEC S:186-187 (and the
    corrected S:185).
"""
from __future__ import annotations

from dataclasses import dataclass
from math import gcd
from typing import Dict, List, Optional, Sequence, Tuple

# ----------------------------------------------------------------------------
# a1: granularity -> block size g_t
# ----------------------------------------------------------------------------


def block_elems(shape: Sequence[int], gran: Tuple) -> int:
    """Sharding block size g_t in elements for one tensor declaration.

    ("flat", q) -> min(q, e_t)            (2048-element 8-bit-Adam blocks, R10)
    ("rows", r) -> r * shape[-1]           (row-wise RaggedShard), capped at e_t
    ("whole",)  -> e_t                     (whole-matrix block)
    ("elem",)   -> 1                       (element granularity)
    Non-dividing blocks are allowed: the tensor's last block is a shorter tail (R5).
    """
    e = 1
    for s in shape:
        e *= int(s)
    if e < 1:
        raise ValueError("tensor must have >= 1 element")
    kind = gran[0]
    if kind == "flat":
        q = int(gran[1])
        if q < 1:
            raise ValueError("flat block must be >= 1")
        return min(q, e)
    if kind == "rows":
        r = int(gran[1])
        if r < 1:
            raise ValueError("rows must be >= 1")
        return min(r * int(shape[-1]), e)
    if kind == "whole":
        return e
    if kind == "elem":
        return 1
    raise ValueError(f"unknown granularity {gran!r}")


def gcoll_elems(elem_bytes: int, gcoll_bytes: int = 16) -> int:
    """g_coll = 16 B / element bytes (NCCL 16-B alignment P:199)."""
    return max(1, gcoll_bytes // elem_bytes)


# ----------------------------------------------------------------------------
# a2: Algorithm 1
# ----------------------------------------------------------------------------


def place(p: int, e: int, g: int, S: int) -> Optional[int]:
    """Leftmost start l >= p at which a tensor (e elements, block g) satisfies
    the Non-Sharded Block constraint against every boundary k*S.

    This is the per-tensor step of CheckValidShard (Alg. 1 l.5-17) in the
    case analysis of P:287:
      (1) the tensor fits inside the shard that contains p;
      (2) it straddles the next boundary B: start at the first l >= p with
          (B - l) = 0 mod g, provided it does not reach B + S;
      (3) it contains whole shards: then every boundary it crosses must be at
          a block edge, which with a start aligned to B holds iff g | S.
    If starting before B fails, the tensor (longer than S) is started in the
    next shard at B + (S mod g), the leftmost start whose crossing of B + S is
    block-aligned; if that still reaches past B + 2*S (and g does not divide S)
    no start works.  Returns None when infeasible.
    """
    B = (p // S + 1) * S                     # next boundary strictly above p
    if p + e <= B:                           # case (1)
        return p
    l1 = p + ((B - p) % g)                   # first start with B - l = 0 (mod g)
    if l1 + e <= B + S or S % g == 0:        # case (2), or case (3) with g | S
        return l1
    l2 = B + (S % g)                         # start inside the next shard
    if l2 + e <= B + 2 * S:
        return l2
    return None


def feasible(es: Sequence[int], gs: Sequence[int], m: int, S: int
             ) -> Tuple[bool, List[int]]:
    """CheckValidShard(S) (Alg. 1 l.5-17).

    dp(t, i; S) of P:250 is realised by leftmost placement: the greedy keeps
    every prefix's end position minimal, so the number of shards it uses is
    the paper's dp value and the test ``dp(t_last, u_last; S) <= m``
    becomes ``end <= m*S``.  Returns (feasible, starts).
    """
    p, ls = 0, []
    for e, g in zip(es, gs):
        l = place(p, e, g, S)
        if l is None:
            return False, ls
        ls.append(l)
        p = l + e
    return p <= m * S, ls


def _ceil(a: int, b: int) -> int:
    return -(-a // b)


def search(es: Sequence[int], gs: Sequence[int], m: int, g: int) -> int:
    """S' = min{k*g : CheckValidShard(k*g)} by binary search (Alg. 1 l.21-25,
    P:287 "we binary-search for the minimal feasible S").

    The probe sequence is pinned (feasibility is not monotone on
    every input): lo = ceil(ceil(E/m)/g), hi = max(lo, ceil(E/g)); hi*g >= E is
    always feasible (all tensors in shard 0, no interior boundary).
    """
    E = sum(es)
    lo = _ceil(_ceil(E, m), g)
    hi = max(lo, _ceil(E, g))
    while lo < hi:
        mid = (lo + hi) // 2
        if feasible(es, gs, m, mid * g)[0]:
            hi = mid
        else:
            lo = mid + 1
    return lo * g


def lcm(a: int, b: int) -> int:
    return a // gcd(a, b) * b


def candidates(es: Sequence[int], gs: Sequence[int], g_coll: int) -> List[int]:
    """LCM prefixes searched by the outer loop (Alg. 1 l.19-26).

    Union of: C0 = g_coll (empty prefix); the chain over distinct g_t sorted
    ascending (Alg. 1 l.21 SortAscending(G)); the chain over g_t of tensors
    sorted by element count, descending, stable ("sort tensors by
    element count ... consider only prefixes").  A chain stops once its LCM
    exceeds E (such S' >= E cannot win).  Returned sorted, deduplicated.
    """
    E = sum(es)
    out = {g_coll}
    g = g_coll
    for gp in sorted(set(gs)):
        g = lcm(g, gp)
        if g > E:
            break
        out.add(g)
    g = g_coll
    order = sorted(range(len(es)), key=lambda i: -es[i])  # stable
    for i in order:
        g = lcm(g, gs[i])
        if g > E:
            break
        out.add(g)
    return sorted(out)


@dataclass
class Layout:
    m: int
    g_coll: int
    numel: List[int]
    block: List[int]
    S: int
    starts: List[int]

    @property
    def E(self) -> int:
        return sum(self.numel)

    @property
    def padding(self) -> int:
        return self.m * self.S - self.E

    @property
    def padding_ratio(self) -> float:
        return self.padding / self.E if self.E else 0.0

    def intervals(self) -> List[Tuple[int, int]]:
        return [(l, l + e) for l, e in zip(self.starts, self.numel)]

    def padding_intervals(self) -> List[Tuple[int, int]]:
        """Complement of the tensor intervals in [0, m*S), sorted."""
        out, p = [], 0
        for l, r in sorted(self.intervals()):
            if l > p:
                out.append((p, l))
            p = max(p, r)
        if p < self.m * self.S:
            out.append((p, self.m * self.S))
        return out


def plan(es: Sequence[int], gs: Sequence[int], m: int, g_coll: int) -> Layout:
    """Algorithm 1: S* = min over LCM prefixes of the minimal
    feasible multiple; layout = leftmost-greedy witness at S* (SURVEY R8).
    Degenerate: no tensors -> S = 0."""
    es, gs = [int(e) for e in es], [int(g) for g in gs]
    if m < 1 or g_coll < 1 or any(e < 1 for e in es) or any(g < 1 for g in gs):
        raise ValueError("invalid plan input")
    if len(es) != len(gs):
        raise ValueError("numel/block length mismatch")
    if not es:
        return Layout(m, g_coll, [], [], 0, [])
    best = None
    for g in candidates(es, gs, g_coll):
        s = search(es, gs, m, g)
        if best is None or s < best:
            best = s
    ok, ls = feasible(es, gs, m, best)
    assert ok, "S* must be feasible"
    return Layout(m, g_coll, es, gs, best, ls)


ORDER_DEFAULT, ORDER_BLOCK, ORDER_SHAPE, ORDER_BEST = 0, 1, 2, 3


def order_perm(es, gs, ordering: int, keys=None) -> List[int]:
    """Tensor orders of P:279: (i) default; (ii) sorted by sharding block
    size; (iii) sorted by tensor shape.  Reading R29: descending,
    stable; the shape order sorts by a caller-supplied shape key (identical
    shapes become adjacent).  Pinned (tests/test_oracle_planner.py): the
    buffer order read off the layout's starts is descending and stable; with
    whole-tensor blocks S is the textbook linear-partition optimum of the
    sorted sequence."""
    idx = list(range(len(es)))
    if ordering == ORDER_DEFAULT:
        return idx
    if ordering == ORDER_BLOCK:
        return sorted(idx, key=lambda i: -gs[i])
    if ordering == ORDER_SHAPE:
        if keys is None:
            raise ValueError("shape order needs keys")
        return sorted(idx, key=lambda i: -keys[i])
    raise ValueError(f"unknown ordering {ordering}")


def plan_ordered(es, gs, m, g_coll, ordering: int = ORDER_DEFAULT, keys=None) -> Layout:
    """Algorithm 1 on a permuted tensor order; starts are returned in
    input order.  ORDER_BEST plans all three orders and keeps the smallest S
    (ties: the earlier order)."""
    if ordering == ORDER_BEST:
        cands = [plan_ordered(es, gs, m, g_coll, o, keys)
                 for o in (ORDER_DEFAULT, ORDER_BLOCK, ORDER_SHAPE) if o != ORDER_SHAPE or keys is not None]
        return min(cands, key=lambda L: L.S)
    perm = order_perm(es, gs, ordering, keys)
    lay = plan([es[i] for i in perm], [gs[i] for i in perm], m, g_coll)
    starts = [0] * len(es)
    for k, i in enumerate(perm):
        starts[i] = lay.starts[k]
    return Layout(m, g_coll, list(es), list(gs), lay.S, starts)


# ----------------------------------------------------------------------------
# Validator: the optimization problem's constraints
# ----------------------------------------------------------------------------


def validate(lay: Layout) -> List[str]:
    """List of violated constraints; empty iff the layout is valid.

    (i)   r_t - l_t = e_t and r_t <= m*S             (contiguity, capacity)
    (ii)  intervals pairwise disjoint
    (iii) for every boundary k*S (k = 1..m): k*S <= l_t or k*S >= r_t or
          (k*S - l_t) = 0 (mod g_t)                 (non-sharded block)
    plus S = 0 (mod g_coll) (16-B aligned shard boundaries, R6).
    """
    v = []
    m, S = lay.m, lay.S
    if lay.numel and S % lay.g_coll != 0:
        v.append(f"S={S} not a multiple of g_coll={lay.g_coll}")
    for t, (l, e) in enumerate(zip(lay.starts, lay.numel)):
        r = l + e
        if l < 0 or r > m * S:
            v.append(f"capacity: t{t} [{l},{r}) outside [0,{m * S})")
        for k in range(1, m + 1):
            b = k * S
            if not (b <= l or b >= r or (b - l) % lay.block[t] == 0):
                v.append(f"sharded block: t{t} boundary {b} at offset {b - l} mod {lay.block[t]}")
    iv = sorted((l, l + e, t) for t, (l, e) in enumerate(zip(lay.starts, lay.numel)))
    for (l0, r0, t0), (l1, r1, t1) in zip(iv, iv[1:]):
        if l1 < r0:
            v.append(f"overlap: t{t0} [{l0},{r0}) and t{t1} [{l1},{r1})")
    return v


# ----------------------------------------------------------------------------
# Brute force (bound check only; tiny inputs, SPEC S:181 limits)
# ----------------------------------------------------------------------------


def exists_layout(es: Sequence[int], gs: Sequence[int], m: int, S: int) -> bool:
    """Exhaustive: is there ANY choice of starts (fixed order) satisfying
    P:226-229 at this S?  Tracks the set of every reachable end position
    (no greedy): tensor t may start at any l >= some reachable end of t-1."""
    import numpy as np
    N = m * S
    reach = np.zeros(N + 1, dtype=bool)
    reach[0] = True
    pos = np.arange(N + 1)
    for e, g in zip(es, gs):
        ok = np.maximum.accumulate(reach) & (pos + e <= N)
        for k in range(1, m):
            b = k * S
            ok &= ~((pos < b) & (b < pos + e) & ((b - pos) % g != 0))
        reach = np.zeros(N + 1, dtype=bool)
        reach[pos[ok] + e] = True
        if not reach.any():
            return False
    return True


def brute_force_min_shard(es: Sequence[int], gs: Sequence[int], m: int, g_coll: int,
                          limit_elems: int = 256) -> int:
    """Exact fixed-order optimum S_opt (smallest multiple of g_coll with a
    feasible layout), by exhaustive search (P:237 NP-hard; used only on tiny
    inputs)."""
    E = sum(es)
    if E > limit_elems or m > 8:
        raise ValueError("brute force limited to tiny inputs")
    if not es:
        return 0
    S = _ceil(_ceil(E, m), g_coll) * g_coll
    while not exists_layout(es, gs, m, S):
        S += g_coll
    return S


def brute_force_any_order(es, gs, m, g_coll) -> int:
    """Optimum over all tensor permutations (the NP-hard problem of P:237)."""
    from itertools import permutations
    best = None
    for perm in permutations(range(len(es))):
        s = brute_force_min_shard([es[i] for i in perm], [gs[i] for i in perm], m, g_coll)
        best = s if best is None else min(best, s)
    return best


# ----------------------------------------------------------------------------
# a3: per-rank tables (DBuffer segment map P:302-308; quant blocks P:419)
# ----------------------------------------------------------------------------


def rank_segments(lay: Layout, rank: int) -> List[Tuple[int, int, int, int]]:
    """(tensor, local offset in shard, length, offset inside tensor) of every
    piece of a tensor that lies in rank's shard [rank*S, (rank+1)*S)."""
    lo, hi = rank * lay.S, (rank + 1) * lay.S
    out = []
    for t, (l, e) in enumerate(zip(lay.starts, lay.numel)):
        a, b = max(l, lo), min(l + e, hi)
        if a < b:
            out.append((t, a - lo, b - a, a - l))
    return out


def rank_blocks(lay: Layout, rank: int, qblock: int) -> List[Tuple[int, int]]:
    """Quantization blocks owned by `rank`: (local offset, length).

    Quant block j of tensor t covers tensor elements [j*q, min((j+1)*q, e_t))
    (R10, contiguous blocks of the flattened tensor, tail shorter).  A block
    must lie wholly in one shard -- the property RaggedShard guarantees when
    g_t is a multiple of q or covers the whole tensor; otherwise this
    raises (the build's EMISMATCH)."""
    lo, hi = rank * lay.S, (rank + 1) * lay.S
    out = []
    for t, (l, e) in enumerate(zip(lay.starts, lay.numel)):
        if l + e <= lo or l >= hi:
            continue
        for j in range(_ceil(e, qblock)):
            a, b = l + j * qblock, l + min((j + 1) * qblock, e)
            if b <= lo or a >= hi:
                continue
            if a < lo or b > hi:
                raise ValueError(f"quant block {j} of tensor {t} straddles a shard boundary")
            out.append((a - lo, b - a))
    return out


def rank_tiles(lay: Layout, rank: int, specs: Sequence[Tuple]) -> List[Tuple[int, int, int, int]]:
    """Quantization blocks of `rank` when tensor t is quantized in 2-D tiles
    (the paper's setup "32x32 blocks ... 32-row block granularity",
    P:419).  specs[t] = ("tile", row_len C, tile_rows tr, tile_cols tc) views
    tensor t as [e_t / C, C] and cuts it into tr x tc tiles (edge tiles
    smaller); ("flat", q) keeps contiguous q-element blocks.  Returns
    (local offset of the tile's first element, rows, cols, pitch) for every
    block whose elements lie in rank's shard, tensors in order, tiles
    row-major; a tile that straddles a shard boundary raises."""
    lo, hi = rank * lay.S, (rank + 1) * lay.S
    out = []
    for t, (l, e) in enumerate(zip(lay.starts, lay.numel)):
        if l + e <= lo or l >= hi:
            continue
        spec = specs[t]
        if spec[0] == "flat":
            out += [(off, 1, n, n) for off, n in _flat_blocks(l, e, int(spec[1]), lo, hi, t)]
            continue
        C, tr, tc = int(spec[1]), int(spec[2]), int(spec[3])
        Rw = e // C
        if Rw * C != e:
            raise ValueError(f"tensor {t}: numel {e} is not a multiple of row_len {C}")
        for i in range(_ceil(Rw, tr)):
            rows = min(tr, Rw - i * tr)
            for j in range(_ceil(C, tc)):
                cols = min(tc, C - j * tc)
                first = l + i * tr * C + j * tc
                last = first + (rows - 1) * C + cols - 1
                if last < lo or first >= hi:
                    continue
                if first < lo or last >= hi:
                    raise ValueError(f"tile ({i},{j}) of tensor {t} straddles a shard boundary")
                out.append((first - lo, rows, cols, C))
    return out


def _flat_blocks(l, e, q, lo, hi, t):
    out = []
    for j in range(_ceil(e, q)):
        a, b = l + j * q, l + min((j + 1) * q, e)
        if b <= lo or a >= hi:
            continue
        if a < lo or b > hi:
            raise ValueError(f"quant block {j} of tensor {t} straddles a shard boundary")
        out.append((a - lo, b - a))
    return out


def to_dict(lay: Layout) -> Dict:
    return {"m": lay.m, "g_coll": lay.g_coll, "S": lay.S, "E": lay.E,
            "padding": lay.padding, "numel": list(lay.numel),
            "block": list(lay.block), "starts": list(lay.starts)}
