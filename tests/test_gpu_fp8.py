"""-m gpu parity of N2 FP8 block quantization + AllGather (rsdb_fp8_*) against
oracle/fp8.py at world 1: codes and per-tile scales bit exact (both sides do
fl(x * fl(448 / A)) in fp32 and an RNE saturating E4M3 conversion, R18/R19);
padding bytes untouched.  Multi-rank parity: tests/dist_parity_worker.py."""
import numpy as np
import pytest
import torch

import paper_2602_22437_b200 as R
from oracle import fp8 as F
from oracle import planner as OP
from synth import hashgen as H

pytestmark = pytest.mark.gpu

SHAPES = [
    [(256, 384), (512, 128), (128, 200), (130, 128), (384, 64)],   # edge tiles, odd widths
    [(2048, 7168), (7168, 2048)],                                   # DSV3 expert matrices
    [(128, 4), (1, 128), (3, 3)],                                   # tiny
]


def _plan(shapes, m):
    es = [r * c for r, c in shapes]
    gs = [min(128, r) * c for r, c in shapes]
    return es, gs, R.plan(es, gs, m, elem_bytes=1), OP.plan(es, gs, m, OP.gcoll_elems(1))


def _master(E, kind, seed=0):
    if kind == "hash":
        return H.values_np(seed, H.STREAM_PARAM, 0, E, 12, outliers=True)
    rng = np.random.default_rng(seed)
    x = rng.normal(0, 0.02, E).astype(np.float32)
    x[rng.random(E) < 1e-3] *= 50
    return x


@pytest.mark.parametrize("shapes", SHAPES)
@pytest.mark.parametrize("kind", ["hash", "normal"])
def test_fp8_quantize_world1(shapes, kind):
    es, gs, lay, o = _plan(shapes, 1)
    assert list(lay.starts) == list(o.starts) and lay.S == o.S
    specs = F.tile_specs([c for _, c in shapes])
    logical = _master(sum(es), kind)
    if shapes is SHAPES[0]:
        logical[: 128 * 384] = 0.0                      # an all-zero tile row (incl. -0.0)
        logical[1:128 * 384:7] = -0.0
    full = np.zeros(lay.m * lay.S, np.float32)
    off = 0
    for l, e in zip(lay.starts, es):
        full[l:l + e] = logical[off:off + e]
        off += e
    exp_codes, exp_scales = F.quantize_all_gather(o, full, specs)
    master = torch.from_numpy(full).cuda()
    codes = torch.full((lay.m * lay.S,), 0xAB, dtype=torch.uint8, device="cuda")
    u0 = R.Fp8Unit(lay, specs, 0, master, codes, torch.empty(1, device="cuda"))
    scales = torch.full((u0.num_tiles,), float("nan"), device="cuda")
    u0.close()
    u = R.Fp8Unit(lay, specs, 0, master, codes, scales)
    assert u.num_tiles == len(exp_scales) and u.first_slot == 0
    u.quantize_all_gather()
    torch.cuda.synchronize()
    got = codes.cpu().numpy()
    mask = np.zeros(lay.m * lay.S, bool)
    for l, e in zip(lay.starts, es):
        mask[l:l + e] = True
    assert np.array_equal(got[mask], exp_codes[mask])
    assert np.all(got[~mask] == 0xAB)                    # padding never written
    assert np.array_equal(scales.cpu().numpy().view(np.uint32), exp_scales.view(np.uint32))


def test_fp8_rejects_bad_units():
    shapes = [(256, 128)]
    es, gs, lay, _ = _plan(shapes, 1)
    lay2 = R.plan(es, gs, 1, elem_bytes=2)
    t = torch.zeros(lay.S, device="cuda")
    c = torch.zeros(lay.S, dtype=torch.uint8, device="cuda")
    with pytest.raises(R.RsdbError):
        R.Fp8Unit(lay2, F.tile_specs([128]), 0, t, c, t)        # not a 1-byte layout
    with pytest.raises(R.RsdbError):
        R.Fp8Unit(lay, [("flat", 2048)], 0, t, c, t)            # needs tile specs
