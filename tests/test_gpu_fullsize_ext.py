"""-m gpu full-size parity of two §8(f) rows at the workload their
measurement scripts time (world 1; N = 2 / 4 are covered at small sizes by
tests/dist_parity_worker.py):

  * N2 FP8 128x128 quantize + AllGather on the DSV3 config-4 FFN unit
    (27 matrices, 396 M params): sampled tiles (and the last one) -- codes and
    scales bit exact against oracle/fp8.py (R18-R20);
  * N3 Muon on the Llama-3-8B decoder layer (BJ config 3): the first step's
    orthogonalised update of the 1024x4096 k_proj matrix against the fp64
    oracle (oracle/muon.py), relative Frobenius error 1e-4 (fp32) / 3e-2 (bf16).

These checks ran inside scripts/bench_fp8.py / bench_muon.py in round 1
(PASS at N = 1 / 2 / 4, profiles/r1/v9_fp8_stages, v10_muon) and moved here
because only tests/ may execute the oracle; non-fatal until this harness has
run on a B200."""
import numpy as np
import pytest
import torch

import paper_2602_22437_b200 as R
from oracle import fp8 as F
from oracle import muon as MU
from oracle import planner as OP
from synth import hashgen as H
from synth import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def test_fp8_fullsize_sampled_tiles():
    unit = W.dsv3_ffn_fp8_unit()
    shapes = [t.shape for t in unit.tensors]
    es = [t.numel for t in unit.tensors]
    gs = [128 * c for _, c in shapes]
    specs = F.tile_specs([c for _, c in shapes])
    lay = R.plan(es, gs, 1, elem_bytes=1)
    S = lay.S
    master = torch.zeros(S, dtype=torch.float32, device="cuda")
    off = 0
    for l, e in zip(lay.starts, es):
        master[l:l + e] = H.values_torch(3, H.STREAM_PARAM, off, e, 12, outliers=True, device="cuda")
        off += e
    codes = torch.zeros(S, dtype=torch.uint8, device="cuda")
    u0 = R.Fp8Unit(lay, specs, 0, master, codes, torch.empty(1, device="cuda"))
    ntiles = u0.num_tiles
    u0.close()
    scales = torch.zeros(ntiles, dtype=torch.float32, device="cuda")
    fu = R.Fp8Unit(lay, specs, 0, master, codes, scales)
    fu.quantize_all_gather(None)
    torch.cuda.synchronize()
    o = OP.plan(es, gs, 1, OP.gcoll_elems(1))
    assert o.S == S and o.starts == lay.starts
    tiles = OP.rank_tiles(o, 0, specs)
    assert len(tiles) == ntiles
    cpu_codes, cpu_scales = codes.cpu().numpy(), scales.cpu().numpy()
    rng = np.random.default_rng(0)
    for i in sorted(set(rng.integers(0, ntiles, 48).tolist() + [0, ntiles - 1])):
        toff, rows, cols, pitch = tiles[i]
        t = max(j for j in range(len(es)) if o.starts[j] <= toff)
        logical0 = sum(es[:t]) + toff - o.starts[t]
        idx = np.arange(rows)[:, None] * pitch + np.arange(cols)[None, :]
        x = H.values_np(3, H.STREAM_PARAM, logical0, int(idx.max()) + 1, 12, outliers=True)[idx]
        q, s = F.quantize_tile(x)
        assert np.array_equal(cpu_codes[toff + idx], q), f"tile {i}: codes"
        assert cpu_scales[i].view(np.uint32) == np.float32(s).view(np.uint32), f"tile {i}: scale"
    fu.close()


@pytest.mark.parametrize("precision,tol", [("f32", 1e-4), ("bf16", 3e-2)])
def test_muon_fullsize_kproj(precision, tol):
    unit = W.llama3_8b_layer(0)
    shapes = [t.shape if len(t.shape) == 2 else None for t in unit.tensors]
    es = [t.numel for t in unit.tensors]
    lay = R.plan(es, [1] * len(es), 1, elem_bytes=2)
    S = lay.S
    master, buf, grad = (H.values_torch(7, st, 0, S, 14, device="cuda") for st in (1, 2, 3))
    u = torch.zeros(S, device="cuda")
    param = torch.zeros(S, dtype=torch.bfloat16, device="cuda")
    mu = R.Muon(lay, shapes, 0, precision=precision)
    ws = torch.zeros(mu.workspace_bytes, dtype=torch.uint8, device="cuda")
    mu.bind(master, buf, grad, u, ws, param_bf16=param)
    tk = next(i for i, t in enumerate(unit.tensors) if "k_proj" in t.name)
    l, e = lay.starts[tk], es[tk]
    before = master[l:l + e].double().cpu().numpy()
    mu.step(R.MuonConfig(), None)
    torch.cuda.synchronize()
    after = master[l:l + e].double().cpu().numpy()
    g = H.values_np(7, 3, l, e, 14).astype(np.float64)
    b0 = H.values_np(7, 2, l, e, 14).astype(np.float64)
    _, uu = MU.momentum_update(b0, g, 0.95)
    rows, cols = shapes[tk]
    o = MU.newton_schulz(uu.reshape(rows, cols)).reshape(-1)
    o_gpu = (before - after) / (0.02 * MU.shape_scale(rows, cols))
    err = float(np.linalg.norm(o_gpu - o) / np.linalg.norm(o))
    assert err <= tol, err
    mu.close()
