"""-m gpu parity of N3 distributed Muon (rsdb_muon_*, Algorithm 2)
against oracle/muon.py (fp64) at world 1; N=2/4 in tests/dist_parity_worker.py.

Tolerances: momentum buffer rtol 1e-6; the orthogonalised
update o (recovered from the master change) per matrix within relative
Frobenius 1e-4 for the fp32 Newton-Schulz (numpy fp32 runs of the same
algorithm differ from fp64 by ~2e-6) and 3e-2 for the bf16 tensor-core mode
(bf16-rounding emulation differs by ~1.1e-2); tensors Muon skips and padding
are untouched; the bf16 shard is RNE(master) exactly."""
import numpy as np
import pytest
import torch

import paper_2602_22437_b200 as R
from oracle import muon as MU
from oracle import planner as OP

pytestmark = pytest.mark.gpu

SHAPES = [(24, 40), None, (40, 24), (16, 16), None, (96, 160), (160, 96), (1, 64)]
TOL = {"f32": 1e-4, "bf16": 3e-2}


def muon_case(m, rank, shapes, seed, steps, precision, comm=None, p2p_factory=None):
    """Runs `steps` Muon steps on rank `rank` of m; returns (ok, messages)."""
    es = [s[0] * s[1] if s else 37 + i for i, s in enumerate(shapes)]
    lay = R.plan(es, [1] * len(es), m, elem_bytes=2)
    o = OP.plan(es, [1] * len(es), m, 8)
    assert list(lay.starts) == list(o.starts) and lay.S == o.S
    S = lay.S
    rng = np.random.default_rng(seed)
    full = []
    for scale in (0.02, 0.01, 0.01):  # master, momentum buffer, gradient
        f = np.zeros(m * S)
        for l, e in zip(lay.starts, es):
            f[l:l + e] = rng.normal(0, scale, e).astype(np.float32)
        full.append(f)
    sh = slice(rank * S, (rank + 1) * S)
    dev = lambda a: torch.from_numpy(a[sh].astype(np.float32)).cuda()  # noqa: E731
    master, buf, grad = dev(full[0]), dev(full[1]), dev(full[2])
    u = torch.zeros(S, device="cuda")
    param = torch.zeros(S, dtype=torch.bfloat16, device="cuda")
    mu = R.Muon(lay, shapes, rank, comm=comm, precision=precision)
    ws = torch.zeros(mu.workspace_bytes, dtype=torch.uint8, device="cuda")
    mu.bind(master, buf, grad, u, ws, param_bf16=param)
    p2p = p2p_factory(u, ws) if p2p_factory else None
    roots_ref = MU.select_roots(o, shapes)
    assert [mu.root(t) for t in range(len(shapes))] == roots_ref
    ref_m, ref_b, ref_g = full
    msgs = []
    m0_gpu = master.cpu().numpy().astype(np.float64)
    for step in range(steps):
        prev = ref_m.copy()
        ref_m, ref_b, _, o_full = MU.muon_step_sharded(o, shapes, ref_m, ref_b, ref_g)
        prev_gpu = master.cpu().numpy().astype(np.float64) if step else m0_gpu
        mu.step(R.MuonConfig(), p2p)
        torch.cuda.synchronize()
        gm = master.cpu().numpy().astype(np.float64)
        gb = buf.cpu().numpy().astype(np.float64)
        if not np.allclose(gb, ref_b[sh], rtol=1e-6, atol=1e-9):
            msgs.append(f"step {step}: momentum buffer off by {np.abs(gb - ref_b[sh]).max():.3e}")
        for t, s in enumerate(shapes):
            a, b = max(lay.starts[t], rank * S), min(lay.starts[t] + es[t], (rank + 1) * S)
            if a >= b:
                continue
            loc = slice(a - rank * S, b - rank * S)
            if s is None:
                if not np.array_equal(gm[loc], prev_gpu[loc]):
                    msgs.append(f"tensor {t} (not a matrix) changed")
                continue
            coef = 0.02 * MU.shape_scale(*s)
            o_gpu = (prev_gpu[loc] - gm[loc]) / coef
            o_ref = o_full[a:b]
            err = np.linalg.norm(o_gpu - o_ref) / max(np.linalg.norm(o_ref), 1e-30)
            # per-piece relative Frobenius (pieces of a straddling matrix share the bound)
            if err > TOL[precision]:
                msgs.append(f"step {step} tensor {t} {s}: o rel err {err:.3e}")
        pad = np.ones(S, bool)
        for l, e in zip(lay.starts, es):
            a, b = max(l, rank * S), min(l + e, (rank + 1) * S)
            if a < b:
                pad[a - rank * S:b - rank * S] = False
        if np.any(gm[pad] != 0):
            msgs.append("padding written")
        # resync the oracle to the GPU state (multi-step: errors must not compound)
        ref_m = ref_m.copy()
        ref_m[sh] = gm
    pb = param.view(torch.int16).cpu().numpy()
    rne = master.to(torch.bfloat16).view(torch.int16).cpu().numpy()
    touched = np.zeros(S, bool)
    for t, s in enumerate(shapes):
        a, b = max(lay.starts[t], rank * S), min(lay.starts[t] + es[t], (rank + 1) * S)
        if s is not None and a < b:
            touched[a - rank * S:b - rank * S] = True
    if not np.array_equal(pb[touched], rne[touched]):
        msgs.append("bf16 shard != RNE(master)")
    if p2p is not None:
        torch.cuda.synchronize()
        p2p.close()
    mu.close()
    return not msgs, msgs


@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_muon_world1(precision):
    ok, msgs = muon_case(1, 0, SHAPES, 0, 2, precision)
    assert ok, msgs


def test_muon_big_matrix_world1():
    ok, msgs = muon_case(1, 0, [(512, 1536), None, (1536, 512)], 1, 1, "f32")
    assert ok, msgs
