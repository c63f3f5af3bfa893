"""CPU tests of the C-ABI library (no compute calls need a GPU here):
  * librsdb.so loads and exports every symbol include/rsdb.h declares;
  * the C++ planner is bit-exact with the oracle (layouts, tables, padding)
    on >= 10,000 random instances, every BJ config and the Fig. 9 sweeps;
  * error behaviour stated in the header; device calls fail loudly (no CPU
    fallback) when there is no GPU;
  * planner speed claim P:491 (< 0.3 s per unit) for the C++ planner.
"""
import ctypes as C
import os
import random
import re
import time

import numpy as np
import pytest
import torch

import paper_2602_22437_b200 as R
from paper_2602_22437_b200 import _capi
from oracle import planner as P
from synth import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "rsdb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rsdb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    syms = _header_symbols()
    assert len(syms) >= 35
    lib = C.CDLL(_capi.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _capi.EXPORTED, f"{s} declared in rsdb.h but not bound"
    assert set(_capi.EXPORTED) == set(syms)
    assert R.lib.rsdb_abi_version() == 1


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def _cmp(es, gs, m, eb):
    gc = P.gcoll_elems(eb)
    o = P.plan(es, gs, m, gc)
    c = R.plan(es, gs, m, elem_bytes=eb)
    assert c.S == o.S, (es, gs, m, eb)
    assert c.starts == o.starts
    assert c.padding == o.padding and c.E == o.E
    assert c.validate() == 0
    assert c.padding_intervals() == o.padding_intervals()
    return o, c


def test_planner_parity_random_tiny():
    rng = random.Random(11)
    for _ in range(10000):
        n = rng.randint(0, 7)
        es = [rng.randint(1, 64) for _ in range(n)]
        gs = [rng.randint(1, 9) for _ in range(n)]
        _cmp(es, gs, rng.randint(1, 9), rng.choice([1, 2, 4]))


def test_planner_parity_random_medium_and_tables():
    rng = random.Random(12)
    for _ in range(400):
        n = rng.randint(1, 30)
        q = rng.choice([16, 64, 2048])
        es = [rng.randint(1, 20000) for _ in range(n)]
        kind = rng.random()
        if kind < 0.4:
            gs = [min(q, e) for e in es]
        elif kind < 0.7:
            gs = [rng.choice([1, e, max(1, e // 7)]) for e in es]
        else:
            gs = [rng.randint(1, 300) for _ in es]
        m = rng.choice([1, 2, 3, 4, 8, 16])
        o, c = _cmp(es, gs, m, rng.choice([2, 4]))
        for r in range(m):
            assert c.rank_segments(r) == [tuple(x) for x in P.rank_segments(o, r)]
            try:
                ob = P.rank_blocks(o, r, q)
            except ValueError:
                with pytest.raises(R.RsdbError) as ei:
                    c.rank_blocks(r, q)
                assert ei.value.status == _capi.RSDB_EMISMATCH
                continue
            assert c.rank_blocks(r, q) == [tuple(x) for x in ob]


@pytest.mark.parametrize("wl", ["toy", "llama", "llama8b", "dsv3"])
def test_planner_parity_bj_configs(wl):
    units = {"toy": W.toy().units, "llama": W.llama32_1b().units[:2],
             "llama8b": [W.llama3_8b_layer(0), W.llama3_8b_root()],
             "dsv3": [W.dsv3_moe_unit()]}[wl]
    for u in units:
        es = [t.numel for t in u.tensors]
        gs = [P.block_elems(t.shape, t.gran) for t in u.tensors]
        assert gs == [R.block_elems(t.shape, t.gran) for t in u.tensors]
        for m in (1, 2, 4, 8):
            o, c = _cmp(es, gs, m, u.elem_bytes)
            assert c.to_json() == P.to_dict(o)


def test_planner_parity_fig9_sweep():
    for mk in (W.deepseek_v3_671b, W.gpt_oss_120b):
        for rows in (1, 16, 128):
            wl = mk(rows)
            seen = set()
            for u in wl.units:
                key = tuple((t.numel, P.block_elems(t.shape, t.gran)) for t in u.tensors)
                if key in seen:
                    continue
                seen.add(key)
                es = [k[0] for k in key]
                gs = [k[1] for k in key]
                for m in (8, 64, 256, 1024):
                    _cmp(es, gs, m, 2)


def test_cpp_planner_time_claim():
    """< 0.3 s per unit; the largest unit (DSV3 MoE layer, 777 tensors)."""
    u = W.deepseek_v3_671b(128).units[10]
    es = [t.numel for t in u.tensors]
    gs = [R.block_elems(t.shape, t.gran) for t in u.tensors]
    for m in (8, 1024):
        t0 = time.perf_counter()
        lay = R.plan(es, gs, m)
        dt = time.perf_counter() - t0
        assert lay.validate() == 0 and dt < 0.3


def test_error_behaviour():
    with pytest.raises(R.RsdbError) as e:
        R.plan([4], [0], 2)
    assert e.value.status == _capi.RSDB_EINVAL
    with pytest.raises(R.RsdbError):
        R.plan([4], [1], 0)
    with pytest.raises(R.RsdbError):
        R.plan([0], [1], 2)
    with pytest.raises(R.RsdbError):
        R.plan([4], [1], 2, elem_bytes=3)
    with pytest.raises(R.RsdbError):
        R.block_elems([4, 0], ("flat", 8))
    with pytest.raises(R.RsdbError):
        R.block_elems([4], ("flat", 0))
    lay = R.plan([], [], 4)
    assert lay.S == 0 and lay.starts == [] and lay.padding == 0
    with pytest.raises(R.RsdbError) as e:
        R.plan([8], [1], 2, elem_bytes=4).rank_blocks(0, 8)
    assert e.value.status == _capi.RSDB_EMISMATCH
    with pytest.raises(R.RsdbError):
        R.plan([8], [1], 2).rank_blocks(5, 8)
    # explicit layouts are validated against P:226-229
    good = R.layout_from_starts([6, 4], [3, 2], 2, 6, [0, 6], elem_bytes=4, gcoll_bytes=4)
    assert good.S == 6 and good.validate() == 0
    with pytest.raises(R.RsdbError):
        R.layout_from_starts([6], [3], 2, 4, [0], elem_bytes=4, gcoll_bytes=4)
    odd = R.layout_from_starts([9], [1], 2, 5, [0], elem_bytes=2, require_gcoll=False)
    assert odd.S == 5


def test_block_elems_kinds():
    assert R.block_elems([256, 128], ("flat", 2048)) == 2048
    assert R.block_elems([256], ("flat", 2048)) == 256
    assert R.block_elems([576, 7168], ("rows", 128)) == 128 * 7168
    assert R.block_elems([100, 10], ("rows", 128)) == 1000
    assert R.block_elems([3, 5], ("whole",)) == 15
    assert R.block_elems([3, 5], ("elem",)) == 1


def test_arena_sizes_alignment_and_disjointness():
    lays = [R.plan([t.numel for t in u.tensors], [R.block_elems(t.shape, t.gran) for t in u.tensors], 4)
            for u in W.llama32_1b().units[:3]]
    for rank in range(4):
        sizes, offs = R.arena_sizes(lays, rank, 2048, 256)
        for k in range(8):
            spans = []
            for u, lay in enumerate(lays):
                assert offs[u][k] % 256 == 0
                per = {0: lay.m * lay.S * 2, 1: lay.m * lay.S * 2, 2: lay.m * lay.S * 4,
                       3: lay.S * 4, 4: lay.S, 5: lay.S,
                       6: 4 * len(lay.rank_blocks(rank, 2048)), 7: 4 * len(lay.rank_blocks(rank, 2048))}[k]
                spans.append((offs[u][k], offs[u][k] + per))
                assert offs[u][k] + per <= sizes[k]
            spans.sort()
            assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:]))
            # master / mq / vq share element offsets
        assert [o[3] // 4 for o in offs] == [o[4] for o in offs] == [o[5] for o in offs]


def test_orderings_match_oracle_and_best_is_best():
    """N4 / P:279: the three tensor orders and their best; C++ == oracle."""
    rng = random.Random(31)
    for _ in range(300):
        n = rng.randint(1, 9)
        es = [rng.randint(1, 500) for _ in range(n)]
        gs = [rng.choice([1, e, max(1, e // 3), 7]) for e in es]
        gs = [min(g, e) for g, e in zip(gs, es)]
        keys = [rng.randint(0, 3) for _ in range(n)]
        m = rng.randint(1, 6)
        for name, o in (("default", 0), ("block", 1), ("shape", 2), ("best", 3)):
            ol = P.plan_ordered(es, gs, m, 4, o, keys)
            cl = R.plan_ordered(es, gs, m, name, keys, elem_bytes=4)
            assert cl.S == ol.S and cl.starts == ol.starts, (name, es, gs, m)
            assert cl.validate() == 0 and P.validate(ol) == []
        best = P.plan_ordered(es, gs, m, 4, 3, keys).S
        assert best <= min(P.plan_ordered(es, gs, m, 4, o, keys).S for o in (0, 1, 2))


def test_tile_tables_match_oracle():
    """N2: 2-D quantization tiles (32x32 with 32-row granularity) --
    C++ tables bit-exact with the oracle's; straddles rejected alike."""
    rng = random.Random(21)
    for _ in range(150):
        n = rng.randint(1, 6)
        shapes, specs, gs = [], [], []
        for _ in range(n):
            if rng.random() < 0.7:
                C_ = rng.choice([16, 40, 64, 96, 130])
                R_ = rng.choice([7, 32, 45, 64, 100])
                tr, tc = rng.choice([(32, 32), (8, 16), (1, C_), (32, 128)])
                shapes.append((R_, C_))
                specs.append(("tile", C_, tr, tc))
                gs.append(rng.choice([tr * C_, R_ * C_, 2 * tr * C_]))
            else:
                e = rng.randint(1, 3000)
                q = rng.choice([64, 1024])
                shapes.append((e,))
                specs.append(("flat", q))
                gs.append(min(q, e))
        es = [int(np.prod(s)) for s in shapes]
        gs = [min(g, e) for g, e in zip(gs, es)]
        m = rng.randint(1, 5)
        o = P.plan(es, gs, m, 4)
        c = R.plan(es, gs, m, elem_bytes=4)
        for r in range(m):
            try:
                ot = P.rank_tiles(o, r, specs)
            except ValueError:
                with pytest.raises(R.RsdbError) as ei:
                    c.rank_tiles(r, specs)
                assert ei.value.status == _capi.RSDB_EMISMATCH
                continue
            assert c.rank_tiles(r, specs) == [tuple(x) for x in ot]


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_device_calls_fail_loudly_without_gpu():
    lay = R.plan([4096], [2048], 1)
    with pytest.raises(R.RsdbError) as e:
        R.Unit(lay, 0, 256, 256, 512, qblock=2048)
    assert e.value.status == _capi.RSDB_ECUDA
    assert "no CPU fallback" in str(e.value)
    with pytest.raises(R.RsdbError) as e:
        R.Comm(b"\0" * 128, 1, 0, 0)
    assert e.value.status == _capi.RSDB_ECUDA


def test_muon_select_roots_matches_oracle():
    """N3 SelectRoot (R24): the C++ assignment equals the oracle's on random
    layouts (matrices straddling ranks, skipped 1-D tensors) and on the
    Llama-3-8B layer unit at element granularity."""
    from oracle import muon as MU
    rng = random.Random(11)
    for _ in range(300):
        m = rng.randint(1, 8)
        shapes = [None if rng.random() < 0.25 else (rng.randint(1, 40), rng.randint(1, 40))
                  for _ in range(rng.randint(1, 12))]
        es = [s[0] * s[1] if s else rng.randint(1, 50) for s in shapes]
        o = P.plan(es, [1] * len(es), m, 8)
        c = R.plan(es, [1] * len(es), m, elem_bytes=2)
        assert R.muon_select_roots(c, shapes) == MU.select_roots(o, shapes)
    u = W.llama3_8b_layer(0)
    shapes = [t.shape if len(t.shape) == 2 else None for t in u.tensors]
    es = [t.numel for t in u.tensors]
    for m in (2, 4, 8):
        o = P.plan(es, [1] * len(es), m, 8)
        c = R.plan(es, [1] * len(es), m, elem_bytes=2)
        assert R.muon_select_roots(c, shapes) == MU.select_roots(o, shapes)
    with pytest.raises(R.RsdbError):
        R.muon_select_roots(R.plan([12], [1], 1), [(5, 3)])  # rows * cols != numel


def test_dynamic_code_maps_match_oracle():
    """N2 dynamic codec (R25): the C++ maps (built independently in double) are
    bit-identical to the oracle's."""
    from oracle import codemap as CM
    m, v = R.dynamic_code_maps()
    assert np.array_equal(np.array(m, np.float32).view(np.uint32), CM.dynamic_map(True).view(np.uint32))
    assert np.array_equal(np.array(v, np.float32).view(np.uint32), CM.dynamic_map(False).view(np.uint32))


def test_fsdp_sweep_tool_accounting():
    """N4 sweep tool (scripts/fsdp_sweep.py, analytic mode): the DBuffer bytes
    are the exact sum of rsdb_arena_sizes, padding and wire bytes follow the
    layouts, and FSDP2's dim-0 padding appears where rows % m != 0."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("fsdp_sweep", os.path.join(ROOT, "scripts", "fsdp_sweep.py"))
    fs = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(fs)
    w = W.dsv3_moe()
    line = fs.sweep_one(w, 7, measure=False)
    u = w.units[0]
    gs = [R.block_elems(t.shape, t.gran) for t in u.tensors]
    lay = R.plan([t.numel for t in u.tensors], gs, 7)
    sizes, _ = R.arena_sizes([lay], 0, 2048, 256, qspec=[[("flat", min(2048, g)) for g in gs]])
    assert line["dbuffer_bytes"] == sum(sizes)
    assert line["ag_wire_bytes_per_rank"] == 6 * lay.S * 2
    assert abs(line["ragged_padding_pct"] - 100.0 * (7 * lay.S - lay.E) / lay.E) < 1e-9
    assert line["fsdp2_dim0_padding_pct"] > 0  # rows not divisible by 7 pad dim 0
    assert line["fsdp2_allocations"] == 8 * len(u.tensors)
    # row-wise-128 padding 0.24 / 0.86 / 2.12 % at m = 2 / 4 / 8
    for m, pct in ((2, 0.24), (4, 0.86), (8, 2.12)):
        assert abs(fs.sweep_one(w, m, measure=False)["fsdp2_rowwise_block_padding_pct"] - pct) < 0.006


def test_extension_entry_points_error_behaviour():
    """The §8(f) / §7 extensions validate their arguments before touching a
    device (header: EINVAL / EMISMATCH), and fail loudly (ECUDA) without one."""
    from oracle import fp8 as F
    lay2 = R.plan([256 * 128], [128 * 128], 1, elem_bytes=2)
    lay1 = R.plan([256 * 128], [128 * 128], 1, elem_bytes=1)
    with pytest.raises(R.RsdbError) as e:          # FP8 units are 1-byte layouts
        R.Fp8Unit(lay2, F.tile_specs([128]), 0, None, None, None)
    assert e.value.status == _capi.RSDB_EMISMATCH
    with pytest.raises(R.RsdbError) as e:          # tile specs required
        R.Fp8Unit(lay1, [("flat", 2048)], 0, None, None, None)
    assert e.value.status == _capi.RSDB_EINVAL
    with pytest.raises(R.RsdbError) as e:          # rows * cols must equal numel
        R.Muon(lay2, [(100, 100)], 0)
    assert e.value.status == _capi.RSDB_EINVAL
    with pytest.raises(R.RsdbError) as e:          # world > 1 needs a comm
        R.Muon(R.plan([64], [1], 2), [(8, 8)], 0)
    assert e.value.status == _capi.RSDB_EINVAL
    with pytest.raises(R.RsdbError) as e:          # valid arguments, no GPU here
        R.Muon(lay2, [(256, 128)], 0)
    assert e.value.status == _capi.RSDB_ECUDA
    with pytest.raises(R.RsdbError) as e:
        R.Ring(0)
    assert e.value.status == _capi.RSDB_EINVAL
    with pytest.raises(R.RsdbError) as e:
        R.Ring(2)
    assert e.value.status == _capi.RSDB_ECUDA


def test_round2_entry_points_error_behaviour():
    """Round-2 entry points check their arguments before any device work:
    rsdb_ns_gemm_bf16(_sym) (N3), rsdb_dbuffer_step_host, rsdb_p2p_channel,
    rsdb_unit_create with qblock < 0; valid GEMM arguments without a GPU give
    ECUDA (no CPU fallback)."""
    lib = _capi.lib
    C = __import__("ctypes")
    f = C.c_float
    # dimensions / leading dimensions: K < 1, ld not a multiple of 8, ld < row length
    for args in ((16, 16, 0, 16, 16, 16), (16, 16, 16, 20, 16, 16), (16, 16, 16, 8, 16, 16)):
        M, N, K, lda, ldb, ldc = args
        st = lib.rsdb_ns_gemm_bf16(M, N, K, 4096, lda, 4096, ldb, f(1.0), f(0.0), None, 0, 4096, ldc,
                                   None, 0, None)
        assert st == _capi.RSDB_EINVAL, args
    st = lib.rsdb_ns_gemm_bf16(16, 16, 16, 4096, 16, 4096, 16, f(1.0), f(0.0), None, 0, 4096, 16, None, 0, None)
    assert st == _capi.RSDB_ECUDA
    assert lib.rsdb_ns_gemm_bf16_sym(16, 16, 4096, 16, 4096, 16, f(1.0), f(2.0), None, 0, 4096, 16,
                                     None) == _capi.RSDB_EINVAL  # beta != 0 needs D
    assert lib.rsdb_dbuffer_step_host(None, None, None, 1, None, None, None) == _capi.RSDB_EINVAL
    out = C.c_void_p()
    assert lib.rsdb_p2p_channel(None, 1, C.byref(out)) == _capi.RSDB_EINVAL
    assert lib.rsdb_p2p_set_max_ctas(None, 4) == _capi.RSDB_EINVAL
    assert lib.rsdb_p2p_barrier(None, None) == _capi.RSDB_EINVAL
    lay = R.plan([4096], [2048], 1)
    bufs = _capi.UnitBufs(4096, 8192, 16384)
    assert lib.rsdb_unit_create(lay.handle, None, 0, C.byref(bufs), -1, C.byref(out)) == _capi.RSDB_EINVAL


# ------------------------------------------------ header <-> binding agreement
_STRUCTS = {  # C typedef -> ctypes class in the binding
    "rsdb_qspec": "QSpec", "rsdb_unit_bufs": "UnitBufs", "rsdb_adam_cfg": "AdamCfg",
    "rsdb_adam_state": "AdamState", "rsdb_segment": "Segment", "rsdb_muon_cfg": "MuonCfg",
    "rsdb_muon_bufs": "MuonBufs",
}


def test_header_defines_match_the_binding():
    import re
    from paper_2602_22437_b200 import _capi as CB
    import paper_2602_22437_b200 as R
    hdr = open(os.path.join(ROOT, "include", "rsdb.h")).read()
    defines = {k: int(v) for k, v in re.findall(r"^#define (RSDB_\w+) (\d+)", hdr, re.M)}
    assert len(defines) >= 25
    for name, val in defines.items():
        if name.startswith("RSDB_ORDER_"):
            assert R.ORDER[name[len("RSDB_ORDER_"):].lower()] == val, name
        else:
            assert getattr(CB, name) == val, name


def test_struct_layouts_match_the_header(tmp_path):
    """sizeof / offsetof of every public struct, compiled from include/rsdb.h
    with gcc, equals the ctypes declaration the binding marshals with."""
    import shutil
    import subprocess
    from paper_2602_22437_b200 import _capi as CB
    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "rsdb.h"', "int main(void) {"]
    for cname, pyname in _STRUCTS.items():
        cls = getattr(CB, pyname)
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "abi.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = {}
    for ln in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines():
        c, f, v = ln.split()
        got[(c, f)] = int(v)
    for cname, pyname in _STRUCTS.items():
        cls = getattr(CB, pyname)
        assert got[(cname, "size")] == C.sizeof(cls), cname
        for f, _ in cls._fields_:
            assert got[(cname, f)] == getattr(cls, f).offset, (cname, f)


def test_plain_c_client(tmp_path):
    """The boundary is usable from plain C: tests/c_client/plan_toy.c, linked
    against librsdb.so, plans BJ config 1 and must reproduce the hand-derived
    layout of tests/golden/toy_config_plan.json."""
    import json
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    lib = os.path.dirname(_capi.LIB_PATH)
    exe = tmp_path / "plan_toy"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c_client", "plan_toy.c"), "-o", str(exe),
                    "-L", lib, "-lrsdb", f"-Wl,-rpath,{lib}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    tok = out.stdout.split()
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "toy_config_plan.json")))
    assert int(tok[tok.index("S") + 1]) == g["S"]
    assert int(tok[tok.index("padding") + 1]) == g["padding"]
    i = tok.index("starts") + 1
    assert [int(x) for x in tok[i:i + len(g["starts"])]] == g["starts"]
    j = tok.index("blocks") + 1
    assert [int(x) for x in tok[j:j + 2]] == [g["rank_blocks_per_rank"]] * 2


def test_tensor_views_alias_the_unit_buffer():
    """a5: R.tensor_views gives each tensor of a unit as a zero-copy
    view at l_t of its m*S buffer -- the oracle's views -- on CPU
    tensors (pure pointer arithmetic, no library compute)."""
    from oracle import dbuffer as OD
    shapes = [(256, 128), (256,), (77,), (40, 50), (2049,)]
    es = [int(np.prod(s)) for s in shapes]
    gs = [min(2048, e) for e in es]
    lay = R.plan(es, gs, 3, elem_bytes=4)
    o = P.plan(es, gs, 3, P.gcoll_elems(4))
    full = torch.zeros(lay.m * lay.S, dtype=torch.float32)
    views = R.tensor_views(lay, full, shapes)
    rng = np.random.default_rng(0)
    logical = rng.normal(size=sum(es)).astype(np.float32)
    off = 0
    for v, s, e, l in zip(views, shapes, es, o.starts):
        assert tuple(v.shape) == s and v.storage_offset() == l and v.untyped_storage().data_ptr() == \
            full.untyped_storage().data_ptr()
        v.copy_(torch.from_numpy(logical[off:off + e]).view(s))  # write through the view
        off += e
    # the buffer is the oracle's placement of the logical tensors, padding untouched (0)
    assert np.array_equal(full.numpy(), OD.place_logical(o, logical))
    with pytest.raises(ValueError):
        R.tensor_views(lay, full, shapes[:-1])
    with pytest.raises(ValueError):
        R.tensor_views(lay, full[:-1], shapes)
    with pytest.raises(ValueError):
        R.tensor_views(lay, full, shapes[:-1] + [(2048,)])


def test_tensor_views_random_plans():
    """SPEC S:511 acceptance: DBuffer aliasing on 200 randomized plans --
    writing every tensor through R.tensor_views reproduces the oracle's
    placement exactly and leaves padding untouched."""
    from oracle import dbuffer as OD
    rng = random.Random(11)
    for _ in range(200):
        n = rng.randint(1, 6)
        shapes = [(rng.randint(1, 9),) if rng.random() < 0.3 else (rng.randint(1, 9), rng.randint(1, 9))
                  for _ in range(n)]
        es = [int(np.prod(s)) for s in shapes]
        gs = [s[-1] * rng.randint(1, 2) if len(s) == 2 and rng.random() < 0.5 else 1 for s in shapes]
        gs = [min(g, e) for g, e in zip(gs, es)]
        m = rng.randint(1, 4)
        lay = R.plan(es, gs, m, elem_bytes=4)
        o = P.plan(es, gs, m, P.gcoll_elems(4))
        full = torch.full((m * lay.S,), -1.0)
        logical = np.arange(1, sum(es) + 1, dtype=np.float32)
        off = 0
        for v, s, e in zip(R.tensor_views(lay, full, shapes), shapes, es):
            v.copy_(torch.from_numpy(logical[off:off + e]).view(s))
            off += e
        assert np.array_equal(full.numpy(), OD.place_logical(o, logical, fill=-1))


def test_arena_sizes_rejects_mixed_worlds():
    """One DBuffer is one FSDP group: units planned for different world sizes
    are refused (EMISMATCH), before any device work."""
    a = R.plan([4096, 100], [2048, 100], 2)
    b = R.plan([4096, 100], [2048, 100], 4)
    R.arena_sizes([a, a], 1)
    with pytest.raises(R.RsdbError) as ei:
        R.arena_sizes([a, b], 1)
    assert ei.value.status == _capi.RSDB_EMISMATCH and "world" in str(ei.value)


def test_fsdp_group_size_selection():
    """P:493 offline FSDP-size choice (scripts/fsdp_sweep.py --select): the
    padding of every candidate equals the oracle planner's, and the choice is
    the least-padding divisor >= min_fsdp, ties to the larger group -- for
    GPT-OSS-120B at 128 rows on 1024 GPUs that is the 5.7 % plateau (m = 512),
    not the 17 % spike at m = 1024."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("fsdp_sweep", os.path.join(ROOT, "scripts", "fsdp_sweep.py"))
    fs = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(fs)
    w = W.gpt_oss_120b(128)
    best, table = fs.select_group_size(w, 1024, 256)
    assert sorted(table) == [256, 512, 1024] and best == 512
    for m, r in table.items():
        pad = tot = 0
        for u in w.units[:2]:  # root + one layer (all layers are identical)
            lay = P.plan([t.numel for t in u.tensors], [P.block_elems(t.shape, t.gran) for t in u.tensors],
                         m, P.gcoll_elems(2))
            k = 1 if u is w.units[0] else len(w.units) - 1
            pad += k * lay.padding
            tot += k * lay.E
        assert r == pytest.approx(pad / tot, rel=1e-12)
    assert table[1024] > 3 * table[512]
    with pytest.raises(ValueError):
        fs.select_group_size(w, 6, 7)


def test_last_error_is_thread_local():
    """Header convention: the error message lives in thread-local storage
    until the next rsdb_* call on the same thread."""
    import threading
    lib = _capi.lib
    one, zero = (C.c_int64 * 1)(4), (C.c_int64 * 1)(0)
    h = C.c_void_p()
    assert lib.rsdb_plan(1, one, zero, 2, 4, 16, C.byref(h)) == _capi.RSDB_EINVAL
    main_msg = lib.rsdb_last_error()
    assert main_msg
    seen = {}

    def other():
        seen["before"] = lib.rsdb_last_error()
        seen["st"] = lib.rsdb_plan(1, one, one, 0, 4, 16, C.byref(C.c_void_p()))
        seen["after"] = lib.rsdb_last_error()

    t = threading.Thread(target=other)
    t.start()
    t.join()
    assert seen["before"] in (b"", None)  # a fresh thread has no error
    assert seen["st"] == _capi.RSDB_EINVAL and seen["after"] and seen["after"] != main_msg
    assert lib.rsdb_last_error() == main_msg  # untouched by the other thread
    assert lib.rsdb_plan(1, one, one, 2, 4, 16, C.byref(h)) == _capi.RSDB_OK
    assert lib.rsdb_last_error() in (b"", None)  # success clears it
    lib.rsdb_layout_free(h)


def test_planner_is_thread_safe_and_deterministic():
    """Header: planning is pure host, deterministic and thread-safe -- eight
    threads planning concurrently (ctypes drops the GIL) reproduce the serial
    layouts exactly."""
    import threading
    u = W.dsv3_moe_unit()
    es = [t.numel for t in u.tensors]
    gs = [R.block_elems(t.shape, t.gran) for t in u.tensors]
    ms = [2, 3, 4, 5, 6, 7, 8, 16]
    serial = {m: (R.plan(es, gs, m).S, R.plan(es, gs, m).starts) for m in ms}
    out, errs = {}, []

    def work(m):
        try:
            for _ in range(20):
                lay = R.plan(es, gs, m)
                out.setdefault(m, set()).add((lay.S, tuple(lay.starts)))
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(m,)) for m in ms]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs
    for m in ms:
        assert out[m] == {(serial[m][0], tuple(serial[m][1]))}


def test_free_functions_accept_null():
    """Header convention: every *_free is a no-op on NULL (run in a child
    process so a crash cannot take the test session down)."""
    import subprocess
    import sys
    frees = [s for s in _header_symbols() if s.endswith("_free")]
    assert len(frees) >= 9
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2602_22437_b200 import _capi as c\n"
            "for f in %r: getattr(c.lib, f)(None)\n"
            "print('ok')\n") % (ROOT, frees)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stderr[-2000:]


def test_planner_parity_large_random_sweep():
    """C++ planner == oracle (S and every start) on 120,000 more random
    instances in two families: tiny (n <= 7, e <= 64, g <= 9, m <= 9) and
    medium (n <= 30, e <= 5000, g <= 600 or whole-tensor, m <= 64), all three
    element sizes (g_coll 4 / 8 / 16)."""
    for seed, (count, nmax, emax, gmax, mmax) in enumerate([(100000, 7, 64, 9, 9),
                                                            (20000, 30, 5000, 600, 64)]):
        rng = random.Random(1000 + seed)
        for _ in range(count):
            n = rng.randint(0, nmax)
            es = [rng.randint(1, emax) for _ in range(n)]
            gs = [min(e, rng.randint(1, gmax)) if rng.random() < 0.7 else e for e in es]
            m = rng.randint(1, mmax)
            eb = rng.choice([1, 2, 4])
            o = P.plan(es, gs, m, P.gcoll_elems(eb))
            c = R.plan(es, gs, m, elem_bytes=eb)
            assert (c.S, c.starts) == (o.S, o.starts), (es, gs, m, eb)
