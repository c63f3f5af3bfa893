"""Static checks of the oracle / product separation (task rule ③): the oracle
and the CUDA path share no code and neither imports the other; `synth/` (the
only shared module) imports neither; the measurement scripts never run the
oracle; nothing on the product path reads /root/reference at run time."""
import ast
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = "paper_2602_22437_b200"


def _py_files(sub):
    d = os.path.join(ROOT, sub)
    for dp, _, fs in os.walk(d):
        for f in fs:
            if f.endswith(".py"):
                yield os.path.join(dp, f)


def _imports(path):
    tree = ast.parse(open(path).read(), path)
    out = set()
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            out.update(a.name.split(".")[0] for a in node.names)
        elif isinstance(node, ast.ImportFrom) and node.level == 0 and node.module:
            out.add(node.module.split(".")[0])
    return out


@pytest.mark.parametrize("sub,forbidden", [
    ("oracle", {PKG}),
    (PKG, {"oracle"}),
    ("synth", {PKG, "oracle"}),
    ("scripts", {"oracle"}),  # measurement scripts: only tests/, smoke() and bench.py's baseline run the oracle
])
def test_no_cross_imports(sub, forbidden):
    files = list(_py_files(sub))
    assert files
    for f in files:
        bad = _imports(f) & forbidden
        assert not bad, f"{os.path.relpath(f, ROOT)} imports {bad}"


def test_oracle_loads_no_native_library():
    for f in _py_files("oracle"):
        bad = _imports(f) & {"ctypes", "cffi", "torch"}
        assert not bad, f"{os.path.relpath(f, ROOT)} imports {bad}"
        src = open(f).read()
        for needle in ("CDLL(", "cdll.", "load_library", "cpp_extension"):
            assert needle not in src, f"{os.path.relpath(f, ROOT)} uses {needle}"


def test_product_sources_do_not_read_the_reference():
    paths = list(_py_files(PKG)) + [os.path.join(ROOT, "bench.py"),
                                    os.path.join(ROOT, "__graft_entry__.py")]
    csrc = os.path.join(ROOT, PKG, "csrc")
    paths += [os.path.join(csrc, f) for f in os.listdir(csrc)]
    for f in paths:
        src = open(f).read()
        assert "/root/reference" not in src, f"{os.path.relpath(f, ROOT)} mentions /root/reference"


def test_csrc_shares_no_file_with_the_oracle():
    csrc = os.path.join(ROOT, PKG, "csrc")
    for f in os.listdir(csrc):
        src = open(os.path.join(csrc, f), errors="replace").read()
        assert "oracle/" not in src and "oracle." not in src, f
