"""-m gpu parity of N3 distributed Muon (rsdb_muon_*, Algorithm 2)
against oracle/muon.py (fp64) at world 1; world 2-8 in
test_gpu_local_ranks.py (logical ranks on one GPU) and test_gpu_multi.py.

Tolerances: momentum buffer rtol 1e-6; the orthogonalised
update o (recovered from the master change) per matrix within relative
Frobenius 1e-4 for the fp32 Newton-Schulz (numpy fp32 runs of the same
algorithm differ from fp64 by ~2e-6) and 3e-2 for the bf16 tensor-core mode
(bf16-rounding emulation differs by ~1.1e-2); tensors Muon skips and padding
are untouched; the bf16 shard is RNE(master) exactly."""
import pytest

from parity_cases import MUON_SHAPES, muon_case
from rank_ctx import ProcCtx, drive_proc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_muon_world1(precision):
    ctx = ProcCtx(0, 1)
    drive_proc(muon_case(ctx, MUON_SHAPES, 0, 2, precision))
    assert not ctx.msgs, ctx.msgs


def test_muon_big_matrix_world1():
    ctx = ProcCtx(0, 1)
    drive_proc(muon_case(ctx, [(512, 1536), None, (1536, 512)], 1, 1, "f32"))
    assert not ctx.msgs, ctx.msgs
