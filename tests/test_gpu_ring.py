"""-m gpu: the K-slot unsharded ring (rsdb_ring_*,
rsdb_unit_set_shard / rsdb_unit_rebind / rsdb_all_gather_shards_p2p) at
world 1.  The case itself (tests/parity_cases.py::ring_case) also runs at
world 2-8 as logical ranks on one GPU (test_gpu_local_ranks.py) and one
process per GPU (test_gpu_multi.py)."""
import pytest

from parity_cases import ring_case
from rank_ctx import ProcCtx, drive_proc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k", [2, 1])
def test_ring_world1(k):
    ctx = ProcCtx(0, 1)
    drive_proc(ring_case(ctx, k=k))
    assert not ctx.msgs, ctx.msgs
