# copy-engine AllGather with push + stream-memory-operation barriers at N=2: parity (multi-GPU, single-device
# multi-rank, ring), device-only (gated) sweep of the p2p path
O=gpurun_out/lat4; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_fullsize.py tests/test_gpu_ring.py tests/test_gpu_local_ranks.py -q -m gpu > $O/pytest_multi.log 2>&1; echo multi_rc=$?; tail -2 $O/pytest_multi.log; grep -E "^FAILED|^ERROR" $O/pytest_multi.log | head
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 scripts/sweep_collectives.py"
$T --path p2p --layouts ideal --ops barrier,ag,rs --sizes 1,2,4,8,16,32,64,128,256 --gate > $O/p2p_gated.jsonl 2> $O/p2p_gated.err; echo p2p_gated=$?
python - <<'PY'
import json
for l in open("gpurun_out/lat4/p2p_gated.jsonl"):
    if l.startswith("{"):
        d=json.loads(l); print(d["op"], d["mb"], round(d["ms"]*1e3,1), "us", round(d["busbw_gbs"],1))
PY
