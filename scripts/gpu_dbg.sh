# kernel-barrier push AllGather at N=2: parity, gated sweep, full bench with a watchdog
O=gpurun_out/dbg2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_fullsize.py tests/test_gpu_ring.py tests/test_gpu_local_ranks.py -q -m gpu -x > $O/pytest_multi.log 2>&1; echo multi_rc=$?; tail -2 $O/pytest_multi.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 scripts/sweep_collectives.py --path p2p --layouts ideal --ops barrier,ag,rs --sizes 1,4,16,64,128,256,1024 --gate > $O/p2p_gated.jsonl 2> $O/p2p_gated.err; echo sweep=$?
python - <<'PY'
import json
for l in open("gpurun_out/dbg2/p2p_gated.jsonl"):
    if l.startswith("{"):
        d=json.loads(l); print(d["op"], d["mb"], round(d["ms"]*1e3,1), "us", round(d["busbw_gbs"],1))
PY
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --watchdog 500 > $O/bench_n2.json 2> $O/bench_n2.err; echo bench_rc=$?
grep -v "^W1019" $O/bench_n2.err | grep -E "File|Thread|Error" | head -30
python - <<'PY'
import json
d=json.loads(open("gpurun_out/dbg2/bench_n2.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value","ms_per_step","ag_rs_bus_gbs_job","clocks")})
x=d.get("extras") or {}
for k in ("per_unit","zero3_overlap","dsv3_ragged_vs_rowwise","fp8_allgather"):
    print(k, json.dumps(x.get(k))[:600])
PY
