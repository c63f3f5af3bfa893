# round 2, N GPUs: multi-GPU parity, bench N (extras: per-unit bus GB/s, ZeRO-3 overlap, NVLink counters), NVLS probe
N=${1:-2}
O=gpurun_out/r2m$N
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi topo -m > $O/topo.txt 2>&1
nvidia-smi nvlink -s -i 0 > $O/nvlink_status.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_fullsize.py -q -m gpu > $O/pytest_multi.log 2>&1; echo multi_rc=$?; tail -3 $O/pytest_multi.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $N > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
python - "$O" <<'PY'
import json, sys
d=json.loads(open(sys.argv[1]+"/bench.json").read().strip().splitlines()[-1])
for k in ("value","value_definition","ms_per_step","hbm_gbs_job","ag_rs_bus_gbs_job","clocks"):
    print(k, d.get(k))
print(json.dumps(d["roofline"]))
print(json.dumps(d.get("nvlink_counters")))
x=d.get("extras") or {}
for k in ("per_unit","zero3_overlap","dsv3_ragged_vs_rowwise","muon_8b_layer"):
    v=x.get(k); print(k, json.dumps(v)[:1500] if v else None)
PY
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29612 scripts/probe_symm_mem.py > $O/symm_probe.log 2>&1; echo probe_rc=$?; tail -12 $O/symm_probe.log
