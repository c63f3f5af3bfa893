# round 2 (4 GPUs): multi-GPU parity at 2/3/4, bench N=2 and N=4 with extras, NVLink counters via ncu
O=gpurun_out/r2m4
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for n in 2 4; do
  timeout 200 python scripts/ncu_nvlink_local.py --gpus $n --steps 5 > $O/local_n$n.json 2> $O/local_n$n.err; rc=$?; echo local_n${n}_rc=$rc; tail -c 600 $O/local_n$n.json; tail -3 $O/local_n$n.err
  [ $rc -eq 0 ] || continue
  timeout 600 ncu --replay-mode application --devices 0 -k regex:"rs_adam" -c 2 --clock-control none \
    --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --csv --log-file $O/ncu_nvlink_n$n.csv python scripts/ncu_nvlink_local.py --gpus $n --steps 3 > $O/ncu_run_n$n.log 2>&1; echo ncu_n${n}_rc=$?; tail -6 $O/ncu_nvlink_n$n.csv
done
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_fullsize.py -q -m gpu > $O/pytest_multi.log 2>&1; echo multi_rc=$?; tail -3 $O/pytest_multi.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n bench.py --gpus $n > $O/bench_n$n.json 2> $O/bench_n$n.err; echo bench_n${n}_rc=$?
  python - $O/bench_n$n.json <<'PY'
import json, sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value","ms_per_step","hbm_gbs_job","ag_rs_bus_gbs_job")})
print(json.dumps(d["roofline"]))
x=d.get("extras") or {}
for k in ("per_unit","zero3_overlap","fp8_allgather","muon_8b_layer"):
    v=x.get(k); print(k, json.dumps(v)[:900] if v else None)
PY
done
