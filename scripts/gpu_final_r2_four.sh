# round 2 final check on 4 GPUs: multi-GPU parity, bench N=4 (N=2 and the NCCL baselines ran on earlier boxes:
# profiles/r2/final3m), NVLink counters at N=4 (single process driving the 4 GPUs)
O=gpurun_out/final7m; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_fullsize.py -q -m gpu > $O/pytest_multi.log 2>&1; echo multi_rc=$?; tail -2 $O/pytest_multi.log
timeout 720 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29814 bench.py --gpus 4 --watchdog 650 > $O/bench_n4.json 2> $O/bench_n4.err; echo bench_n4_rc=$?
grep -v "^W1019" $O/bench_n4.err | grep -E "File|Thread|Error" | head -20
python - $O/bench_n4.json <<'PY'
import json, sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value","ms_per_step","ag_rs_bus_gbs_job","params_updated_per_s","clocks")})
print(json.dumps(d["roofline"])); print(json.dumps(d["e2e"]))
x=d.get("extras") or {}
for k in ("per_unit","zero3_overlap","fp8_allgather","muon_8b_layer","dsv3_ragged_vs_rowwise"):
    v=x.get(k); print(k, json.dumps(v)[:700] if v else None)
PY
export CUDA_MODULE_LOADING=EAGER
timeout 300 python scripts/ncu_nvlink_local.py --gpus 4 --steps 5 > $O/local_n4.json 2> $O/local_n4.err; rc=$?; echo local_rc=$rc; tail -c 400 $O/local_n4.json
if [ $rc -eq 0 ]; then
timeout 600 ncu --replay-mode application --devices 0 -k regex:"rs_adam" -c 2 --clock-control none \
  --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum \
  --csv --log-file $O/ncu_nvlink_n4.csv python scripts/ncu_nvlink_local.py --gpus 4 --steps 2 > $O/ncu_run_n4.log 2>&1; echo ncu_rc=$?; grep -E "nvl|duration" $O/ncu_nvlink_n4.csv | tail -5 | awk -F'","' '{print $(NF-2), $NF}'
fi
