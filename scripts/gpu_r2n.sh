# round 2 (2 GPUs): NVLink protocol overhead of peer loads alone; ZeRO-3 overlap (RS on its own stream); memory replay
O=gpurun_out/r2n; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
export CUDA_MODULE_LOADING=EAGER
for mode in noag rs; do
timeout 400 ncu --replay-mode application --devices 0 -k regex:"rs_" -c 2 --clock-control none \
  --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum \
  --csv --log-file $O/ncu_nvlink_$mode.csv python scripts/ncu_nvlink_local.py --gpus 2 --steps 2 --mode $mode > $O/ncu_run_$mode.log 2>&1; echo ncu_${mode}_rc=$?; grep -E "nvl|duration" $O/ncu_nvlink_$mode.csv | tail -5 | awk -F'","' '{print $(NF-2), $NF}'
done
unset CUDA_MODULE_LOADING
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29677 bench.py --gpus 2 --steps 20 --no-e2e --extras zero3_overlap > $O/bench_n2.json 2> $O/bench_n2.err; echo bench_rc=$?
python -c "import json;d=json.loads(open('$O/bench_n2.json').read().strip().splitlines()[-1]);print(json.dumps(d['extras']));print(json.dumps(d['roofline']))"
timeout 600 python bench.py --steps 20 --no-e2e --no-cpu-baseline --extras memory_replay,fp8_allgather > $O/bench_n1.json 2> $O/bench_n1.err; echo bench1_rc=$?
python -c "import json;d=json.loads(open('$O/bench_n1.json').read().strip().splitlines()[-1]);print(json.dumps(d['extras']))"
