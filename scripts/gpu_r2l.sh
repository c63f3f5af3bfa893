# round 2 (2 GPUs): single-process multi-GPU fused step + ncu NVLink counters (EAGER module loading)
O=gpurun_out/r2l; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
export CUDA_MODULE_LOADING=EAGER
timeout 240 python scripts/ncu_nvlink_local.py --gpus 2 --steps 5 > $O/local_n2.json 2> $O/local_n2.err; rc=$?; echo local_rc=$rc; tail -c 800 $O/local_n2.json; tail -8 $O/local_n2.err
if [ $rc -eq 0 ]; then
timeout 500 ncu --replay-mode application --devices 0 -k regex:"rs_adam" -c 2 --clock-control none \
  --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum \
  --csv --log-file $O/ncu_nvlink_n2.csv python scripts/ncu_nvlink_local.py --gpus 2 --steps 3 > $O/ncu_run_n2.log 2>&1; echo ncu_rc=$?; tail -8 $O/ncu_nvlink_n2.csv
fi
