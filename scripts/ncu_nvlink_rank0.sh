# NVLink counters of an N>1 fused-step kernel: rank 0 under ncu (one pass,
# application replay: no kernel replay, so the barrier kernels still meet
# their unprofiled peers), ranks 1..N-1 plain.  Usage: ncu_nvlink_rank0.sh N OUTDIR
N=$1; O=$2; mkdir -p $O
export MASTER_ADDR=127.0.0.1 MASTER_PORT=29655 WORLD_SIZE=$N
B="bench.py --gpus $N --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
for r in $(seq 1 $((N-1))); do
  RANK=$r LOCAL_RANK=$r timeout 600 python $B > $O/rank$r.log 2>&1 &
done
RANK=0 LOCAL_RANK=0 timeout 600 ncu --replay-mode application --clock-control none -k regex:"rs_adam" -c 4 \
  --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --csv --log-file $O/ncu_nvlink_rank0.csv python $B > $O/rank0.log 2>&1
echo ncu_rc=$?
wait
tail -3 $O/rank0.log; cat $O/ncu_nvlink_rank0.csv | tail -30
