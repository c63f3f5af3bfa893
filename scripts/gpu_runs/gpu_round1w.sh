mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for w in llama1b llama8b dsv3; do
  timeout 600 python scripts/fsdp_sweep.py --workload $w --ms 2,4,8,16,64 --measure > gpurun_out/sweep_mem_$w.jsonl 2> gpurun_out/sweep_mem_$w.err; echo ${w}_rc=$?; tail -2 gpurun_out/sweep_mem_$w.err
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_w_n1.json 2> gpurun_out/bench_w_n1.err; echo n1_rc=$?; tail -2 gpurun_out/bench_w_n1.err
P=29400
for n in 2 4; do P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n > gpurun_out/bench_w_n$n.json 2> gpurun_out/bench_w_n$n.err; echo n${n}_rc=$?; grep -i error gpurun_out/bench_w_n$n.err | head -3
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_w_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f, round(d["value"],1), round(d["ms_per_step"],3), d["e2e"])
PY
