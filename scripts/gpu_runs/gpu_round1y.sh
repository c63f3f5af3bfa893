mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -q -m gpu -k "fused or multi or fullsize or dbuffer or adam8 or dynamic or smoke" > gpurun_out/pytest_y.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_y.log; grep -E "^FAILED|Error" gpurun_out/pytest_y.log | head
for rep in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_y_n1_r$rep.json 2> gpurun_out/bench_y_n1.err; echo n1_rc=$?
done
P=29300
for n in 2 4; do P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --no-e2e > gpurun_out/bench_y_n$n.json 2> gpurun_out/bench_y_n$n.err; echo n${n}_rc=$?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_y_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f, round(d["value"],1), round(d["ms_per_step"],3), r["bound"], round(r["achieved"],1), round(r["frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/plain_y.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rs_adam" -c 1 -o gpurun_out/prof_y_fused $B > gpurun_out/ncu_y.log 2>&1; echo ncu_rc=$?
