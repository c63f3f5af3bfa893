mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -q -m gpu -k "multi or fused or fullsize" > gpurun_out/pytest_aa.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_aa.log; grep -E "^FAILED|Error|owner" gpurun_out/pytest_aa.log | head
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_aa_n1.json 2>/dev/null; echo n1_rc=$?
P=29000
for n in 2 4 4; do P=$((P+1));
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --no-e2e > gpurun_out/bench_aa_n${n}_$P.json 2>/dev/null; echo n${n}_rc=$?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_aa_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), round(r["achieved"],1), round(r["frac"],3), d["clocks"])
PY
