mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -q -m gpu -k "fused or fullsize or multi or dbuffer" > gpurun_out/pytest_aq.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_aq.log; grep -E "^FAILED" gpurun_out/pytest_aq.log | head
for rep in 1 2 3; do for c in 0 1; do
  RSDB_RSA_COMPACT=$c timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_aq_n1_c${c}_r$rep.json 2>/dev/null; echo n1_c${c}_rc=$?
done; done
P=27900
for n in 2 4; do for rep in 1 2; do for c in 0 1; do P=$((P+1));
  RSDB_RSA_COMPACT=$c timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --no-e2e > gpurun_out/bench_aq_n${n}_c${c}_r$rep.json 2>/dev/null; echo n${n}_c${c}_rc=$?
done; done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_aq_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), round(r["frac"],3))
PY
