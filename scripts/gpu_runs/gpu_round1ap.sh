mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -q -m gpu -k "fused or fullsize or multi" > gpurun_out/pytest_ap.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_ap.log; grep -E "^FAILED" gpurun_out/pytest_ap.log | head
for rep in 1 2 3; do for v in base cur; do
  if [ $v = base ]; then export RSDB_LIB=$PWD/paper_2602_22437_b200/librsdb_base.so; else unset RSDB_LIB; fi
  timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_ap_n1_${v}_r$rep.json 2>/dev/null; echo n1_${v}_rc=$?
done; done
P=28100
for n in 2 4; do for rep in 1 2; do for v in base cur; do P=$((P+1));
  if [ $v = base ]; then export RSDB_LIB=$PWD/paper_2602_22437_b200/librsdb_base.so; else unset RSDB_LIB; fi
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --no-e2e > gpurun_out/bench_ap_n${n}_${v}_r$rep.json 2>/dev/null; echo n${n}_${v}_rc=$?
done; done; done
unset RSDB_LIB
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_ap_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), round(r["frac"],3))
PY
