mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_al.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_al.log; grep -E "^FAILED" gpurun_out/pytest_al.log | head
timeout 300 python scripts/interleave_check.py 2>/dev/null | tail -1
RSDB_STATE_LAYOUT=interleaved timeout 300 python scripts/interleave_check.py 2>/dev/null | tail -1
for rep in 1 2 3; do for L in split interleaved; do
  RSDB_STATE_LAYOUT=$L timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_al_n1_${L}_r$rep.json 2>gpurun_out/bench_al.err; echo n1_${L}_rc=$?
done; done
P=28300
for n in 2 4; do for L in split interleaved; do P=$((P+1));
  RSDB_STATE_LAYOUT=$L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --no-e2e > gpurun_out/bench_al_n${n}_$L.json 2>/dev/null; echo n${n}_${L}_rc=$?
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_al_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); r=d["roofline"]
        print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), round(r["achieved"],1), round(r["frac"],3), d["clocks"]["sm_mhz"])
    except Exception as e: print(f, "ERR", e)
PY
