mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_ao.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_ao.log; grep -E "^FAILED" gpurun_out/pytest_ao.log | head
for rep in 1 2; do for v in prev cur; do
  if [ $v = prev ]; then export RSDB_LIB=$PWD/paper_2602_22437_b200/librsdb_prev.so; else unset RSDB_LIB; fi
  timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_ao_n1_${v}_r$rep.json 2>/dev/null; echo n1_${v}_rc=$?
done; done
unset RSDB_LIB
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_ao_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), round(r["frac"],3), d["clocks"]["sm_mhz"])
PY
