mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
RSDB_RSA_BULKST=1 timeout 900 python -m pytest tests -q -m gpu -k "fused or fullsize or dbuffer" > gpurun_out/pytest_ad.log 2>&1; echo pytest_bulk_rc=$?; tail -2 gpurun_out/pytest_ad.log; grep -E "^FAILED|Error" gpurun_out/pytest_ad.log | head -5
RSDB_RSA_BULKST=1 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for rep in 1 2 3; do for k in 0 1; do
  RSDB_RSA_BULKST=$k timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_ad_n1_b${k}_r$rep.json 2>/dev/null; echo n1_b${k}_rc=$?
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_ad_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), round(r["achieved"],1), round(r["frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
