mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for rep in 1 2 3; do for v in prev cur b40; do
  if [ $v = prev ]; then export RSDB_LIB=$PWD/paper_2602_22437_b200/librsdb_prev.so; elif [ $v = b40 ]; then export RSDB_LIB=$PWD/paper_2602_22437_b200/librsdb_40.so; else unset RSDB_LIB; fi
  timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_an_n1_${v}_r$rep.json 2>gpurun_out/bench_an.err; echo n1_${v}_rc=$?
done; done
unset RSDB_LIB
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_an_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); r=d["roofline"]
        print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), round(r["frac"],3), d["clocks"]["sm_mhz"])
    except Exception as e: print(f, "ERR", e)
PY
tail -3 gpurun_out/bench_an.err
