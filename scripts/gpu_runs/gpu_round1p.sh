mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -q -m gpu -k "multi or fullsize or fused" > gpurun_out/pytest_p.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_p.log; grep -E "^FAILED|Error" gpurun_out/pytest_p.log | head
for rep in 1 2; do for h in 0 1 8; do
  RSDB_ADAM_HINTS=$h timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench_p_n1_h${h}_r$rep.json 2>/dev/null; echo n1_h${h}_rc=$?
done; done
P=29800
for n in 2 4; do for h in 0 1; do P=$((P+1));
  RSDB_ADAM_HINTS=$h timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n > gpurun_out/bench_p_n${n}_h$h.json 2>/dev/null; echo n${n}_h${h}_rc=$?
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_p_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        r=d["roofline"]
        print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), r["kernel"], r["bound"], round(r["achieved"],1), round(r["frac"],3), r.get("hbm_frac") and round(r["hbm_frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["e2e"] and round(d["e2e"]["value"],1), d["gpu_launches"])
    except Exception as e: print(f, "ERR", e)
PY
