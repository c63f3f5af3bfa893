mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -q -m gpu -k "multi or fullsize or fused" > gpurun_out/pytest_o.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_o.log; grep -E "^FAILED|Error" gpurun_out/pytest_o.log | head
for h in 0 1 2 4 5 8; do
  RSDB_ADAM_HINTS=$h timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/bench_o_n1_h$h.json 2>/dev/null; echo n1_h${h}_rc=$?
done
P=29900
for n in 2 4; do for h in 0 1 5; do P=$((P+1));
  RSDB_ADAM_HINTS=$h timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --fused-scope dbuffer --fuse-ag --steps 50 --no-e2e > gpurun_out/bench_o_n${n}_ag_h$h.json 2>/dev/null; echo n${n}_h${h}_rc=$?
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_o_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        r=d["roofline"]
        print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), r["kernel"], r["bound"], round(r["achieved"],1), round(r["frac"],3), r.get("hbm_frac") and round(r["hbm_frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e: print(f, "ERR", e)
PY
