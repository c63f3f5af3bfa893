mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -q -m gpu -k "fp8 or multi" > gpurun_out/pytest_r.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_r.log; grep -E "^FAILED|Error|assert" gpurun_out/pytest_r.log | head -20
for rep in 1 2; do for s in 2 3 4; do
  RSDB_RSA_STAGES=$s timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench_r_n1_st${s}_r$rep.json 2>/dev/null; echo n1_st${s}_rc=$?
done; done
P=29600
for s in 2 3 4; do P=$((P+1));
  RSDB_RSA_STAGES=$s timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --no-e2e > gpurun_out/bench_r_n2_st$s.json 2>/dev/null; echo n2_st${s}_rc=$?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_r_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        r=d["roofline"]
        print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), r["bound"], round(r["achieved"],1), round(r["frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e: print(f, "ERR", e)
PY
timeout 600 python scripts/bench_fp8.py > gpurun_out/fp8_n1.json 2> gpurun_out/fp8_n1.err; echo fp8_n1_rc=$?; cat gpurun_out/fp8_n1.json; tail -3 gpurun_out/fp8_n1.err
P=29650
for n in 2 4; do P=$((P+1));
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P scripts/bench_fp8.py > gpurun_out/fp8_n$n.json 2> gpurun_out/fp8_n$n.err; echo fp8_n${n}_rc=$?; cat gpurun_out/fp8_n$n.json; tail -3 gpurun_out/fp8_n$n.err
done
