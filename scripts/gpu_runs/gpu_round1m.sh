mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_m.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_m.log; grep -E "^FAILED|Error|fullsize" gpurun_out/pytest_m.log | head
timeout 900 python bench.py > gpurun_out/bench_m_n1.json 2> gpurun_out/bench_m_n1.err; echo n1_rc=$?; tail -2 gpurun_out/bench_m_n1.err
P=29990
for n in 2 4; do for opt in "" "--fused-scope dbuffer"; do P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n $opt > "gpurun_out/bench_m_n${n}${opt// /}.json" 2>/dev/null; echo n${n}${opt}_rc=$?
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_m_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        po={k:(round(v,3) if isinstance(v,float) else v) for k,v in d["per_op"].items() if k!="bytes_per_rank"}
        r=d["roofline"]
        print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), r["kernel"], r["bound"], round(r["achieved"],1), round(r["frac"],3), r.get("hbm_frac") and round(r["hbm_frac"],3), "e2e", d["e2e"] and round(d["e2e"]["value"],1), d["clocks"], d.get("gpu_launches"))
        print("   ", json.dumps(po))
    except Exception as e: print(f, "ERR", e)
PY
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/plain_m.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_m.csv $B > gpurun_out/ncu_m1.log 2>&1; echo ncu1_rc=$?
timeout 600 $B > gpurun_out/plain_m2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rs_adam" -c 1 -o gpurun_out/prof_m_fused $B > gpurun_out/ncu_m2.log 2>&1; echo ncu2_rc=$?
