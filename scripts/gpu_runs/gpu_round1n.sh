mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_n.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_n.log; grep -E "^FAILED|Error" gpurun_out/pytest_n.log | head
timeout 900 python bench.py --no-cpu-baseline --fuse-ag > gpurun_out/bench_n_n1ag.json 2> gpurun_out/bench_n_n1ag.err; echo n1_rc=$?; tail -2 gpurun_out/bench_n_n1ag.err
P=29950
for n in 2 4; do for opt in "--fused-scope dbuffer" "--fused-scope dbuffer --fuse-ag" "--fuse-ag"; do P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n $opt > "gpurun_out/bench_n_n${n}${opt// /}.json" 2> "gpurun_out/bench_n_n${n}${opt// /}.err"; echo "n${n}${opt}_rc=$?"; tail -2 "gpurun_out/bench_n_n${n}${opt// /}.err" | grep -i error
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_n_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        po={k:(round(v,3) if isinstance(v,float) else v) for k,v in d["per_op"].items() if k!="bytes_per_rank"}
        r=d["roofline"]
        print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), r["kernel"], r["bound"], round(r["achieved"],1), round(r["frac"],3), r.get("hbm_frac") and round(r["hbm_frac"],3), "e2e", d["e2e"] and round(d["e2e"]["value"],1), d["clocks"], d.get("gpu_launches"))
        print("   ", json.dumps(po))
    except Exception as e: print(f, "ERR", e)
PY
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/plain_n.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rs_adam|adam8|cast_scale|ag_|rs_p2p|rs_tma|copy_seg|p2p_barrier" --csv --log-file gpurun_out/launches_n.csv $B > gpurun_out/ncu_n1.log 2>&1; echo ncu1_rc=$?
