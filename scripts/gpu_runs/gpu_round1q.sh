mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_q.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_q.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_q.log; grep -E "^FAILED|Error" gpurun_out/pytest_q.log | head
timeout 900 python bench.py > gpurun_out/bench_q_n1.json 2> gpurun_out/bench_q_n1.err; echo n1_rc=$?
P=29700
for n in 2 4; do P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n > gpurun_out/bench_q_n$n.json 2> gpurun_out/bench_q_n$n.err; echo n${n}_rc=$?
done
P=29750
for n in 2 4; do for opt in "--no-fuse-ag" "--fused-scope unit" "--collectives nccl"; do P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n $opt --no-e2e > "gpurun_out/bench_q_n${n}${opt// /}.json" 2>/dev/null; echo "n${n}${opt}_rc=$?"
done; done
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_q_ref.json 2>&1; echo ref_rc=$?
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_q_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        r=d.get("roofline") or {}
        print(f.split('/')[-1], round(d["value"],2), round(d["ms_per_step"],3), r.get("kernel"), r.get("bound"), r.get("achieved") and round(r["achieved"],1), r.get("frac") and round(r["frac"],3), r.get("hbm_frac") and round(r["hbm_frac"],3), d.get("clocks") and d["clocks"].get("sm_mhz"), d.get("clocks") and d["clocks"].get("reasons"), d.get("e2e") and round(d["e2e"]["value"],1), d.get("gpu_launches"), d.get("cpu_baseline") and round(d["cpu_baseline"]["value"],3))
    except Exception as e: print(f, "ERR", e)
PY
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/plain_q.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rs_adam|adam8|cast_scale|ag_|rs_p2p|rs_tma|copy_seg|p2p_barrier" --csv --log-file gpurun_out/launches_q.csv $B > gpurun_out/ncu_q1.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rs_adam" -c 1 -o gpurun_out/prof_q_fused $B > gpurun_out/ncu_q2.log 2>&1; echo ncu2_rc=$?
