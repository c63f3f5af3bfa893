mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_final2.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke_final2.log
timeout 2000 python -m pytest tests -q -m gpu > gpurun_out/pytest_final2.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_final2.log; grep -E "^FAILED|Error" gpurun_out/pytest_final2.log | head
timeout 900 python bench.py > gpurun_out/bench_final2_n1.json 2> gpurun_out/bench_final2_n1.err; echo n1_rc=$?
P=29100
for n in 2 4; do P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n > gpurun_out/bench_final2_n$n.json 2> gpurun_out/bench_final2_n$n.err; echo n${n}_rc=$?
done
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_final2_ref.json 2>&1; echo ref_rc=$?
P=29150
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --impl reference --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_final2_ref_n2.json 2>/dev/null; echo ref_n2_rc=$?
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_final2_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); r=d.get("roofline") or {}
        print(f.split('/')[-1], round(d["value"],2), round(d["ms_per_step"],3), r.get("kernel"), r.get("frac") and round(r["frac"],3), d.get("e2e") and round(d["e2e"]["value"],1), d.get("gpu_launches"), d.get("clocks") and d["clocks"].get("sm_mhz"), d.get("cpu_baseline") and round(d["cpu_baseline"]["value"],3))
    except Exception as e: print(f, "ERR", e)
PY
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/plain_final2.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rs_adam|adam8|cast_scale|ag_|rs_p2p|rs_tma|copy_seg|p2p_barrier|fp8|muon" --csv --log-file gpurun_out/launches_final2.csv $B > gpurun_out/ncu_final2a.log 2>&1; echo ncu1_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final2_all.csv $B > gpurun_out/ncu_final2b.log 2>&1; echo ncu2_rc=$?
