mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_final3.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke_final3.log
timeout 2000 python -m pytest tests -q -m gpu > gpurun_out/pytest_final3.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_final3.log; grep -E "^FAILED" gpurun_out/pytest_final3.log | head
timeout 900 python bench.py > gpurun_out/bench_final3_n1.json 2> gpurun_out/bench_final3_n1.err; echo n1_rc=$?
P=28000
for n in 2 4; do P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n > gpurun_out/bench_final3_n$n.json 2> gpurun_out/bench_final3_n$n.err; echo n${n}_rc=$?
done
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_final3_ref.json 2>&1; echo ref_rc=$?
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_final3_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); r=d.get("roofline") or {}
        print(f.split('/')[-1], round(d["value"],2), round(d["ms_per_step"],3), r.get("kernel"), r.get("frac") and round(r["frac"],3), d.get("e2e") and round(d["e2e"]["value"],1), d.get("gpu_launches"), d.get("clocks"))
    except Exception as e: print(f, "ERR", e)
PY
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/plain_final3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rs_adam|adam8|cast_scale|ag_|rs_p2p|rs_tma|copy_seg|p2p_barrier|fp8|muon" --csv --log-file gpurun_out/launches_final3.csv $B > gpurun_out/ncu_final3a.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rs_adam" -c 1 -o gpurun_out/prof_final3_fused $B > gpurun_out/ncu_final3b.log 2>&1; echo ncu2_rc=$?
