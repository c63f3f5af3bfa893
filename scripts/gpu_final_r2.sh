# round 2 final check on 1 GPU: build, smoke, pytest -m gpu, default bench, reference arm, ncu launch list + full capture
O=gpurun_out/final6; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1; echo pytest_rc=$?; tail -2 $O/pytest.log; grep -E "^FAILED|^ERROR" $O/pytest.log | head
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo bench_rc=$?
python - <<'PY'
import json
d=json.loads(open("gpurun_out/final6/bench_n1.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value","ms_per_step","clocks","gpu_launches","params_updated_per_s")})
print(json.dumps(d["roofline"])); print(json.dumps(d["e2e"]))
for k,v in d["extras"].items(): print(k, json.dumps(v)[:400])
PY
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.json 2>&1; echo ref_rc=$?
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
timeout 600 $B > $O/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_n1.csv $B > $O/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rs_adam" -c 1 -o $O/rs_adam_n1 $B > $O/ncu_full.log 2>&1; echo ncu2_rc=$?
