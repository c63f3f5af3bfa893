# mid-session check on 1 GPU: build + smoke, every -m gpu test, default bench (with extras)
O=gpurun_out/mid3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1; echo pytest_rc=$?; tail -2 $O/pytest.log; grep -E "^FAILED|^ERROR" $O/pytest.log | head
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo bench_rc=$?
python - <<'PY'
import json
d=json.loads(open("gpurun_out/mid3/bench_n1.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value","ms_per_step","clocks","gpu_launches")})
print(json.dumps(d["roofline"])); print(json.dumps(d["e2e"]))
for k,v in d["extras"].items(): print(k, json.dumps(v)[:300])
PY
