mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_am.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_am.log; grep -E "^FAILED" gpurun_out/pytest_am.log | head
timeout 600 python bench.py --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
