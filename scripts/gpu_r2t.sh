O=gpurun_out/r2t; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 400 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "step_host" > $O/pytest.log 2>&1; echo rc=$?; tail -2 $O/pytest.log
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 10 > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
python -c "import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(d['value'], json.dumps(d['e2e']))"
