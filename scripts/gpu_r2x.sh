O=gpurun_out/r2x; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "dynamic or nonfinite or tiny or zero_gradient or full_mantissa" > $O/pytest.log 2>&1; echo rc=$?; tail -2 $O/pytest.log
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --extras kernels > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
python -c "import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(json.dumps(d['extras']['kernels']['adam8_dynamic']))"
