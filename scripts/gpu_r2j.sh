# round 2 (2 GPUs): paired tiles with 2 stages; NVLink counter probe
mkdir -p gpurun_out/r2j
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2j/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tiles" > gpurun_out/r2j/pytest.log 2>&1; echo rc=$?; tail -2 gpurun_out/r2j/pytest.log
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --extras tiles_32x32 > gpurun_out/r2j/bench.json 2> gpurun_out/r2j/bench.err; echo bench_rc=$?
python -c "import json;d=json.loads(open('gpurun_out/r2j/bench.json').read().strip().splitlines()[-1]);print(json.dumps(d['extras']))"
timeout 120 python scripts/probe_nvlink_counters.py > gpurun_out/r2j/nvlink_probe.log 2>&1; echo probe_rc=$?; cat gpurun_out/r2j/nvlink_probe.log | head -80
