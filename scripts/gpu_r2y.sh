O=gpurun_out/r2y; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tiles or adam8_parity or dbuffer" > $O/pytest.log 2>&1; echo rc=$?; tail -2 $O/pytest.log
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --extras tiles_32x32,kernels > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
python -c "import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(json.dumps(d['extras']))"
B3="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --extras tiles_32x32"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"adam8_pair" -c 1 -o $O/adam8_pair $B3 > $O/ncu.log 2>&1; echo ncu_rc=$?
