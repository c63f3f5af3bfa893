O=gpurun_out/r2s; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/smoke.log
timeout 600 python -m pytest tests/test_gpu_ns_gemm.py tests/test_gpu_muon.py tests/test_gpu_parity.py -q -m gpu > $O/pytest.log 2>&1; echo rc=$?; tail -2 $O/pytest.log; grep -E "^FAILED" $O/pytest.log | head
python scripts/one_gemm.py 4096 14336 4096; python scripts/one_gemm.py 4096 4096 14336
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --extras muon_8b_layer,pcie > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
python -c "import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(json.dumps(d['e2e']));print(json.dumps(d['extras']))"
