# round 2: 2-CTA (cta_group::2) tcgen05 Newton-Schulz GEMM
O=gpurun_out/r2p; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 240 python -m pytest tests/test_gpu_ns_gemm.py -q -x -m gpu > $O/pytest_gemm.log 2>&1; rc=$?; echo gemm_rc=$rc; tail -25 $O/pytest_gemm.log
if [ $rc -eq 0 ]; then
timeout 300 python -m pytest tests/test_gpu_muon.py tests/test_gpu_local_ranks.py -q -m gpu > $O/pytest_muon.log 2>&1; echo muon_rc=$?; tail -3 $O/pytest_muon.log
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --extras muon_8b_layer,pcie > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
python -c "import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(json.dumps(d['extras']))"
fi
