mkdir -p gpurun_out/r2c
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2c/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/r2c/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2c/pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/r2c/pytest.log; grep -E "^FAILED" gpurun_out/r2c/pytest.log | head
timeout 600 python bench.py > gpurun_out/r2c/bench_n1.json 2> gpurun_out/r2c/bench_n1.err; echo n1_rc=$?; cat gpurun_out/r2c/bench_n1.json
