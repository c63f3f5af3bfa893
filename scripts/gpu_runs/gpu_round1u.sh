mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -q -m gpu -k "dynamic or adam8" > gpurun_out/pytest_u.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_u.log; grep -E "^FAILED|Error|assert" gpurun_out/pytest_u.log | head -20
timeout 600 python scripts/kbench.py > gpurun_out/kbench_u.json 2> gpurun_out/kbench_u.err; echo kbench_rc=$?; cat gpurun_out/kbench_u.json; tail -3 gpurun_out/kbench_u.err
