mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -q -m gpu -k "ring or multi" > gpurun_out/pytest_ag.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_ag.log; grep -E "^FAILED|Error|ring|assert" gpurun_out/pytest_ag.log | head -20
