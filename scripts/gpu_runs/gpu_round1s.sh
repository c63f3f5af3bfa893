mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -q -m gpu -k "muon or multi" -x > gpurun_out/pytest_s.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_s.log; grep -E "^FAILED|Error|assert|rel err|Muon" gpurun_out/pytest_s.log | head -30
