mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -q -m gpu -k "dynamic" > gpurun_out/pytest_ae.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_ae.log; grep -E "^FAILED|Error|assert" gpurun_out/pytest_ae.log | head -5
RSDB_ADAM_DYN=direct timeout 900 python -m pytest tests -q -m gpu -k "dynamic" > gpurun_out/pytest_ae_direct.log 2>&1; echo pytest_direct_rc=$?; tail -1 gpurun_out/pytest_ae_direct.log
for rep in 1 2; do
timeout 600 python scripts/kbench.py > gpurun_out/kbench_ae_tma_r$rep.json 2>/dev/null; echo k_rc=$?; cat gpurun_out/kbench_ae_tma_r$rep.json
RSDB_ADAM_DYN=direct timeout 600 python scripts/kbench.py > gpurun_out/kbench_ae_direct_r$rep.json 2>/dev/null; echo kd_rc=$?; cat gpurun_out/kbench_ae_direct_r$rep.json
done
