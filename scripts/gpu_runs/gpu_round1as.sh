mkdir -p gpurun_out
timeout 380 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_final5.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_final5.log; grep -E "^FAILED" gpurun_out/pytest_final5.log | head
