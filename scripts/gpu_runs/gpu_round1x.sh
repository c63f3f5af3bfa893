mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py -k "adam8_parity or fused or dynamic or cast or tiles" > gpurun_out/sanitizer_memcheck_parity.log 2>&1; echo memcheck_parity_rc=$?; tail -5 gpurun_out/sanitizer_memcheck_parity.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fp8.py tests/test_gpu_muon.py > gpurun_out/sanitizer_memcheck_fp8_muon.log 2>&1; echo memcheck_fp8_muon_rc=$?; tail -5 gpurun_out/sanitizer_memcheck_fp8_muon.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py -k "fused_rs_adam_world1 or adam8_parity" > gpurun_out/sanitizer_racecheck.log 2>&1; echo racecheck_rc=$?; tail -5 gpurun_out/sanitizer_racecheck.log
