# round 2: tcgen05 Newton-Schulz GEMM + lane-replicated dynamic codec, first GPU check
mkdir -p gpurun_out/r2e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e/build.log 2>&1
timeout 180 python -m pytest tests/test_gpu_ns_gemm.py -q -x -m gpu > gpurun_out/r2e/pytest_gemm.log 2>&1; echo gemm_rc=$?; tail -15 gpurun_out/r2e/pytest_gemm.log
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_muon.py -q -m gpu -k "dynamic or muon or nonfinite or tiny" > gpurun_out/r2e/pytest_dyn_muon.log 2>&1; echo dm_rc=$?; tail -5 gpurun_out/r2e/pytest_dyn_muon.log
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --extras kernels,muon_8b_layer > gpurun_out/r2e/bench.json 2> gpurun_out/r2e/bench.err; echo bench_rc=$?
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2e/bench.json").read().strip().splitlines()[-1])
print(json.dumps(d["extras"], indent=1)[:3000])
PY
