# round 2: symmetric NS GEMM, cp.async-staged 32x32 tiles; ncu of the dynamic-codec kernel
mkdir -p gpurun_out/r2f
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_ns_gemm.py tests/test_gpu_muon.py -q -x -m gpu > gpurun_out/r2f/pytest_gemm.log 2>&1; echo gemm_rc=$?; tail -4 gpurun_out/r2f/pytest_gemm.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tiles or adam8_parity or dynamic or dbuffer" > gpurun_out/r2f/pytest_tiles.log 2>&1; echo tiles_rc=$?; tail -4 gpurun_out/r2f/pytest_tiles.log
timeout 600 python -m pytest tests/test_gpu_local_ranks.py -q -m gpu > gpurun_out/r2f/pytest_local.log 2>&1; echo local_rc=$?; tail -3 gpurun_out/r2f/pytest_local.log
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --extras kernels,tiles_32x32,muon_8b_layer > gpurun_out/r2f/bench.json 2> gpurun_out/r2f/bench.err; echo bench_rc=$?
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2f/bench.json").read().strip().splitlines()[-1])
x=d["extras"]
print(json.dumps({k:(v if k!="muon_8b_layer" else {kk:vv for kk,vv in v.items() if kk!="roots"}) for k,v in x.items()}, indent=0)[:3500])
PY
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --extras kernels"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"adam8_dyn" -c 1 -o gpurun_out/r2f/adam8_dyn $B > gpurun_out/r2f/ncu_dyn.log 2>&1; echo ncu_dyn_rc=$?
B2="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --extras muon_8b_layer"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"umma_gemm" -s 40 -c 1 -o gpurun_out/r2f/umma_gemm $B2 > gpurun_out/r2f/ncu_umma.log 2>&1; echo ncu_umma_rc=$?
