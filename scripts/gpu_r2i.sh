# round 2: branch-free dynamic codec (fp64 exact quotient), paired 32x32 tiles
mkdir -p gpurun_out/r2i
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2i/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tiles or dynamic or nonfinite or tiny or zero_gradient or full_mantissa" > gpurun_out/r2i/pytest.log 2>&1; echo rc=$?; tail -4 gpurun_out/r2i/pytest.log
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --extras kernels,tiles_32x32 > gpurun_out/r2i/bench.json 2> gpurun_out/r2i/bench.err; echo bench_rc=$?
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2i/bench.json").read().strip().splitlines()[-1])
print(json.dumps(d["extras"], indent=0)[:2000])
PY
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --extras kernels"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"adam8_dyn" -c 1 -o gpurun_out/r2i/adam8_dyn $B > gpurun_out/r2i/ncu_dyn.log 2>&1; echo ncu_dyn_rc=$?
B3="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --extras tiles_32x32"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"adam8_pair" -c 1 -o gpurun_out/r2i/adam8_pair $B3 > gpurun_out/r2i/ncu_pair.log 2>&1; echo ncu_pair_rc=$?
