# round 2: extras (symmetric NS GEMM, staged tiles) + ncu of the dynamic-codec and tcgen05 kernels + default bench
mkdir -p gpurun_out/r2g
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g/build.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --extras kernels,tiles_32x32,muon_8b_layer > gpurun_out/r2g/bench.json 2> gpurun_out/r2g/bench.err; echo bench_rc=$?
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2g/bench.json").read().strip().splitlines()[-1])
x=d["extras"]
print(json.dumps({k:(v if k!="muon_8b_layer" else {kk:vv for kk,vv in v.items() if kk!="roots"}) for k,v in x.items()}, indent=0)[:3500])
PY
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --extras kernels"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"adam8_dyn" -c 1 -o gpurun_out/r2g/adam8_dyn $B > gpurun_out/r2g/ncu_dyn.log 2>&1; echo ncu_dyn_rc=$?
B2="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --extras muon_8b_layer"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"umma_gemm" -s 40 -c 1 -o gpurun_out/r2g/umma_gemm $B2 > gpurun_out/r2g/ncu_umma.log 2>&1; echo ncu_umma_rc=$?
B3="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --extras tiles_32x32"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"adam8_tma" -c 1 -o gpurun_out/r2g/adam8_tiles $B3 > gpurun_out/r2g/ncu_tiles.log 2>&1; echo ncu_tiles_rc=$?
timeout 900 python bench.py > gpurun_out/r2g/bench_default.json 2> gpurun_out/r2g/bench_default.err; echo default_rc=$?
