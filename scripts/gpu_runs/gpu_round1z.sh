mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests -q -m gpu -k "fused or fullsize" > gpurun_out/pytest_z.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_z.log
RSDB_RSA_KERNEL=ws timeout 600 python -m pytest tests -q -m gpu -k "fused or fullsize" > gpurun_out/pytest_z_ws.log 2>&1; echo pytest_ws_rc=$?; tail -2 gpurun_out/pytest_z_ws.log
for rep in 1 2 3; do for k in simple ws; do
  RSDB_RSA_KERNEL=$k timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_z_n1_${k}_r$rep.json 2>/dev/null; echo n1_${k}_rc=$?
done; done
P=29200
for n in 2 4; do for rep in 1 2; do for k in simple ws; do P=$((P+1));
  RSDB_RSA_KERNEL=$k timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --no-e2e > gpurun_out/bench_z_n${n}_${k}_r$rep.json 2>/dev/null; echo n${n}_${k}_rc=$?
done; done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_z_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), r["kernel"], round(r["achieved"],1), round(r["frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
