mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
P=28500
for n in 4 2; do for rep in 1 2; do for s in 2 3; do P=$((P+1));
  RSDB_RSA_STAGES=$s timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --no-e2e > gpurun_out/bench_aj_n${n}_st${s}_r$rep.json 2>/dev/null; echo n${n}_st${s}_rc=$?
done; done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_aj_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), round(r["achieved"],1), round(r["frac"],3))
PY
