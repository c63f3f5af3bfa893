mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_final4_n1.json 2> gpurun_out/bench_final4_n1.err; echo n1_rc=$?
P=27800
for n in 2 4; do P=$((P+1));
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n > gpurun_out/bench_final4_n$n.json 2> gpurun_out/bench_final4_n$n.err; echo n${n}_rc=$?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_final4_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); r=d.get("roofline") or {}
        print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), r.get("frac") and round(r["frac"],3), d.get("e2e") and round(d["e2e"]["value"],1), d.get("clocks"))
    except Exception as e: print(f, "ERR", e)
PY
