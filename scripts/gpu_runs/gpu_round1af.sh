mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for opt in "--collectives nccl" "--no-fuse-adam" "--fused-scope unit" "--no-fuse-ag" "--layers 32"; do
  timeout 600 python bench.py --steps 20 --no-cpu-baseline $opt > "gpurun_out/bench_af_n1${opt// /}.json" 2> "gpurun_out/bench_af_n1${opt// /}.err"; echo "n1 $opt rc=$?"; grep -i "error\|Traceback" "gpurun_out/bench_af_n1${opt// /}.err" | head -3
done
P=28800
for opt in "--collectives nccl" "--no-fuse-adam" "--fused-scope unit --no-fuse-ag"; do P=$((P+1));
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --steps 20 $opt > "gpurun_out/bench_af_n2${opt// /}.json" 2> "gpurun_out/bench_af_n2${opt// /}.err"; echo "n2 $opt rc=$?"; grep -i "error\|Traceback" "gpurun_out/bench_af_n2${opt// /}.err" | head -3
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_af_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); r=d["roofline"]
        print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), r["kernel"], round(r["frac"],3), d["e2e"] and round(d["e2e"]["value"],1), d["gpu_launches"], d.get("nccl_calls"))
    except Exception as e: print(f, "ERR", e)
PY
