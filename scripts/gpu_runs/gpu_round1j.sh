mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_j.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_j.log; grep -E "FAILED|Error" gpurun_out/pytest_j.log | head
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_j_n1.json 2> gpurun_out/bench_j_n1.err; echo n1_rc=$?; tail -c 2500 gpurun_out/bench_j_n1.json
P=29900
for n in 2 4; do P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n > gpurun_out/bench_j_n$n.json 2> gpurun_out/bench_j_n$n.err; echo n${n}_rc=$?
  P=$((P+1)); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P scripts/bench_rowwise.py --path p2p > gpurun_out/rowwise_j_n$n.jsonl 2>/dev/null; echo rw${n}_rc=$?
  for w in llama8b-layer llama8b-root dsv3 llama1b-layer llama1b-root; do for pth in p2p nccl; do P=$((P+1));
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P scripts/sweep_collectives.py --workload $w --path $pth 2>/dev/null | grep '^{'
  done; done >> gpurun_out/units_j.jsonl
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_j_n*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        po={k:(round(v,3) if isinstance(v,float) else v) for k,v in d["per_op"].items() if k!="bytes_per_rank"}
        print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), "e2e", d["e2e"] and round(d["e2e"]["value"],1), d["clocks"], d.get("cpu_baseline") and round(d["cpu_baseline"]["value"],3))
        print("   ", json.dumps(po))
    except Exception as e: print(f, "ERR", e)
for l in open("gpurun_out/units_j.jsonl"):
    d=json.loads(l); print(d["workload"], d["m"], d["path"], d["op"], "S", d["S"], "pad", d["pad"], round(d["ms"],3), "bus", round(d["busbw_gbs"],1), "good", round(d["goodput_gbs"],1))
for f in sorted(glob.glob("gpurun_out/rowwise_j_n*.jsonl")):
    for l in open(f):
        if l.startswith("{"): print(f, l.strip()[:300])
PY
