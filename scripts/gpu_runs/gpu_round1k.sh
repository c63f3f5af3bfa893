mkdir -p gpurun_out
nvidia-smi -L | wc -l
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -rs > gpurun_out/pytest_k.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_k.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1"
timeout 900 $T --master-port 29951 bench.py --gpus 8 > gpurun_out/bench_k_n8_p2p.json 2> gpurun_out/bench_k_n8_p2p.err; echo n8p2p_rc=$?
timeout 900 $T --master-port 29952 bench.py --gpus 8 --collectives nccl > gpurun_out/bench_k_n8_nccl.json 2> gpurun_out/bench_k_n8_nccl.err; echo n8nccl_rc=$?
P=29960
for w in llama8b-layer llama8b-root dsv3 llama1b-layer llama1b-root; do for pth in p2p nccl; do P=$((P+1));
  timeout 600 $T --master-port $P scripts/sweep_collectives.py --workload $w --path $pth 2>/dev/null | grep '^{'
done; done > gpurun_out/units_k.jsonl
P=$((P+1)); timeout 900 $T --master-port $P scripts/sweep_collectives.py --path nccl > gpurun_out/sweep_k_nccl.jsonl 2>/dev/null; echo swn_rc=$?
P=$((P+1)); timeout 900 $T --master-port $P scripts/sweep_collectives.py --path p2p --layouts ragged > gpurun_out/sweep_k_p2p.jsonl 2>/dev/null; echo swp_rc=$?
P=$((P+1)); timeout 900 $T --master-port $P scripts/bench_rowwise.py --path p2p > gpurun_out/rowwise_k_n8.jsonl 2>/dev/null; echo rw_rc=$?
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_k_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        po={k:(round(v,3) if isinstance(v,float) else v) for k,v in d["per_op"].items() if k!="bytes_per_rank"}
        print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), "e2e", d["e2e"] and round(d["e2e"]["value"],1), d["clocks"])
        print("   ", json.dumps(po))
    except Exception as e: print(f, "ERR", e)
for fn in ["units_k","sweep_k_nccl","sweep_k_p2p"]:
    for l in open(f"gpurun_out/{fn}.jsonl"):
        if not l.startswith("{"): continue
        d=json.loads(l); print(fn, d["workload"], d["mb"], d["layout"], d["m"], d["path"], d["op"], "pad", d["pad"], round(d["ms"],3), "bus", round(d["busbw_gbs"],1), "good", round(d["goodput_gbs"],1))
for l in open("gpurun_out/rowwise_k_n8.jsonl"):
    if l.startswith("{"): print(l.strip()[:300])
PY
