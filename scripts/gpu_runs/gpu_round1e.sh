mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_e.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_e.log
B1="python bench.py --steps 30 --warmup 3"
timeout 900 $B1 > gpurun_out/bench_e_n1_p2p.json 2> gpurun_out/bench_e_n1_p2p.err; echo n1p2p_rc=$?
timeout 900 $B1 --collectives nccl > gpurun_out/bench_e_n1_nccl.json 2> gpurun_out/bench_e_n1_nccl.err; echo n1nccl_rc=$?
for n in 2 4; do for c in p2p nccl; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 295$n${#c} bench.py --gpus $n --steps 30 --warmup 3 --collectives $c > gpurun_out/bench_e_n${n}_$c.json 2> gpurun_out/bench_e_n${n}_$c.err; echo n${n}${c}_rc=$?
done; done
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $T4 --master-port 29561 scripts/sweep_collectives.py --path p2p --layouts ragged --sizes 16,64,256,1024 > gpurun_out/sweep_n4_p2p.jsonl 2>/dev/null; echo sw4p_rc=$?
timeout 900 $T4 --master-port 29562 scripts/sweep_collectives.py --path nccl --layouts ragged,even --sizes 16,64,256,1024 > gpurun_out/sweep_n4_nccl.jsonl 2>/dev/null; echo sw4n_rc=$?
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_e_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        po={k:(round(v,3) if isinstance(v,float) else v) for k,v in d["per_op"].items() if k!="bytes_per_rank"}
        print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), "e2e", d["e2e"] and round(d["e2e"]["value"],1), d["clocks"])
        print("   ", json.dumps(po))
    except Exception as e: print(f, "ERR", e)
for f in ["sweep_n4_p2p","sweep_n4_nccl"]:
    for l in open(f"gpurun_out/{f}.jsonl"):
        if l.startswith('{'):
            d=json.loads(l); print(f, d["mb"], d["layout"], d["op"], round(d["busbw_gbs"],1), round(d["ms"],3))
PY
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/plain_e.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"adam8|rs_p2p" -c 2 -o gpurun_out/prof_e $B > gpurun_out/ncu_e.log 2>&1; echo ncu_rc=$?
