mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_d.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_d.log
grep -E "rank|FAIL|Error" gpurun_out/pytest_d.log | head -20
for v in direct128 direct256 tma2 tma3; do RSDB_ADAM_KERNEL=$v timeout 300 python scripts/kbench.py 2>/dev/null | tail -1; done > gpurun_out/kbench_d.jsonl
cat gpurun_out/kbench_d.jsonl
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $T --master-port 29531 scripts/sweep_collectives.py --path p2p --layouts ragged > gpurun_out/sweep_n2_p2p.jsonl 2> gpurun_out/sweep_p2p.err; echo sweep_rc=$?
grep '^{' gpurun_out/sweep_n2_p2p.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['mb'], d['layout'], d['op'], d['path'], round(d['busbw_gbs'],1), round(d['ms'],3))"
tail -3 gpurun_out/sweep_p2p.err
for c in p2p nccl; do timeout 900 $T --master-port 2954${#c} bench.py --gpus 2 --steps 20 --warmup 3 --collectives $c > gpurun_out/bench_n2_$c.json 2> gpurun_out/bench_n2_$c.err; echo bench_${c}_rc=$?; tail -2 gpurun_out/bench_n2_$c.err; done
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo bench1_rc=$?
python - <<'PY'
import json
for f in ["bench_n1","bench_n2_p2p","bench_n2_nccl"]:
    try:
        d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, round(d["value"],1), round(d["ms_per_step"],3), json.dumps({k:(round(v,3) if isinstance(v,float) else v) for k,v in d["per_op"].items() if k!="bytes_per_rank"}), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), d["e2e"] and round(d["e2e"]["value"],1))
    except Exception as e: print(f, "ERR", e)
PY
