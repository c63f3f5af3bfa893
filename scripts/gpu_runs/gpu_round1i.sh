mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
P=29800
RSDB_P2P_RS=tma RSDB_P2P_AG=tma timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29799 tests/dist_parity_worker.py > gpurun_out/parity_i.log 2>&1; echo "parity rc=$? $(grep -h 'dist parity' gpurun_out/parity_i.log)"
for n in 2 4; do
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
for v in tma ce push; do
  P=$((P+1)); RSDB_P2P_AG=$v timeout 600 $T --master-port $P scripts/sweep_collectives.py --path p2p --layouts ragged --ops ag --sizes 64,256,1024 2>/dev/null | grep '^{' | sed "s/^{/{\"variant\": \"$v\", /"
done
done > gpurun_out/p2p_variants3.jsonl
python - <<'PY'
import json
for l in open("gpurun_out/p2p_variants3.jsonl"):
    d=json.loads(l); print(d["m"], d["op"], d["variant"], d["mb"], round(d["busbw_gbs"],1), round(d["ms"],3))
PY
for n in 2 4; do for ag in tma ce; do
  P=$((P+1)); RSDB_P2P_RS=tma RSDB_P2P_AG=$ag timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --steps 50 --warmup 3 --no-e2e > gpurun_out/bench_i_n${n}_$ag.json 2> gpurun_out/bench_i_n${n}_$ag.err; echo bench n$n $ag rc=$?
done; done
for n in 2 4; do for pth in p2p nccl; do
  P=$((P+1)); RSDB_P2P_RS=tma RSDB_P2P_AG=tma timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P scripts/bench_rowwise.py --path $pth > gpurun_out/rowwise_n${n}_$pth.jsonl 2> gpurun_out/rowwise_n${n}_$pth.err; echo rowwise n$n $pth rc=$?; cat gpurun_out/rowwise_n${n}_$pth.jsonl | grep '^{'
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_i_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        po={k:(round(v,3) if isinstance(v,float) else v) for k,v in d["per_op"].items() if k!="bytes_per_rank"}
        print(f.split('/')[-1], round(d["value"],1), round(d["ms_per_step"],3), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), d["clocks"])
        print("   ", json.dumps(po))
    except Exception as e: print(f, "ERR", e)
PY
