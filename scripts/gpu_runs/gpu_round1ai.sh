mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
RSDB_P2P_RS=ce timeout 900 python -m pytest tests -q -m gpu -k "multi" > gpurun_out/pytest_ai.log 2>&1; echo pytest_ce_rc=$?; tail -2 gpurun_out/pytest_ai.log; grep -E "FAIL|not bit" gpurun_out/pytest_ai.log | head -5
P=28600
for n in 2 4; do for v in tma ce; do P=$((P+1));
  RSDB_P2P_RS=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P scripts/sweep_collectives.py --path p2p --ops rs --layouts ragged --sizes 64,256,1024 > gpurun_out/rs_${v}_n$n.jsonl 2>/dev/null; echo n${n}_${v}_rc=$?
done; done
P=28650
for n in 2 4; do for v in tma ce; do P=$((P+1));
  RSDB_P2P_RS=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P scripts/sweep_collectives.py --path p2p --ops rs --workload llama1b-layer > gpurun_out/rsu_${v}_n$n.jsonl 2>/dev/null; echo u_n${n}_${v}_rc=$?
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/rs_*.jsonl"))+sorted(glob.glob("gpurun_out/rsu_*.jsonl")):
    for l in open(f):
        try:
            d=json.loads(l); print(f.split('/')[-1], {k:d[k] for k in d if k in ("mb","layout","op","busbw_gbs","ms","workload","wire_gbs","bus_gbs")})
        except Exception as e: print(f, l[:200])
PY
