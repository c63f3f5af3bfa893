mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
P=29700
for cfg in "v8cv push" "tma tma" "v4cv ce" "v8nc pullcv"; do
  set -- $cfg; P=$((P+1))
  RSDB_P2P_RS=$1 RSDB_P2P_AG=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P tests/dist_parity_worker.py > gpurun_out/parity_$1_$2.log 2>&1; echo "parity rs=$1 ag=$2 rc=$? $(grep -h 'dist parity' gpurun_out/parity_$1_$2.log)"
done
for n in 2 4; do
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
for v in v8cv tma; do
  P=$((P+1)); RSDB_P2P_RS=$v timeout 600 $T --master-port $P scripts/sweep_collectives.py --path p2p --layouts ragged --ops rs --sizes 64,256,1024 2>/dev/null | grep '^{' | sed "s/^{/{\"variant\": \"$v\", /"
done
for v in push tma ce; do
  P=$((P+1)); RSDB_P2P_AG=$v timeout 600 $T --master-port $P scripts/sweep_collectives.py --path p2p --layouts ragged --ops ag --sizes 64,256,1024 2>/dev/null | grep '^{' | sed "s/^{/{\"variant\": \"$v\", /"
done
done > gpurun_out/p2p_variants2.jsonl
python - <<'PY'
import json
for l in open("gpurun_out/p2p_variants2.jsonl"):
    d=json.loads(l); print(d["m"], d["op"], d["variant"], d["mb"], round(d["busbw_gbs"],1), round(d["ms"],3))
PY
