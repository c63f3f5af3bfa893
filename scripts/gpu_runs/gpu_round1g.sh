mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
P=29600
for n in 2 4; do
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
for v in v4cv v4nc v4ld v8cv v8nc v8ld; do
  P=$((P+1)); RSDB_P2P_RS=$v timeout 600 $T --master-port $P scripts/sweep_collectives.py --path p2p --layouts ragged --ops rs --sizes 64,256,1024 2>/dev/null | grep '^{' | sed "s/^{/{\"variant\": \"$v\", /"
done
for v in pullcv pullnc push; do
  P=$((P+1)); RSDB_P2P_AG=$v timeout 600 $T --master-port $P scripts/sweep_collectives.py --path p2p --layouts ragged --ops ag --sizes 64,256,1024 2>/dev/null | grep '^{' | sed "s/^{/{\"variant\": \"$v\", /"
done
done > gpurun_out/p2p_variants.jsonl
python - <<'PY'
import json
for l in open("gpurun_out/p2p_variants.jsonl"):
    d=json.loads(l); print(d["m"], d["op"], d["variant"], d["mb"], round(d["busbw_gbs"],1), round(d["ms"],3))
PY
