mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_f.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_f.log
for n in 2 4; do
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
for v in v4cv v4nc v4ld v8cv v8nc v8ld; do
  RSDB_P2P_RS=$v timeout 600 $T --master-port 296$n$RANDOM scripts/sweep_collectives.py --path p2p --layouts ragged --ops rs --sizes 64,256,1024 2>/dev/null | grep '^{' | sed "s/^{/{\"variant\": \"$v\", /"
done
for v in pullcv pullnc push; do
  RSDB_P2P_AG=$v timeout 600 $T --master-port 297$n$RANDOM scripts/sweep_collectives.py --path p2p --layouts ragged --ops ag --sizes 64,256,1024 2>/dev/null | grep '^{' | sed "s/^{/{\"variant\": \"$v\", /"
done
done > gpurun_out/p2p_variants.jsonl
python - <<'PY'
import json
for l in open("gpurun_out/p2p_variants.jsonl"):
    d=json.loads(l); print(d["m"], d["op"], d["variant"], d["mb"], round(d["busbw_gbs"],1), round(d["ms"],3))
PY
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/plain_f.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"adam8" -c 1 -o gpurun_out/prof_f_adam $B > gpurun_out/ncu_f.log 2>&1; echo ncu_rc=$?
