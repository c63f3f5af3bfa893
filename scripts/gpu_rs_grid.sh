# p2p ReduceScatter vs CTA budget at N=2 (device-only gated sweep)
O=gpurun_out/rsgrid; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for c in 0 1184 592 296 148 74; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 scripts/sweep_collectives.py --path p2p --layouts ideal --ops rs --sizes 16,64,128,256 --gate --max-ctas $c > $O/rs_$c.jsonl 2> $O/rs_$c.err
python - $O/rs_$c.jsonl $c <<'PY'
import json,sys
print(sys.argv[2], [(json.loads(l)["mb"], round(json.loads(l)["ms"]*1e3,1), round(json.loads(l)["busbw_gbs"])) for l in open(sys.argv[1]) if l.startswith("{")])
PY
done
