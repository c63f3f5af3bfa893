mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python scripts/bench_ring.py > gpurun_out/ring_n1_k2.json 2> gpurun_out/ring_n1.err; echo n1_rc=$?; cat gpurun_out/ring_n1_k2.json; tail -3 gpurun_out/ring_n1.err
P=28700
for n in 2 4; do for k in 2 4; do P=$((P+1));
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P scripts/bench_ring.py --k $k > gpurun_out/ring_n${n}_k$k.json 2> gpurun_out/ring_n${n}_k$k.err; echo n${n}_k${k}_rc=$?; cat gpurun_out/ring_n${n}_k$k.json; grep -i "error\|Traceback" gpurun_out/ring_n${n}_k$k.err | head -3
done; done
