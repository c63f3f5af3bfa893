mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python scripts/bench_muon.py > gpurun_out/muon2_n1_bf16.json 2> gpurun_out/muon2_n1.err; echo n1_rc=$?; cat gpurun_out/muon2_n1_bf16.json; tail -2 gpurun_out/muon2_n1.err
P=28900
for n in 2 4; do for prec in bf16 f32; do P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P scripts/bench_muon.py --precision $prec > gpurun_out/muon2_n${n}_$prec.json 2> gpurun_out/muon2_n${n}_$prec.err; echo n${n}_${prec}_rc=$?; cat gpurun_out/muon2_n${n}_$prec.json; grep -i "error\|Traceback" gpurun_out/muon2_n${n}_$prec.err | head -3
done; done
