mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for prec in bf16 f32; do
  timeout 600 python scripts/bench_muon.py --precision $prec > gpurun_out/muon_n1_$prec.json 2> gpurun_out/muon_n1_$prec.err; echo muon_n1_${prec}_rc=$?; cat gpurun_out/muon_n1_$prec.json; tail -2 gpurun_out/muon_n1_$prec.err
done
P=29500
for n in 2 4; do for prec in bf16 f32; do P=$((P+1));
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P scripts/bench_muon.py --precision $prec > gpurun_out/muon_n${n}_$prec.json 2> gpurun_out/muon_n${n}_$prec.err; echo muon_n${n}_${prec}_rc=$?; cat gpurun_out/muon_n${n}_$prec.json; grep -i error gpurun_out/muon_n${n}_$prec.err | head -3
done; done
timeout 300 python scripts/bench_fp8.py --iters 5 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fp8_quant" -c 1 -o gpurun_out/prof_t_fp8 python scripts/bench_fp8.py --iters 1 --samples 1 > gpurun_out/ncu_t_fp8.log 2>&1; echo ncu_fp8_rc=$?
