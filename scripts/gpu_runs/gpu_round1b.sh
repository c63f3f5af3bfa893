mkdir -p gpurun_out
set -x
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -q -m gpu -rs > gpurun_out/pytest_gpu2.log 2>&1; echo pytest_rc=$?
tail -8 gpurun_out/pytest_gpu2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo bench2_rc=$?
tail -3 gpurun_out/bench_n2.err; cat gpurun_out/bench_n2.json
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/plain_b.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"adam8" -c 1 -o gpurun_out/prof_r1_adam $B > gpurun_out/ncu_full_adam.log 2>&1; echo ncu_rc=$?
tail -2 gpurun_out/ncu_full_adam.log
