mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -q -m gpu -k "multi" > gpurun_out/pytest_ak.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_ak.log; grep -E "FAIL|rank [0-9]\]" gpurun_out/pytest_ak.log | head -20
P=28400
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 3 > gpurun_out/bench_ak_n3.json 2> gpurun_out/bench_ak_n3.err; echo n3_rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_ak_n3.json').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],3), d['roofline']['frac'], d['e2e']['value'])"
