mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -q -m gpu -k "multi" > gpurun_out/pytest_ab.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_ab.log; grep -E "^FAILED|Error|tiles" gpurun_out/pytest_ab.log | head
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/stream_mix scripts/stream_mix.cu && timeout 300 gpurun_out/stream_mix > gpurun_out/stream_mix.jsonl; echo mix_rc=$?; cat gpurun_out/stream_mix.jsonl
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_ab_n1.json 2>/dev/null; echo n1_rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_ab_n1.json').read().strip().splitlines()[-1]); print(d['roofline']['frac'], d['step_ms'], d['clocks'])"
