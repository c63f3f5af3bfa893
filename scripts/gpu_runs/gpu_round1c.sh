mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_c.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_c.log
for v in direct tma2 tma3 tma4; do RSDB_ADAM_KERNEL=$v timeout 300 python scripts/kbench.py 2>/dev/null | tail -1; done > gpurun_out/kbench_c.jsonl
cat gpurun_out/kbench_c.jsonl
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $T --master-port 29521 scripts/sweep_collectives.py > gpurun_out/sweep_n2_default.jsonl 2> gpurun_out/sweep_err.log; echo sweep_rc=$?
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING timeout 600 $T --master-port 29522 scripts/sweep_collectives.py --sizes 64,1024 --layouts ragged > gpurun_out/sweep_n2_info.jsonl 2> gpurun_out/sweep_n2_info.err; echo info_rc=$?
NCCL_MIN_NCHANNELS=32 timeout 600 $T --master-port 29523 scripts/sweep_collectives.py --sizes 16,64,256,1024 --layouts ragged > gpurun_out/sweep_n2_ch32.jsonl 2>/dev/null; echo ch_rc=$?
NCCL_PROTO=Simple NCCL_MIN_NCHANNELS=64 NCCL_MAX_NCHANNELS=64 timeout 600 $T --master-port 29524 scripts/sweep_collectives.py --sizes 16,64,256,1024 --layouts ragged > gpurun_out/sweep_n2_ch64.jsonl 2>/dev/null; echo ch64_rc=$?
python - <<'PY'
import json
for f in ["sweep_n2_default","sweep_n2_ch32","sweep_n2_ch64"]:
    try:
        for l in open(f"gpurun_out/{f}.jsonl"):
            d=json.loads(l); print(f, d["mb"], d["layout"], d["op"], round(d["busbw_gbs"],1))
    except Exception as e: print(f, e)
PY
grep -iE "NVLS|channel|algo|proto|Ring|Tree" gpurun_out/sweep_n2_info.err | sort | uniq -c | sort -rn | head -30
