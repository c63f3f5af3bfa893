mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for w in llama1b llama8b dsv3; do
  timeout 600 python scripts/fsdp_sweep.py --workload $w --ms 2,4,8,16,64 --measure > gpurun_out/sweep_mem_$w.jsonl 2> gpurun_out/sweep_mem_$w.err; echo ${w}_rc=$?; tail -2 gpurun_out/sweep_mem_$w.err
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/sweep_mem_*.jsonl")):
    for l in open(f):
        d=json.loads(l)
        print(d["workload"], d["m"], "pad%", round(d["ragged_padding_pct"],3), round(d["fsdp2_dim0_padding_pct"],3), "dbuf GB", round(d["dbuffer_bytes"]/1e9,3), "res", round(d["dbuffer_reserved"]/1e9,3), "fsdp2 req", round(d["fsdp2_requested_bytes"]/1e9,3), "res", round(d["fsdp2_reserved"]/1e9,3), "ratio", round(d["reserved_fsdp2_over_dbuffer"],4))
PY
