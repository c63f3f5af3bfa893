# Round 2, first GPU call: confirm the R26 kernel (moments and code decision
# spelled with _rn intrinsics) on a B200 -- the xfail(strict=False) test
# test_adam8_codes_exact_r26 must XPASS; if it does, drop the xfail and make
# the code tolerance exact everywhere.  Then re-measure N=1 (the kernel's FP
# instruction mix is unchanged, so the step time should be too).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/r2_smoke.log
timeout 2000 python -m pytest tests -q -m gpu -rxX > gpurun_out/r2_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2_pytest.log; grep -E "^(FAILED|XPASS|XFAIL)" gpurun_out/r2_pytest.log | head -20
timeout 900 python bench.py > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench_n1.err; echo n1_rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2_bench_n1.json").read().strip().splitlines()[-1])
r = d["roofline"]
print(round(d["value"], 1), round(d["ms_per_step"], 3), r["kernel"], round(r["frac"], 3), d["clocks"])
PY
timeout 600 python scripts/bench_tiles.py --reps 20 > gpurun_out/r2_tiles.json 2> gpurun_out/r2_tiles.err; echo tiles_rc=$?; cat gpurun_out/r2_tiles.json
