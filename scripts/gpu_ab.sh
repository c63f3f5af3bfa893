# A/B of two prebuilt librsdb.so (ab/librsdb_old.so, ab/librsdb_new.so) on one box: bench_tiles + kbench, alternating
O=gpurun_out/ab; mkdir -p $O
for round in 1 2; do
for v in old new; do
  cp ab/librsdb_$v.so paper_2602_22437_b200/librsdb.so
  timeout 600 python scripts/bench_tiles.py --reps 20 > $O/tiles_${v}_$round.json 2>/dev/null
  python - $O/tiles_${v}_$round.json $v <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], "tile", round(d["tile"]["ms_p50"],3), round(d["tile"]["frac"],3), "flat", round(d["flat"]["ms_p50"],3))
PY
done; done
