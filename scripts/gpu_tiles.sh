# 32x32-tile 8-bit Adam (adam8_pair_kernel): parity, timing, one full ncu capture
O=gpurun_out/tiles; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -k "tile or Tile or adam8 or fullsize" > $O/pytest_tiles.log 2>&1; echo pytest=$?; tail -2 $O/pytest_tiles.log
timeout 600 python scripts/bench_tiles.py --reps 20 > $O/bench_tiles.json 2> $O/bench_tiles.err; echo bt=$?; tail -c 1500 $O/bench_tiles.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"adam8_pair" -c 1 -o $O/adam8_pair python scripts/bench_tiles.py --reps 2 > $O/ncu.log 2>&1; echo ncu=$?
