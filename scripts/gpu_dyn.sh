# dynamic-code-map 8-bit Adam: parity, timing, one full ncu capture
O=gpurun_out/dyn4; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -k "dynamic or dyn" > $O/pytest_dyn.log 2>&1; echo pytest=$?; tail -2 $O/pytest_dyn.log
timeout 300 python scripts/kbench.py > $O/kbench.json 2> $O/kbench.err; echo kb=$?; cat $O/kbench.json
KB_REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"adam8_dyn" -c 1 -o $O/adam8_dyn python scripts/kbench.py > $O/ncu.log 2>&1; echo ncu=$?
