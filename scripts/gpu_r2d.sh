# round 2: new bench line (physical value, extras, host-buffer e2e) + tests + ncu of the current build
mkdir -p gpurun_out/r2d
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2d/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python -m pytest tests -q -m gpu -x -k "step_host or channels or local_ranks" > gpurun_out/r2d/pytest_new.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/r2d/pytest_new.log
timeout 900 python bench.py > gpurun_out/r2d/bench_n1.json 2> gpurun_out/r2d/bench_n1.err; echo n1_rc=$?; tail -c 6000 gpurun_out/r2d/bench_n1.json
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d/launches_n1.csv $B > gpurun_out/r2d/ncu_launch.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rs_adam" -c 1 -o gpurun_out/r2d/rs_adam_n1 $B > gpurun_out/r2d/ncu_full.log 2>&1; echo ncu2_rc=$?
