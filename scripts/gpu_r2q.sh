O=gpurun_out/r2q; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python scripts/one_gemm.py 4096 14336 4096
timeout 300 ncu --set full --clock-control none -k regex:"umma_gemm" -s 3 -c 1 -o $O/umma2 python scripts/one_gemm.py 4096 14336 4096 > $O/ncu.log 2>&1; echo ncu_rc=$?
