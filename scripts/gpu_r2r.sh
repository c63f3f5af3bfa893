O=gpurun_out/r2r; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
echo "== pair (cta_group::2)"; python scripts/one_gemm.py 4096 14336 4096
sed -i 's/const bool pair = M > UG_BM;/const bool pair = false;/' paper_2602_22437_b200/csrc/ns_umma.cu
python -c "import __graft_entry__ as g; g.build()" > $O/build1.log 2>&1
echo "== single CTA"; python scripts/one_gemm.py 4096 14336 4096
timeout 300 ncu --set full --clock-control none -k regex:"umma_gemm" -s 3 -c 1 -o $O/umma1 python scripts/one_gemm.py 4096 14336 4096 > $O/ncu1.log 2>&1; echo ncu_rc=$?
