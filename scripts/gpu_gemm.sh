# tcgen05 NS GEMM: timings at the Muon shapes + cuBLAS beside, one full ncu capture of the big shape
O=gpurun_out/gemm; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for s in "4096 4096 14336" "4096 14336 4096" "8192 8192 8192" "1024 4096 4096"; do timeout 120 python scripts/one_gemm.py $s; done 2>&1 | tee $O/times.txt
python - <<'PY' 2>&1 | tee -a gpurun_out/gemm/times.txt
import torch
for M,N,K in ((4096,4096,14336),(4096,14336,4096),(8192,8192,8192)):
    a=torch.randn(M,K,device="cuda").bfloat16(); b=torch.randn(N,K,device="cuda").bfloat16()
    for _ in range(3): c=a@b.T
    torch.cuda.synchronize(); e0,e1=torch.cuda.Event(True),torch.cuda.Event(True); e0.record()
    for _ in range(10): c=a@b.T
    e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/10
    print(f"cuBLAS {M}x{N}x{K}: {ms:.4f} ms, {2*M*N*K/ms/1e9:.1f} TFLOP/s")
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"umma_gemm" -s 3 -c 1 -o $O/umma_big python scripts/one_gemm.py 4096 14336 4096 > $O/ncu.log 2>&1; echo ncu=$?
