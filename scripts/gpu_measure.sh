#!/bin/bash
# Round-2 measurement recipes (run on a gpurun box from the repo root):
#   bash scripts/gpu_measure.sh <name>
# latency  N=2: barrier / copy-engine probe (scripts/probe_barrier.cu) + device-only gated sweep of the p2p
#          collectives (profiles/r2/latency/)
# engines  N=2: NVLink engine probe (scripts/probe_bulk_nvlink.cu)
# rsgrid   N=2: p2p ReduceScatter against its CTA budget (profiles/r2/latency/rs_grid.txt)
# dyn      N=1: dynamic-map 8-bit Adam timing + ncu --set full (profiles/r2/dyn/)
# gemm     N=1: tcgen05 NS GEMM vs cuBLAS at the Muon shapes + ncu --set full
# tiles    N=1: 32x32-tile 8-bit Adam parity, timing, ncu --set full
set -u
name=${1:?usage: gpu_measure.sh latency|engines|rsgrid|dyn|gemm|tiles}
O=gpurun_out/measure_$name; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531"
case $name in
latency)
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/pb scripts/probe_barrier.cu -lcuda &&
    timeout 120 /tmp/pb > $O/probe_barrier.txt 2>&1
  timeout 600 $T2 scripts/sweep_collectives.py --path p2p --layouts ideal --ops barrier,ag,rs \
    --sizes 1,4,16,64,128,256,1024 --gate > $O/p2p_gated.jsonl 2> $O/p2p_gated.err
  timeout 600 $T2 scripts/sweep_collectives.py --path nccl --layouts ideal --ops ag,rs \
    --sizes 1,4,16,64,128,256,1024 --gate > $O/nccl_gated.jsonl 2> $O/nccl_gated.err ;;
engines)
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/pbn scripts/probe_bulk_nvlink.cu &&
    timeout 120 /tmp/pbn > $O/bulk_nvlink.txt 2>&1 ;;
rsgrid)
  for c in 0 592 296 148 74; do
    timeout 300 $T2 scripts/sweep_collectives.py --path p2p --layouts ideal --ops rs --sizes 16,64,128,256 \
      --gate --max-ctas $c > $O/rs_$c.jsonl 2> $O/rs_$c.err
  done ;;
dyn)
  timeout 300 python scripts/kbench.py > $O/kbench.json 2> $O/kbench.err
  KB_REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"adam8_dyn" -c 1 \
    -o $O/adam8_dyn python scripts/kbench.py > $O/ncu.log 2>&1 ;;
gemm)
  for s in "4096 4096 14336" "4096 14336 4096" "8192 8192 8192"; do timeout 120 python scripts/one_gemm.py $s; done > $O/times.txt 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"umma_gemm" -s 3 -c 1 \
    -o $O/umma_big python scripts/one_gemm.py 4096 14336 4096 > $O/ncu.log 2>&1 ;;
tiles)
  timeout 900 python -m pytest tests -q -m gpu -k "tile or Tile or adam8" > $O/pytest_tiles.log 2>&1
  timeout 600 python scripts/bench_tiles.py --reps 20 > $O/bench_tiles.json 2> $O/bench_tiles.err
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"adam8_pair" -c 1 \
    -o $O/adam8_pair python scripts/bench_tiles.py --reps 2 > $O/ncu.log 2>&1 ;;
*) echo "unknown: $name"; exit 2 ;;
esac
echo "$name done: $O"
