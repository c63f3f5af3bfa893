# round 2 (2 GPUs): NVLink counters of the fused step at N=2 through ncu on rank 0
mkdir -p gpurun_out/r2k
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2k/build.log 2>&1
bash scripts/ncu_nvlink_rank0.sh 2 gpurun_out/r2k
