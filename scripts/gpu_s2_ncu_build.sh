#!/bin/bash
# ncu --set full of one launch each of the build's non-sort kernels at C4
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2nb}
for K in segment_kernel pack_kernel presence_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$K" -c 1 -o gpurun_out/${T}_$K python scripts/prof_build.py c4 1 > gpurun_out/${T}_ncu_$K.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^pr_spmv" -s 3 -c 1 -o gpurun_out/${T}_pr_spmv python scripts/prof_pagerank.py c4 1 > gpurun_out/${T}_ncu_pr.log 2>&1
echo done
