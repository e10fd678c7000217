#!/bin/bash
# ncu --set full of the two C4 triangle count kernels (one launch each)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s2ntc}
for K in tc_count_warp_kernel tc_count_cta_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$K" -c 1 -o gpurun_out/${T}_$K python scripts/prof_tc.py c4 1 > gpurun_out/${T}_ncu_$K.log 2>&1
done
echo done
