#!/bin/bash
# full ncu captures (with source) of the two triangle count kernels at C4
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=${1:-s4tc}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_count_warp_kernel -s 1 -c 1 \
  -o gpurun_out/${T}_warp python scripts/prof_tc.py c4 2 > gpurun_out/${T}_ncu_warp.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_count_cta_kernel -s 1 -c 1 \
  -o gpurun_out/${T}_cta python scripts/prof_tc.py c4 2 > gpurun_out/${T}_ncu_cta.log 2>&1
echo done
